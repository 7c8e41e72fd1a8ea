"""Issue-cycle budget of one kernel from an .ncu-rep (read here, no GPU).

Each SASS instruction costs (warp instructions executed) x (2 for an FP64-pipe
instruction -- DFMA/DADD/DMUL/DSETP: 16 FP64 lanes per SM sub-partition --,
else 1); the costs are attributed to source lines with the cubin's line
table (tools/ncu_lines.py) and summed per line and per function region.

    python tools/ncu_issue.py gpurun_out/prof.ncu-rep hybrid [lib.so] [top]
"""
import collections
import csv
import io
import re
import subprocess
import sys

from ncu_lines import line_table

FP64 = re.compile(r"^(@!?U?P\w+\s+)?(DFMA|DADD|DMUL|DSETP)\b")


def sass_counts(rep, ksub):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    out, kernel, hdr = {}, None, None
    for r in rows:
        if r and r[0] == "Kernel Name":
            kernel = r[1]
            out[kernel] = []
            continue
        if r and r[0] == "Address":
            hdr = r
            continue
        if hdr and kernel and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            try:
                out[kernel].append((int(d["Address"], 16), d["Source"].strip(), int(d["Instructions Executed"] or 0)))
            except ValueError:
                pass
    return next(v for k, v in out.items() if ksub in k)


def main():
    rep, ksub = sys.argv[1], sys.argv[2]
    lib = sys.argv[3] if len(sys.argv) > 3 else "paper_2105_12415_b200/libtricontact_b200.so"
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 30
    rows = sass_counts(rep, ksub if ksub != "hybrid" else "hybrid_kernel")
    mangled = {"hybrid": "hybrid_kernelIdLb0ELb1", "iterative": "iterative_kernelIdLb0ELb1",
               "comparison": "comparison_kernelIdLb0ELb1"}.get(ksub, ksub)
    table = line_table(lib, mangled)
    base = min(a for a, _, _ in rows)
    by_line = collections.Counter()
    fp64 = other = 0
    for addr, src, n in rows:
        c = n * (2 if FP64.match(src) else 1)
        if FP64.match(src):
            fp64 += c
        else:
            other += c
        by_line[table.get(addr - base, ("?", 0))] += c
    tot = fp64 + other
    print(f"{ksub}: {tot / 1e9:.3f} G issue cycles (FP64 {fp64 / tot:.1%} of them)")
    for (f, ln), c in by_line.most_common(top):
        print(f"{100.0 * c / tot:6.2f}%  {f}:{ln}")


if __name__ == "__main__":
    main()
