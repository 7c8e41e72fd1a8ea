"""Attribute ncu warp-stall samples of one kernel to CUDA source lines.

    python tools/ncu_lines.py gpurun_out/prof.ncu-rep <kernel-substring> [lib.so] [top] [mangled-substring]

Reads the SASS source page of the report (per-instruction stall samples) and
the line table of the cubin inside the library (nvdisasm -g), then prints the
source lines (and tc_pair.cuh functions) with the most samples.
"""
import collections
import csv
import io
import os
import re
import subprocess
import sys
import tempfile


def sass_samples(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    out = {}
    kernel = None
    hdr = None
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
                out[kernel].append((int(d["Address"], 16), d["Source"], int(d["Warp Stall Sampling (All Samples)"] or 0)))
            except ValueError:
                pass
    return out


def line_table(lib, mangled_substr):
    tmp = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=tmp, capture_output=True)
    cubins = [f for f in os.listdir(tmp) if f.endswith(".cubin")]
    table = {}
    for cb in cubins:
        txt = subprocess.run(["nvdisasm", "-g", os.path.join(tmp, cb)], capture_output=True, text=True).stdout
        cur_fn = None
        loc = None
        for line in txt.splitlines():
            m = re.match(r"^\.text\.(\S+):\s*$", line)
            if m:
                cur_fn = m.group(1)
                loc = None
                continue
            m = re.search(r'//## File "([^"]+)", line (\d+)', line)
            if m:
                loc = (os.path.basename(m.group(1)), int(m.group(2)))
                continue
            m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", line)
            if m and cur_fn and mangled_substr in cur_fn and loc:
                table[int(m.group(1), 16)] = loc
    return table


def main():
    rep, ksub = sys.argv[1], sys.argv[2]
    lib = sys.argv[3] if len(sys.argv) > 3 else "paper_2105_12415_b200/libtricontact_b200.so"
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
    samples = sass_samples(rep)
    kname = next(k for k in samples if ksub in k)
    mangled = {"hybrid": "hybrid_kernelIdLb0ELb1", "iterative": "iterative_kernelIdLb0ELb1",
               "comparison": "comparison_kernelIdLb0ELb1"}.get(ksub, ksub)
    if len(sys.argv) > 5:  # mangled-name substring given separately from the demangled one
        mangled = sys.argv[5]
    table = line_table(lib, mangled)
    by_line = collections.Counter()
    total = 0
    base = min(a for a, _, _ in samples[kname])
    for addr, src, n in samples[kname]:
        total += n
        by_line[table.get(addr - base, ("?", 0))] += n
    print(f"{kname}: {total} samples, {len(table)} mapped instructions")
    src_cache = {}
    for (f, ln), n in by_line.most_common(top):
        text = ""
        for d in ("paper_2105_12415_b200/csrc",):
            pth = os.path.join(d, f)
            if os.path.exists(pth):
                src_cache.setdefault(pth, open(pth).read().splitlines())
                if 0 < ln <= len(src_cache[pth]):
                    text = src_cache[pth][ln - 1].strip()[:90]
        print(f"{100.0 * n / max(total, 1):6.2f}%  {f}:{ln:<5} {text}")


if __name__ == "__main__":
    main()
