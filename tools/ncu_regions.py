"""Issue accounting of one kernel from an .ncu-rep, per code region (tools only).

Per SASS instruction: warp instructions executed (ncu source page) and its
pipe class; the instruction's inlining chain (nvdisasm -gi of the library that
was profiled) names the region it belongs to -- the iterative sweep, its setup
and epilogue, the fallback phases, the queue / staging / store plumbing.
Reports, per region, warp instructions, FP64-pipe instructions (DFMA/DADD/
DMUL, 2 cycles per warp on B200), ALU-pipe ones (FSEL/SEL/ISETP/LOP3/...,
also half rate, tools/rf_probe.cu) and stall samples.

    python tools/ncu_regions.py gpurun_out/x.ncu-rep hybrid_kernelIdLb0ELb1 [lib.so]
"""
import collections
import csv
import io
import os
import re
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CSRC = os.path.join(ROOT, "paper_2105_12415_b200", "csrc")

FP64 = {"DFMA", "DADD", "DMUL"}
ALU = {"FSEL", "SEL", "ISETP", "LOP3", "SHF", "VIMNMX", "IMNMX", "PLOP3", "P2R", "R2P", "FSETP", "LEA", "PRMT",
       "IABS", "BMSK", "POPC", "FLO", "BREV", "SGXT", "FMNMX"}

# regions: (name, file, signature regex); a function's span runs to its closing brace
REGIONS = [
    ("sweep", "tc_pair.cuh", r"void sweep\(\)"),
    ("iter_init", "tc_pair.cuh", r"void init\(const R\* A, const R\* B"),
    ("iter_epilogue", "tc_pair.cuh", r"void (prelast|finish|points)\("),
    ("iter_strict", "tc_pair.cuh", r"void iterative_pair\("),
    ("phase1", "tc_pair.cuh", r"bool comparison_phase1\("),
    ("phase2", "tc_pair.cuh", r"void comparison_phase2_impl\("),
    ("degenerate", "tc_pair.cuh", r"bool degenerate_tri_t\("),
    ("stage_pair", "tc_kernels.cu", r"void stage_pair\("),
    ("store_rec", "tc_kernels.cu", r"void store_rec(_full)?\("),
    ("load_tri", "tc_kernels.cu", r"void load_tri\("),
    ("stash_pair", "tc_kernels.cu", r"void stash_pair\("),
    ("push", "tc_kernels.cu", r"void push\(int64_t\* q"),
    ("tally", "tc_kernels.cu", r"struct Tally"),
    ("prefetch", "tc_kernels.cu", r"void prefetch_tile\("),
    ("drain", "tc_kernels.cu", r"void drain\(const Src& src"),
    ("ws_kernel_body", "tc_kernels.cu", r"hybrid_ws_kernel\(Args<T> a\)"),
]


def spans():
    out = []
    for name, fn, sig in REGIONS:
        lines = open(os.path.join(CSRC, fn)).read().split("\n")
        for i, l in enumerate(lines):
            if re.search(sig, l):
                depth, started, j = 0, False, i
                while j < len(lines):
                    depth += lines[j].count("{") - lines[j].count("}")
                    started = started or "{" in lines[j]
                    if started and depth <= 0:
                        break
                    j += 1
                out.append((name, fn, i + 1, j + 1))
    return out


def line_chains(lib, mangled):
    tmp = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=tmp, capture_output=True)
    cub = [f for f in os.listdir(tmp) if f.endswith(".cubin")][0]
    txt = subprocess.run(["nvdisasm", "-gi", os.path.join(tmp, cub)], capture_output=True, text=True).stdout
    chains, cur, locs, infn = {}, None, [], False
    for line in txt.splitlines():
        m = re.match(r"^\.text\.(\S+):\s*$", line)
        if m:
            infn = mangled in m.group(1)
            locs = []
            continue
        if not infn:
            continue
        if line.strip().startswith("//## File"):
            if not cur:
                locs = []
            cur = True
            locs += [(os.path.basename(f), int(n)) for f, n in re.findall(r'"([^"]+)", line (\d+)', line)]
            continue
        m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
        if m:
            chains[int(m.group(1), 16)] = list(locs)
            cur = False
    return chains


def sass_rows(rep, ksub):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    out, kernel, hdr = {}, None, None
    for r in csv.reader(io.StringIO(raw)):
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
                out[kernel].append((int(d["Address"], 16), d["Source"].strip(), int(d["Instructions Executed"] or 0),
                                    int(d["Warp Stall Sampling (All Samples)"] or 0)))
            except ValueError:
                pass
    k = [k for k in out if ksub.replace("IdLb0ELb1", "") in k]
    return out[k[0]]


def main():
    rep, mangled = sys.argv[1], sys.argv[2]
    lib = sys.argv[3] if len(sys.argv) > 3 else os.path.join(ROOT, "paper_2105_12415_b200", "libtricontact_b200.so")
    sp = spans()
    chains = line_chains(lib, mangled)
    m = re.match(r"(\w+?)I([df])Lb([01])ELb([01])E?(?:Li(\d+)ELi(\d+)E)?((?:Lb[01]E)*)", mangled)
    ksub = mangled
    if m:
        ksub = f"{m.group(1)}<{'double' if m.group(2) == 'd' else 'float'}, (bool){m.group(3)}, (bool){m.group(4)}"
        if m.group(5):
            ksub += f", (int){m.group(5)}, (int){m.group(6)}" + "".join(f", (bool){b}" for b in re.findall(r"Lb([01])E", m.group(7) or "")) + ">"
        else:
            ksub += ">"
    rows = sass_rows(rep, ksub)
    base = min(a for a, *_ in rows)
    agg = collections.defaultdict(lambda: collections.Counter())
    tot = collections.Counter()
    for addr, src, n, smp in rows:
        op = re.sub(r"^@!?U?P\w+\s+", "", src).split()[0].split(".")[0] if src else "?"
        ch = chains.get(addr - base, [])
        reg = "other"
        for name, fn, lo, hi in sp:
            if any(f == fn and lo <= ln <= hi for f, ln in ch):
                reg = name
                break
        c = agg[reg]
        c["warp_inst"] += n
        c["fp64"] += n if op in FP64 else 0
        c["alu"] += n if op in ALU else 0
        c["samples"] += smp
        for k in ("warp_inst", "fp64", "alu", "samples"):
            tot[k] += c[k] * 0
        tot["warp_inst"] += n
        tot["fp64"] += n if op in FP64 else 0
        tot["alu"] += n if op in ALU else 0
        tot["samples"] += smp
    print(f"{'region':15s} {'warp inst':>11s} {'%inst':>6s} {'fp64':>10s} {'alu':>10s} {'pipe cyc':>10s} {'%samples':>8s}")
    for reg, c in sorted(agg.items(), key=lambda kv: -kv[1]["samples"]):
        pc = 2 * c["fp64"] + 2 * c["alu"]
        print(f"{reg:15s} {c['warp_inst']:11d} {100 * c['warp_inst'] / tot['warp_inst']:6.1f} {c['fp64']:10d} "
              f"{c['alu']:10d} {pc:10d} {100 * c['samples'] / max(tot['samples'], 1):8.1f}")
    print(f"{'total':15s} {tot['warp_inst']:11d} {'':6s} {tot['fp64']:10d} {tot['alu']:10d} "
          f"{2 * tot['fp64'] + 2 * tot['alu']:10d}")


if __name__ == "__main__":
    main()
