"""Per-source-line executed warp instructions and stall samples of one kernel
(tools only): python tools/ncu_linecount.py rep.ncu-rep hybrid_kernelIdLb0ELb1 [lib.so] [file:lo-hi ...]"""
import collections
import os
import re
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from ncu_regions import ROOT, line_chains, sass_rows  # noqa: E402

rep, mangled = sys.argv[1], sys.argv[2]
rest = sys.argv[3:]
lib = rest.pop(0) if rest and rest[0].endswith(".so") else os.path.join(ROOT, "paper_2105_12415_b200",
                                                                         "libtricontact_b200.so")
ranges = [(r.split(":")[0], *map(int, r.split(":")[1].split("-"))) for r in rest] or [("tc_pair.cuh", 1, 99999)]
m = re.match(r"(\w+?)I([df])Lb([01])ELb([01])E?(?:Li(\d+)ELi(\d+)E)?((?:Lb[01]E)*)", mangled)
ksub = mangled
if m:
    ksub = f"{m.group(1)}<{'double' if m.group(2) == 'd' else 'float'}, (bool){m.group(3)}, (bool){m.group(4)}"
    if m.group(5):
            ksub += f", (int){m.group(5)}, (int){m.group(6)}" + "".join(f", (bool){b}" for b in re.findall(r"Lb([01])E", m.group(7) or "")) + ">"
        else:
            ksub += ">"
chains = line_chains(lib, mangled)
rows = sass_rows(rep, ksub)
base = min(a for a, *_ in rows)
for fn, lo, hi in ranges:
    inst, smp, ops = collections.Counter(), collections.Counter(), collections.defaultdict(collections.Counter)
    for addr, src, n, s in rows:
        ch = chains.get(addr - base, [])
        hit = [l for f, l in ch if f == fn and lo <= l <= hi]
        if not hit:
            continue
        ln = hit[0]
        inst[ln] += n
        smp[ln] += s
        op = re.sub(r"^@!?U?P\w+\s+", "", src).split()[0].split(".")[0] if src else "?"
        ops[ln][op] += n
    print(f"== {fn}:{lo}-{hi}  warp inst {sum(inst.values())/1e6:.1f}M  samples {sum(smp.values())}")
    for ln in sorted(inst):
        top = ", ".join(f"{o}:{c/1e6:.1f}" for o, c in ops[ln].most_common(4))
        print(f"  {ln:5d} {inst[ln]/1e6:8.2f}M {smp[ln]:7d}  {top}")
