"""Hybrid launches for a DRAM-traffic breakdown under ncu: full record, then reduce-only."""
import sys
from pathlib import Path
ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import torch
from paper_2105_12415_b200 import device as D, workloads as W
n = 1 << 24
A, B = W.random_pairs(n)
planes = torch.from_numpy(W.to_soa(A, B)).to("cuda", torch.float64)
ta, tb = planes[:9], planes[9:]
P = D.Params(n_iterative=16, epsilon=1e-6)
out = D.alloc_outputs(n, torch.float64, "cuda", soa=True)
st = D.new_stats()
for mode in ("full", "reduce", "full", "reduce"):
    D.run("hybrid", ta, tb, P, soa=True, out=out if mode == "full" else {}, stats=st, n=n)
    torch.cuda.synchronize()
print("ok")
