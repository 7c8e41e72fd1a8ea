"""Decompose the hybrid time: iterative alone, hybrid without fallback,
comparison alone on exactly the fallback pairs, full hybrid (cfg1 inputs)."""
import sys
from pathlib import Path
ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import torch
from paper_2105_12415_b200 import device as D, workloads as W

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 24
A, B = W.random_pairs(n)
planes = torch.from_numpy(W.to_soa(A, B)).to("cuda", torch.float64)
ta, tb = planes[:9], planes[9:]
P = D.Params(n_iterative=16, epsilon=1e-6)
out = D.alloc_outputs(n, torch.float64, "cuda", soa=True)


def t(fn, reps=5):
    fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


res = {}
res["iterative"] = t(lambda: D.run("iterative", ta, tb, P, soa=True, out=out, n=n))
kind = out["kind"].clone()
open_ = (kind == 2)
no = torch.zeros(n, dtype=torch.uint8, device="cuda")
res["hybrid_nofb"] = t(lambda: D.run("hybrid", ta, tb, P, soa=True, out=out, n=n, allow=no))
res["hybrid"] = t(lambda: D.run("hybrid", ta, tb, P, soa=True, out=out, n=n))
idx = open_.nonzero().squeeze(1)
m = idx.numel()
sa, sb = ta[:, idx].contiguous(), tb[:, idx].contiguous()
out2 = D.alloc_outputs(m, torch.float64, "cuda", soa=True)
res["comparison_on_fallbacks"] = t(lambda: D.run("comparison", sa, sb, P, soa=True, out=out2, n=m))
res["comparison_all"] = t(lambda: D.run("comparison", ta, tb, P, soa=True, out=out, n=n))
res["n"] = n
res["fallbacks"] = m
res["overhead_ms"] = res["hybrid"] - res["iterative"] - res["comparison_on_fallbacks"]
print(res)
