"""Decompose the hybrid's time on cfg1 (tools only): iterative kernel alone,
hybrid with fallback suppressed, comparison on the compacted open pairs, full hybrid.

    python tools/decomp3.py [--dtype f64|f32]
"""
import argparse, ctypes, sys
from pathlib import Path
ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import torch
from paper_2105_12415_b200 import _abi, device as D

ap = argparse.ArgumentParser()
ap.add_argument("--dtype", default="f64")
ap.add_argument("--n", type=int, default=1 << 24)
args = ap.parse_args()
dt = torch.float64 if args.dtype == "f64" else torch.float32
n = args.n
lib = _abi.load()
planes = torch.empty((18, n), dtype=torch.float64, device="cuda")
_abi.check(lib.tc_random_pairs_soa_f64(0, 0, n, -0.1, 0.5, ctypes.c_void_p(planes.data_ptr()), None), "gen")
planes = planes.to(dt)
P = D.Params(n_iterative=16, epsilon=1e-6)
ta, tb = planes[:9], planes[9:]


def timeit(fn, reps=10):
    for _ in range(2):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


out = D.alloc_outputs(n, dt, "cuda", soa=True, ids=True)
st = D.new_stats()
D.run("hybrid", ta, tb, P, soa=True, out=out, ids=True, stats=st)
torch.cuda.synchronize()
fb = (out["ids"][:, 3] & 4) > 0
idx = torch.nonzero(fb).squeeze(1)
m = idx.numel()
ca, cb = ta[:, idx].contiguous(), tb[:, idx].contiguous()
inter = ((out["ids"][idx, 3] & 16) > 0).sum().item()
out2 = D.alloc_outputs(n, dt, "cuda", soa=True)
o_m = D.alloc_outputs(m, dt, "cuda", soa=True)
no_fb = torch.zeros(n, dtype=torch.uint8, device="cuda")
r = {
    "iterative (all n)": timeit(lambda: D.run("iterative", ta, tb, P, soa=True, out=out2)),
    "hybrid, fallback suppressed": timeit(lambda: D.run("hybrid", ta, tb, P, soa=True, out=out2, allow=no_fb)),
    f"comparison on the {m} open pairs (compacted)": timeit(lambda: D.run("comparison", ca, cb, P, soa=True, out=o_m)),
    "comparison (all n)": timeit(lambda: D.run("comparison", ta, tb, P, soa=True, out=out2)),
    "hybrid": timeit(lambda: D.run("hybrid", ta, tb, P, soa=True, out=out2)),
}
print(f"{args.dtype} n={n} open={m} ({m / n:.3f}) of which intersecting {inter}")
for k, v in r.items():
    print(f"  {k:55s} {v:7.3f} ms")
