"""Run one kernel variant a few times on the cfg1 generator (for ncu captures).

    python tools/kbench.py --variant hybrid --dtype f64 --n 4194304 [--strict] [--reps 3]
"""
import argparse, sys
from pathlib import Path
ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import torch
from paper_2105_12415_b200 import device as D, workloads as W

ap = argparse.ArgumentParser()
ap.add_argument("--variant", default="hybrid")
ap.add_argument("--dtype", default="f64")
ap.add_argument("--n", type=int, default=1 << 22)
ap.add_argument("--strict", action="store_true")
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--aos", action="store_true")
args = ap.parse_args()
dt = torch.float64 if args.dtype == "f64" else torch.float32
A, B = W.random_pairs(args.n)
soa = not args.aos
if soa:
    planes = torch.from_numpy(W.to_soa(A, B)).to("cuda", dt)
    ta, tb = planes[:9], planes[9:]
else:
    ta, tb = torch.from_numpy(A).to("cuda", dt), torch.from_numpy(B).to("cuda", dt)
out = D.alloc_outputs(args.n, dt, "cuda", soa=soa)
st = D.new_stats()
P = D.Params(n_iterative=16, epsilon=1e-6)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for variant in args.variant.split(","):
    for r in range(args.reps):
        e0.record()
        D.run(variant, ta, tb, P, soa=soa, strict=args.strict, out=out, stats=st, n=args.n)
        e1.record()
        torch.cuda.synchronize()
        print(f"{variant} {args.dtype} strict={args.strict} n={args.n}: {e0.elapsed_time(e1):.3f} ms "
              f"{args.n / e0.elapsed_time(e1) / 1e6:.3f} Gpairs/s")
print(D.read_stats(st))
