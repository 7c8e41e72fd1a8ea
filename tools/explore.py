"""Exploration on the GPU: fast-vs-strict agreement and per-variant timings."""
import sys, time
from pathlib import Path
ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "oracle"))
import numpy as np, torch
from paper_2105_12415_b200 import device as D, workloads as W

n = int(sys.argv[1]) if len(sys.argv) > 1 else (1 << 24)
t0 = time.time()
A, B = W.random_pairs(n)
print(f"gen {n} pairs {time.time()-t0:.1f}s", flush=True)
P = D.Params(n_iterative=16, epsilon=1e-6)
L = np.sqrt(np.maximum(((np.roll(A, -1, 1) - A) ** 2).sum(2).max(1), ((np.roll(B, -1, 1) - B) ** 2).sum(2).max(1)))

for dt in (torch.float64, torch.float32):
    ta = torch.from_numpy(A).to("cuda", dt); tb = torch.from_numpy(B).to("cuda", dt)
    planes = torch.from_numpy(W.to_soa(A, B)).to("cuda", dt); sa, sb = planes[:9].contiguous(), planes[9:].contiguous()
    # agreement fast vs strict (hybrid)
    s = D.run("hybrid", ta, tb, P, strict=True, ids=True); f = D.run("hybrid", ta, tb, P, strict=False, ids=True)
    torch.cuda.synchronize()
    ks, kf = s["kind"].cpu().numpy(), f["kind"].cpu().numpy()
    ds, df = s["distance"].cpu().numpy().astype(np.float64), f["distance"].cpu().numpy().astype(np.float64)
    fbs = (s["ids"].cpu().numpy()[:, 3] & 4) > 0; fbf = (f["ids"].cpu().numpy()[:, 3] & 4) > 0
    same = (ks == kf) & (fbs == fbf)
    rel = np.abs(ds - df) / np.maximum(ds, L)
    pa_s, pa_f = s["point_a"].cpu().numpy().astype(np.float64), f["point_a"].cpu().numpy().astype(np.float64)
    prel = np.abs(pa_s - pa_f).max(1) / np.maximum(np.abs(pa_s).max(1), L)
    print(f"{dt}: kind/fb mismatches {int((~same).sum())} of {n}; fallback strict {fbs.mean():.4f} fast {fbf.mean():.4f}")
    print(f"   distance rel err (same path): max {rel[same].max():.3e} p99.99 {np.quantile(rel[same], 0.9999):.3e}")
    print(f"   point_a rel err (same path): max {prel[same].max():.3e} p99.99 {np.quantile(prel[same], 0.9999):.3e} n>1e-9 {(prel[same] > 1e-9).sum()}")
    del s, f
    for variant in ("iterative", "comparison", "hybrid"):
        for strict in (True, False):
            for soa in (False, True):
                for reduce_only in (False, True):
                    xa, xb = (sa, sb) if soa else (ta, tb)
                    out = {} if reduce_only else D.alloc_outputs(n, dt, "cuda", soa=soa)
                    st = D.new_stats()
                    for _ in range(2):
                        D.run(variant, xa, xb, P, soa=soa, strict=strict, out=out, stats=st, n=n)
                    torch.cuda.synchronize()
                    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
                    reps = 5
                    e0.record()
                    for _ in range(reps):
                        D.run(variant, xa, xb, P, soa=soa, strict=strict, out=out, stats=st, n=n)
                    e1.record(); torch.cuda.synchronize()
                    ms = e0.elapsed_time(e1) / reps
                    print(f"  {str(dt):14s} {variant:10s} strict={int(strict)} soa={int(soa)} reduce={int(reduce_only)}: "
                          f"{ms:8.3f} ms  {n/ms/1e6:8.3f} Gpairs/s", flush=True)
                    del out
