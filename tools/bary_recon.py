"""Measurement: on intersecting rows in fp32, how far is the point named by the reported
barycentrics from the reported point (self-consistency), GPU fast build and oracle."""
import sys
from pathlib import Path
ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "oracle")); sys.path.insert(0, str(ROOT / "tests"))
import numpy as np, torch
import oracle, parity
from paper_2105_12415_b200 import device as D, workloads as W
oracle.build()
PK = dict(n_iterative=16, epsilon=1e-6)
def recon(A, B, r, L):
    return np.maximum(parity.rel_err(parity.bary_point(A, r["bary_a"]), r["point_a"], L),
                      parity.rel_err(parity.bary_point(B, r["bary_b"]), r["point_b"], L))
sets = {"cfg1": W.random_pairs(1 << 20, seed=5, sep=(-0.1, 0.5))}
A3, B3 = W.adversarial_pairs(1 << 18)
for k, name in enumerate(W.CFG3_CLASSES):
    sets[f"cfg3_{name}"] = (A3[k << 18:(k + 1) << 18], B3[k << 18:(k + 1) << 18])
for name, (A, B) in sets.items():
    A32, B32 = A.astype(np.float32), B.astype(np.float32)
    out = D.run("hybrid", torch.from_numpy(A32).cuda(), torch.from_numpy(B32).cuda(), D.Params(**PK), strict=False, ids=True)
    torch.cuda.synchronize()
    got = {k: v.cpu().numpy() for k, v in out.items()}
    ref, _, rc = oracle.hybrid(A32, B32, oracle.make_params(**PK), 1e-6, dtype=np.float32, threads=oracle.default_threads())
    L = parity.longest_edge(A32.astype(np.float64), B32.astype(np.float64))
    for who, r in (("gpu", got), ("oracle", ref)):
        rows = (r["ids"][:, 3] & 16) != 0
        e = recon(A32.astype(np.float64), B32.astype(np.float64), {k: v.astype(np.float64) if v.dtype == np.float32 else v for k, v in r.items()}, L)
        ei = e[rows]
        print(name, who, "intersecting", int(rows.sum()), "recon err max %.3g  p99.9 %.3g  frac>1e-4 %.3g  frac>1e-3 %.3g" % (
            ei.max() if len(ei) else 0, np.quantile(ei, 0.999) if len(ei) else 0, (ei > 1e-4).mean() if len(ei) else 0, (ei > 1e-3).mean() if len(ei) else 0),
            "| other rows max %.3g frac>1e-4 %.3g" % (e[~rows].max(), (e[~rows] > 1e-4).mean()),
            "| weight range violation max (a, b) %.3g %.3g" % tuple(
                float(np.max(np.maximum.reduce([-r[k][:, 0].astype(np.float64), -r[k][:, 1].astype(np.float64),
                                                r[k][:, 0].astype(np.float64) + r[k][:, 1] - 1.0, np.zeros(len(e))])))
                for k in ("bary_a", "bary_b")), flush=True)
