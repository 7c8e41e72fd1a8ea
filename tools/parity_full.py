"""Full-size parity evidence for the fast build (GPU box; minutes): the fast
hybrid on BASELINE.json cfg3 (4 x 2^20 adversarial pairs) and on 2^22 fresh
cfg1 pairs, against the C oracle with the tie-aware checker of tests/parity.py,
fp64 and fp32.  Prints one report per (set, dtype).

    python tools/parity_full.py > profiles/r02_parity_full.txt
"""
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
sys.path.insert(0, str(ROOT / "oracle"))
import numpy as np
import torch

import oracle
import parity
from paper_2105_12415_b200 import device as D, workloads as W

oracle.build()
PK = dict(n_iterative=16, epsilon=1e-6)
sets = {"cfg3 (4 x 2^20 adversarial)": W.adversarial_pairs(1 << 20, seed=3),
        "cfg1 (2^22 fresh pairs)": W.random_pairs(1 << 22, seed=0, sep=(-0.1, 0.5), start=1 << 23)}
for name, (A, B) in sets.items():
    for dt, tdt in ((np.float64, torch.float64), (np.float32, torch.float32)):
        a = np.ascontiguousarray(A, dt)
        b = np.ascontiguousarray(B, dt)
        ta, tb = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
        st = D.new_stats()
        out = D.run("hybrid", ta, tb, D.Params(**PK), strict=False, ids=True, stats=st)
        torch.cuda.synchronize()
        got = {k: v.cpu().numpy() for k, v in out.items()}
        t0 = time.time()
        rep = parity.compare_fast(oracle, "hybrid", a, b, PK, got, dt)
        rep["check_s"] = round(time.time() - t0, 1)
        rep["stats"] = D.read_stats(st)
        print(f"{name} {np.dtype(dt).name}: {rep}", flush=True)

# Strict build: bit-identical to the oracle (= the reference) on every pair of
# the full cfg1 batch (2^24) and the full cfg3 set, both precisions.
full = {"cfg1 (2^24, the bench batch)": W.random_pairs_mp(1 << 24, seed=0, sep=(-0.1, 0.5)),
        "cfg3 (4 x 2^20 adversarial)": sets["cfg3 (4 x 2^20 adversarial)"]}
for name, (A, B) in full.items():
    for dt, tdt in ((np.float64, torch.float64), (np.float32, torch.float32)):
        a = np.ascontiguousarray(A, dt)
        b = np.ascontiguousarray(B, dt)
        ta, tb = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
        st = D.new_stats()
        out = D.run("hybrid", ta, tb, D.Params(**PK), strict=True, ids=True, stats=st)
        torch.cuda.synchronize()
        got = {k: v.cpu().numpy() for k, v in out.items()}
        del ta, tb, out
        ref, counts, rc = oracle.hybrid(a, b, oracle.make_params(**PK), PK["epsilon"], dtype=dt,
                                        threads=oracle.default_threads())
        diff = {k: int((got[k] != ref[k]).reshape(len(a), -1).any(axis=1).sum()) for k in ref}
        s = D.read_stats(st)
        same_counts = [s["iterative"], s["comparison"], s["fallback"], s["degenerate"]] == list(counts[:4])
        print(f"STRICT {name} {np.dtype(dt).name}: n={len(a)} rows differing per column {diff} "
              f"counters equal {same_counts} rc {rc}", flush=True)
