"""cfg4-scale parity evidence (GPU box, ~2 min): all 2^28 pairs of BASELINE.json
config 4 (sep U[-0.05, 0.2]) in 2^24-pair chunks (the shards of a 16-way
split), reduce-only hybrid (tc_stats only, as the bench runs it): the strict
build's counters and minimum distance against the C oracle's, and the fast
build's beside them.

    python tools/parity_cfg4.py > profiles/r01_parity_cfg4.txt
"""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))
import numpy as np
import torch

import oracle
from paper_2105_12415_b200 import device as D, workloads as W

oracle.build()
PK = dict(n_iterative=16, epsilon=1e-6)
N, CH = 1 << 28, 1 << 24
names = ("iterative", "comparison", "fallback", "degenerate", "contacts", "intersecting")
acc = {"strict": np.zeros(6, np.int64), "fast": np.zeros(6, np.int64), "oracle": np.zeros(5, np.int64)}
mins = {"strict": np.inf, "fast": np.inf, "oracle": np.inf}
for c0 in range(0, N, CH):
    A, B = W.random_pairs_mp(CH, seed=0, sep=(-0.05, 0.2), start=c0)
    planes = torch.from_numpy(W.to_soa(A, B)).cuda()
    for mode in ("strict", "fast"):
        st = D.new_stats()
        D.run("hybrid", planes[:9], planes[9:], D.Params(**PK), soa=True, strict=mode == "strict", out={},
              stats=st, n=CH)
        s = D.read_stats(st)
        acc[mode] += np.array([s[k] for k in names], np.int64)
        mins[mode] = min(mins[mode], s["min_distance"])
    del planes
    ref, counts, rc = oracle.hybrid(A, B, oracle.make_params(**PK), PK["epsilon"],
                                    threads=oracle.default_threads())
    acc["oracle"][:4] += np.asarray(counts[:4], np.int64)
    acc["oracle"][4] += int((ref["kind"] == 1).sum())
    mins["oracle"] = min(mins["oracle"], float(ref["distance"][ref["kind"] != 3].min()))
o = acc["oracle"].tolist()
for mode in ("strict", "fast"):
    g = acc[mode].tolist()
    print(f"cfg4 {N} pairs, {mode}: counters {dict(zip(names, g))}; oracle iterative/comparison/fallback/"
          f"degenerate/contacts {o}; equal {g[:5] == o}; min distance {mins[mode]!r} vs oracle "
          f"{mins['oracle']!r}", flush=True)
