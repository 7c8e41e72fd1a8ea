"""Whole-scene parity evidence for the particle-block kernel (GPU box, ~2 min):
BASELINE.json cfg2 (2,048 icosphere particles, 5,632 blocks, 576.7M triangle
pairs), strict hybrid fp64 at the bench's (16, 1e-6) and at a 5e-2 halo (with
contacts), against the C oracle over every pair (blocks materialised in
chunks): counters, contact lists and minimum distance.

    python tools/parity_cfg2.py > profiles/r01_parity_cfg2.txt
"""
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))
import numpy as np
import torch

import oracle
from paper_2105_12415_b200 import device as D, particles as PT

oracle.build()
meshes, blocks, gaps = PT.cfg2_scene()
T = meshes.shape[1]
nb = len(blocks)
for pk in (dict(n_iterative=16, epsilon=1e-6), dict(n_iterative=16, epsilon=5e-2)):
    t0 = time.time()
    st = D.new_stats()
    out = PT.blocks_hybrid(torch.from_numpy(meshes).cuda(), torch.from_numpy(blocks).cuda(), D.Params(**pk),
                           strict=True, stats=st, max_contacts=1 << 24)
    torch.cuda.synchronize()
    got = PT.sort_contacts(out)
    s = D.read_stats(st)
    p = oracle.make_params(**pk)
    tot = np.zeros(4, np.int64)
    mind = np.inf
    idx_ref, dist_ref = [], []
    chunk = 64
    for b0 in range(0, nb, chunk):
        which = list(range(b0, min(nb, b0 + chunk)))
        A, B = PT.block_pairs(meshes, blocks, which)
        ref, counts, rc = oracle.hybrid(A, B, p, p.epsilon, threads=oracle.default_threads())
        tot += np.asarray(counts[:4], np.int64)
        ok = ref["kind"] != 3
        mind = min(mind, float(ref["distance"][ok].min()))
        rows = np.nonzero(ref["kind"] == 1)[0]
        idx_ref.append(np.stack([b0 + rows // (T * T), (rows % (T * T)) // T, rows % T], 1))
        dist_ref.append(ref["distance"][rows])
    idx_ref = np.concatenate(idx_ref).astype(np.int32)
    dist_ref = np.concatenate(dist_ref)
    order = np.lexsort((idx_ref[:, 2], idx_ref[:, 1], idx_ref[:, 0]))
    idx_ref, dist_ref = idx_ref[order], dist_ref[order]
    same_contacts = got["n_contacts"] == len(idx_ref) and np.array_equal(got["idx"], idx_ref) \
        and np.array_equal(got["distance"], dist_ref)
    counters = [s["iterative"], s["comparison"], s["fallback"], s["degenerate"]]
    print(f"cfg2 strict {pk}: pairs {s['iterative']} ({nb} blocks x {T}x{T}); counters {counters} vs oracle "
          f"{tot.tolist()} equal {counters == tot.tolist()}; contacts {got['n_contacts']} vs {len(idx_ref)} "
          f"identical {same_contacts}; min distance {s['min_distance']!r} vs {mind!r} equal "
          f"{s['min_distance'] == mind}; {time.time() - t0:.0f} s", flush=True)
