"""Small launches of every batched kernel, for compute-sanitizer (memcheck /
racecheck / synccheck / initcheck): hybrid, comparison and iterative (fp64 and
fp32, fast and strict, SoA and AoS, with per-pair halos, an allow mask and
degenerate triangles so the fallback queues, the degenerate screen and the
partial final batches all run), the all-pairs particle blocks (with motions),
the multiscale frontier kernels, point-triangle and degenerate helpers, and
the host pipeline.

    compute-sanitizer --tool racecheck --kernel-name regex:tc:: python tools/sanitize_run.py
"""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import numpy as np
import torch
from paper_2105_12415_b200 import device as D, kernels as K, multiscale as MS, particles as PT, workloads as W

n = int(sys.argv[1]) if len(sys.argv) > 1 else 3000
A, B = W.random_pairs(n, seed=11, sep=(-0.1, 0.5))
rng = np.random.default_rng(1)
sel = rng.random(n) < 0.03
A[sel, 2] = A[sel, 0] + 0.5 * (A[sel, 1] - A[sel, 0])  # degenerate triangles on some fallbacks
eps = rng.uniform(1e-7, 1e-3, n)
allow = (rng.random(n) < 0.8).astype(np.uint8)
for dt in (torch.float64, torch.float32):
    for soa in (False, True):
        if soa:
            pl = torch.from_numpy(W.to_soa(A, B)).to("cuda", dt)
            ta, tb = pl[:9].contiguous(), pl[9:].contiguous()
        else:
            ta, tb = torch.from_numpy(A).to("cuda", dt), torch.from_numpy(B).to("cuda", dt)
        for strict in (False, True):
            st = D.new_stats()
            P = D.Params(n_iterative=16, epsilon=1e-6)
            D.run("hybrid", ta, tb, P, soa=soa, strict=strict, ids=True, stats=st,
                  eps=torch.from_numpy(eps).to("cuda", dt), allow=torch.from_numpy(allow).cuda())
            D.run("comparison", ta, tb, P, soa=soa, strict=strict, ids=True, stats=st)
            D.run("iterative", ta, tb, P, soa=soa, strict=strict, ids=True, stats=st)
            D.run("hybrid", ta, tb, P, soa=soa, strict=strict, out={}, stats=st)
    torch.cuda.synchronize()
# point-triangle / degenerate helpers
P3 = torch.from_numpy(rng.normal(size=(n, 3))).cuda()
T3 = torch.from_numpy(rng.normal(size=(n, 3, 3))).cuda()
D.closest_point_triangle(P3, T3)
D.degenerate_mask(T3, rel_tol=1e-6)
# particle blocks, with and without motions (small ragged meshes)
tm = torch.from_numpy(np.ascontiguousarray(np.stack([A[:80], B[:80], A[80:160]]))).cuda()
tb_ = torch.tensor([[0, 1], [1, 2], [2, 2]], dtype=torch.int32, device="cuda")
for strict in (False, True):
    st = D.new_stats()
    out = PT.blocks_hybrid(tm, tb_, D.Params(epsilon=5e-2), strict=strict, stats=st, max_contacts=80 * 80 * 3)
    mo = torch.tensor([[1.0, 0, 0, 0, 0, 0, 0], [0.9, 0.1, 0.3, 0.2, 0.1, 0, 0], [0.5, 0.5, 0.5, 0.5, 0, 0.1, 0]],
                      dtype=torch.float64)
    mo[:, :4] /= mo[:, :4].norm(dim=1, keepdim=True)
    PT.blocks_hybrid(tm, tb_, D.Params(epsilon=5e-2), motions=mo, mesh_tris=[80, 70, 60], strict=strict, stats=st,
                     max_contacts=80 * 80 * 3)
torch.cuda.synchronize()
# multiscale traversal on one of the reference's own scenes
g = np.load(ROOT / "tests" / "golden" / "ms_float64.npz")
sc = "s80_rest"
trees = [MS.FlatTreeArrays(g[f"{sc}_{s}_tris"].reshape(-1, 3, 3), g[f"{sc}_{s}_eps"], g[f"{sc}_{s}_child_off"],
                           g[f"{sc}_{s}_child_ids"], g[f"{sc}_{s}_height"], int(g[f"{sc}_{s}_n_nodes"]))
         for s in ("i", "j")]
forest = MS.build_forest(trees, dtype=np.float64)
for strict in (False, True):
    MS.multiscale_contacts(forest, [(0, 1)], K.KernelParams(), strict=strict)
# host pipeline (pageable arrays: staged)
K.set_rounding("fast")
try:
    K.hybrid_batch(A[:2000], B[:2000], K.KernelParams(), None, eps[:2000], allow_fallback=allow[:2000].astype(bool))
except K.DegenerateTriangle:
    pass  # the injected degenerate triangles reach the fallback: the reference raises too
torch.cuda.synchronize()
print("sanitize_run ok")
