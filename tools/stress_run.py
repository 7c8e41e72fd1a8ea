"""Queue / batch stress of the batched kernels (tests/test_gpu_stress.py runs
it with the TC_DEBUG library, TC_LIB_PATH=.../libtricontact_b200_debug.so):
every kernel at several CTA caps (1, 2, 7, 37, the occupancy maximum), so the
fallback queues see every fill pattern; a device trap (queue overflow,
out-of-range index, leftover entry) fails the launch and this script.
Results must be identical across caps (strict and fast) and, in strict mode,
bit-identical to the oracle.  Prints 'stress ok'."""
import ctypes
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path[:0] = [str(ROOT), str(ROOT / "oracle")]
import numpy as np
import torch
import oracle
from paper_2105_12415_b200 import _abi, device as D, particles as PT, workloads as W

lib = _abi.load()
print("library", lib._name, flush=True)
CAPS = (1, 2, 7, 37, 0)


def cols(out):
    return {k: v.cpu().numpy() for k, v in out.items()}


def same(a, b, what):
    for k in a:
        assert np.array_equal(a[k], b[k]), (what, k)


for dt, real in ((np.float64, torch.float64), (np.float32, torch.float32)):
    for n in (1, 127, 129, 4097, 3 * 4096 + 5):
        A, B = W.random_pairs(n, seed=n, sep=(-0.1, 0.5))
        rng = np.random.default_rng(n)
        sel = rng.random(n) < 0.05
        A[sel, 2] = A[sel, 0] + 0.25 * (A[sel, 1] - A[sel, 0])
        A, B = A.astype(dt), B.astype(dt)
        eps = rng.uniform(1e-7, 1e-3, n).astype(dt)
        allow = (rng.random(n) < 0.8).astype(np.uint8)
        ta, tb = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
        te, tl = torch.from_numpy(eps).cuda(), torch.from_numpy(allow).cuda()
        P = D.Params(n_iterative=16, epsilon=1e-6)
        for strict in (True, False):
            for variant in ("hybrid", "comparison", "iterative"):
                ref = None
                for cap in CAPS:
                    lib.tc_debug_set_max_ctas(cap)
                    st = D.new_stats()
                    kw = dict(eps=te, allow=tl) if variant == "hybrid" else dict(eps=te)
                    out = cols(D.run(variant, ta, tb, P, strict=strict, ids=True, stats=st, **kw))
                    torch.cuda.synchronize()
                    out["stats"] = np.array(list(D.read_stats(st).values()))
                    if ref is None:
                        ref = out
                    else:
                        same(ref, out, (variant, n, strict, cap))
                if strict and variant == "hybrid":
                    o, counts, rc = oracle.hybrid(A, B, oracle.make_params(n_iterative=16, epsilon=1e-6), eps,
                                                  allow_fallback=allow, dtype=dt)
                    for k in ("kind", "distance", "point_a", "point_b", "bary_a", "bary_b", "ids"):
                        assert np.array_equal(ref[k], o[k]), ("oracle", n, k)
lib.tc_debug_set_max_ctas(0)
# particle blocks: ragged meshes, self blocks, at several caps
rng = np.random.default_rng(5)
M = rng.random((3, 90, 3, 3))
tm = torch.from_numpy(M).cuda()
blocks = torch.tensor([[0, 1], [1, 1], [2, 0], [2, 2]], dtype=torch.int32, device="cuda")
for strict in (True, False):
    ref = None
    for cap in CAPS:
        lib.tc_debug_set_max_ctas(cap)
        st = D.new_stats()
        out = PT.sort_contacts(PT.blocks_hybrid(tm, blocks, D.Params(epsilon=5e-2), mesh_tris=[90, 80, 70],
                                                strict=strict, stats=st, max_contacts=4 * 90 * 90))
        res = (out["idx"], out["point_a"], np.array(list(D.read_stats(st).values())))
        if ref is None:
            ref = res
        else:
            for a, b in zip(ref, res):
                assert np.array_equal(a, b), ("blocks", strict, cap)
lib.tc_debug_set_max_ctas(0)
torch.cuda.synchronize()
print("stress ok", flush=True)
