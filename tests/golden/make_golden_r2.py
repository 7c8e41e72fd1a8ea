"""Round-2 golden fixtures, produced by the reference implementation itself.

Runs in THIS container only: it imports the read-only reference package and
its own test helpers from /root/reference/pkg (src and tests); the fixtures
it writes are committed, so no test needs the reference at run time.

    python tests/golden/make_golden_r2.py     # writes tests/golden/r2_float{64,32}.npz

Contents
* ``crit1_*`` -- acceptance criterion 1 (RT/test_acceptance.py:69-87): the
  10,000 scene-drawn pairs of ``scene_drawn_pairs(20260801, 10000)``, the
  reference's ``comparison_batch`` and ``hybrid_batch`` results at the default
  KernelParams (with the comparison ids re-derived like make_golden.py) and the
  independent sampling oracle's distance and bound
  (RT/oracles.py:78-131 ``sampling_distance_batch``).  float64 only, like the
  criterion.
* ``grad_*`` -- acceptance criterion 2's points (RT/test_acceptance.py:90-118,
  seed 20260802): the reference's ``gradient_of_J`` and ``functional_value``
  at 400 (A, B, x) points.  float64 only.
* ``degtol_*`` -- ``geometry.degenerate_mask(T, rel_tol)`` (RK/geometry.py:68-75)
  on the round-1 degenerate inputs at several rel_tol, float64 and float32.
"""

from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REPO = HERE.parent.parent
REF = Path("/root/reference/pkg")
REL_TOLS = (0.0, 1e-15, 1e-9, 1e-6, 1e-3)


def worker(dst: str) -> None:
    sys.path[:0] = [str(REF / "src"), str(REF / "tests"), str(HERE)]
    import tricontact.kernels as K
    from tricontact.geometry import degenerate_mask
    out = {}
    inputs = dict(np.load(HERE / "inputs.npz"))
    T = np.asarray(inputs["degenerate_T"], K.REAL)
    for i, tol in enumerate(REL_TOLS):
        out[f"degtol_{i}"] = degenerate_mask(T, rel_tol=tol)
    out["degtol_rel_tols"] = np.array(REL_TOLS)
    if K.REAL == np.float64:
        from make_golden import comparison_ids
        from oracles import sampling_distance_batch
        from test_acceptance import scene_drawn_pairs
        # criterion 1
        p = K.KernelParams()
        A, B = scene_drawn_pairs(20260801, 10000)
        A = np.ascontiguousarray(A)
        B = np.ascontiguousarray(B)
        eps = np.full(len(A), p.epsilon)
        exact = K.comparison_batch(A, B, eps)
        hybrid = K.hybrid_batch(A, B, p, None, eps)
        oracle_d, bound = sampling_distance_batch(A, B)
        out["crit1_A"], out["crit1_B"] = A, B
        for name, res in (("comparison", exact), ("hybrid", hybrid)):
            for col in ("kind", "distance", "point_a", "point_b", "bary_a", "bary_b"):
                out[f"crit1_{name}_{col}"] = getattr(res, col)
        out["crit1_comparison_ids"] = comparison_ids(A, B, exact)
        out["crit1_oracle_distance"], out["crit1_oracle_bound"] = oracle_d, bound
        band = np.abs(exact.distance - 2.0 * p.epsilon) <= p.c_factor * p.epsilon
        assert int(((hybrid.kind != exact.kind) & ~band).sum()) == 0
        # criterion 2's points
        rng = np.random.default_rng(20260802)
        pts, grads, vals = [], [], []
        while len(pts) < 400:
            a = rng.normal(size=(3, 3))
            b = rng.normal(size=(3, 3)) + rng.normal(scale=1.0, size=3)
            x = rng.uniform(-0.4, 1.4, size=4)
            pts.append(np.concatenate([a.ravel(), b.ravel(), x]))
            grads.append(K.gradient_of_J(a, b, *x, p))
            vals.append(K.functional_value(a, b, *x, p))
        out["grad_points"] = np.array(pts)
        out["grad_gradient"] = np.array(grads)
        out["grad_value"] = np.array(vals)
    np.savez_compressed(dst, **out)


def main():
    if len(sys.argv) > 2 and sys.argv[1] == "--worker":
        worker(sys.argv[2])
        return
    for real in ("float64", "float32"):
        env = dict(os.environ, TRICONTACT_REAL=real, PYTHONPATH=f"{REF / 'src'}:{REPO}")
        dst = HERE / f"r2_{real}.npz"
        subprocess.run([sys.executable, __file__, "--worker", str(dst)], env=env, check=True)
        print("wrote", dst, dst.stat().st_size, "bytes")


if __name__ == "__main__":
    main()
