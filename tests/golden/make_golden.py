"""Generate the golden fixtures from the reference implementation itself.

Runs in THIS container only (it imports the read-only reference from
/root/reference/pkg/src); the fixtures it writes are committed so that the
oracle and GPU parity tests never need the reference at run time.

    python tests/golden/make_golden.py            # writes tests/golden/*.npz

The reference's scalar type is fixed at import from TRICONTACT_REAL
(RK/geometry.py:23), so the float32 fixtures are produced by re-running this
script in a child interpreter with TRICONTACT_REAL=float32 on the float64
inputs cast to float32.

Besides the BatchResult columns, every comparison result carries ``ids``
re-derived from the reference's own private helpers
(closest_point_triangle_batch, _closest_segment_segment,
_segment_triangle_crossings): argmin feature row, the winning test's region
(point-triangle claim order) or segment branch code, the crossing pair
i0*6+i1, and flag bits.  The re-derived distance must be bit-identical to
comparison_batch's, which this script asserts.
"""

from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REPO = HERE.parent.parent
REF_SRC = Path("/root/reference/pkg/src")
sys.path.insert(0, str(REPO))
sys.path.insert(0, str(REF_SRC))

from paper_2105_12415_b200 import workloads  # noqa: E402

PARAM_SETS = {
    "def": dict(),                                   # reference defaults (4, 1e-2)
    "bl": dict(n_iterative=16, epsilon=1e-6),        # BASELINE.json config 0
}


def special_pairs():
    """Known-answer geometries of RT/test_kernels.py restated as inputs."""
    U = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0]], float)
    pairs = [
        (U, U),                                                   # identical
        (U, U + [0, 0, 1.0]),                                     # parallel offset 1
        (U, np.array([[2, 0, 0], [3, 0, 0], [2, 1, 0]], float)),  # vertex-vertex
        (U, np.array([[0.5, -0.5, 1.0], [0.5, 0.5, 1.0], [0.5, 0.0, 2.0]])),  # edge-edge
        (U, np.array([[0.2, 0.2, -0.5], [0.4, 0.2, 0.5], [0.3, 0.4, 0.5]])),  # intersecting
        (U, np.array([[0.1, 0.1, 0.0], [0.3, 0.1, 0.0], [0.1, 0.3, 0.0]])),   # coplanar overlap
        (U, U + [5.0, 0, 0]),                                     # coplanar far apart
        (U, U + [40.0, 0, 0.01]),                                 # crawling configuration
        (U, U + [0, 0, 0.005]),                                   # near contact
        (U, U + [0.3, 0.3, 0.0]),                                 # coplanar partial overlap
        (U, np.array([[0.25, 0.25, 0.0], [0.25, 0.25, 1.0], [0.5, 0.5, 1.0]])),  # touching vertex on face
        (U, np.array([[0.0, 0.0, 0.0], [-1.0, 0.0, 0.0], [0.0, -1.0, 0.0]])),    # shared vertex
    ]
    A = np.array([p[0] for p in pairs])
    B = np.array([p[1] for p in pairs])
    return A, B


def degenerate_cases(rng):
    """Triangles around the degenerate_mask threshold (RK/geometry.py:68-75)."""
    tris = [np.array([[0, 0, 0], [1, 0, 0], [2, 0, 0]], float),      # collinear
            np.zeros((3, 3)),                                         # point
            np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0]], float)]
    for h in (1e-3, 1e-5, 1e-6, 2e-6, 5e-7, 1e-7, 1e-9):
        tris.append(np.array([[0, 0, 0], [1, 0, 0], [0.5, h, 0]], float))
    T = np.concatenate([np.array(tris), rng.normal(size=(200, 3, 3))])
    # slivers of aspect 10^U(3, 7)
    v0 = rng.random((200, 3))
    d = rng.normal(size=(200, 3)); d /= np.linalg.norm(d, axis=1, keepdims=True)
    p = np.cross(d, rng.normal(size=(200, 3))); p /= np.linalg.norm(p, axis=1, keepdims=True)
    asp = 10.0 ** rng.uniform(3, 7, 200)
    S = np.stack([v0, v0 + d, v0 + 0.5 * d + p / asp[:, None]], axis=1)
    return np.concatenate([T, S])


# ---------------------------------------------------------------------------
# ids re-derived through the reference's own helpers
# ---------------------------------------------------------------------------

def _region_ids(p, tris):
    """Claim-order region (RK/kernels.py:193-218) of closest_point_triangle_batch."""
    import tricontact.kernels as K
    p = np.asarray(p, K.REAL)
    a, b, c = tris[:, 0], tris[:, 1], tris[:, 2]
    ab, ac = b - a, c - a
    ap, bp, cp = p - a, p - b, p - c
    dot = lambda x, y: np.einsum("ij,ij->i", x, y)
    d1, d2, d3, d4, d5, d6 = dot(ab, ap), dot(ac, ap), dot(ab, bp), dot(ac, bp), dot(ab, cp), dot(ac, cp)
    vc = d1 * d4 - d3 * d2
    vb = d5 * d2 - d1 * d6
    va = d3 * d6 - d5 * d4
    conds = [(d1 <= 0.0) & (d2 <= 0.0), (d3 >= 0.0) & (d4 <= d3), (vc <= 0.0) & (d1 >= 0.0) & (d3 <= 0.0),
             (d6 >= 0.0) & (d5 <= d6), (vb <= 0.0) & (d2 >= 0.0) & (d6 <= 0.0),
             (va <= 0.0) & (d4 - d3 >= 0.0) & (d5 - d6 >= 0.0)]
    region = np.full(p.shape[0], 6, np.uint8)
    for r in range(5, -1, -1):
        region[conds[r]] = r
    return region


def _segment_codes(p1, q1, p2, q2):
    import tricontact.kernels as K
    d1, d2, r = q1 - p1, q2 - p2, p1 - p2
    dot = lambda x, y: np.einsum("ij,ij->i", x, y)
    a, e, f, c, b = dot(d1, d1), dot(d2, d2), dot(d2, r), dot(d1, r), dot(d1, d2)
    s, _, _, _ = K._closest_segment_segment(p1, q1, p2, q2)
    denom = a * e - b * b
    s0 = np.where(denom > K._TINY, np.clip((b * f - c * e) / np.where(denom > K._TINY, denom, 1.0), 0.0, 1.0), 0.0)
    t = (b * s0 + f) / np.where(e > K._TINY, e, 1.0)
    return ((denom > K._TINY).astype(np.uint8) | ((t < 0.0).astype(np.uint8) << 1)
            | ((t > 1.0).astype(np.uint8) << 2))


def comparison_ids(A, B, res):
    """(n, 4) uint8 ids of comparison_batch results; asserts bitwise distance."""
    import tricontact.kernels as K
    n = A.shape[0]
    d2 = np.empty((15, n), K.REAL)
    code = np.empty((15, n), np.uint8)
    row = 0
    for src, dst in ((A, B), (B, A)):
        for k in range(3):
            closest, _ = K.closest_point_triangle_batch(src[:, k], dst)
            diff = src[:, k] - closest
            d2[row] = np.einsum("ij,ij->i", diff, diff)
            code[row] = _region_ids(src[:, k], dst)
            row += 1
    for ka in range(3):
        for kb in range(3):
            args = (A[:, K._EDGE_START[ka]], A[:, K._EDGE_END[ka]], B[:, K._EDGE_START[kb]], B[:, K._EDGE_END[kb]])
            _, _, c1, c2 = K._closest_segment_segment(*args)
            diff = c1 - c2
            d2[row] = np.einsum("ij,ij->i", diff, diff)
            code[row] = _segment_codes(*args)
            row += 1
    best = np.argmin(d2, axis=0)
    idx = np.arange(n)
    ok = np.zeros((6, n), bool)
    pts = np.zeros((6, n, 3), K.REAL)
    for k in range(3):
        ok[k], pts[k] = K._segment_triangle_crossings(A[:, K._EDGE_START[k]], A[:, K._EDGE_END[k]], B)
        ok[k + 3], pts[k + 3] = K._segment_triangle_crossings(B[:, K._EDGE_START[k]], B[:, K._EDGE_END[k]], A)
    inter = ok.any(axis=0)
    diff = pts[:, None] - pts[None, :]
    pd2 = np.where(ok[:, None] & ok[None, :], np.einsum("ijkl,ijkl->ijk", diff, diff), -1.0).reshape(36, n)
    pair = np.where(inter, np.argmax(pd2, axis=0), 255).astype(np.uint8)
    dist = np.where(inter, 0.0, np.sqrt(d2[best, idx])).astype(K.REAL)
    assert np.array_equal(dist, res.distance), "re-derived distance differs from comparison_batch"
    ids = np.stack([best.astype(np.uint8), code[best, idx], pair, (inter.astype(np.uint8) << 4)], axis=1)
    return ids


def _cols(res, prefix):
    return {f"{prefix}_{k}": getattr(res, k) for k in ("kind", "distance", "point_a", "point_b", "bary_a", "bary_b")}


def run_reference(inputs: dict) -> dict:
    """Run the reference on every case of ``inputs``; returns output arrays."""
    import tricontact.kernels as K
    from tricontact.geometry import degenerate_mask
    out = {}
    for case in ("cfg0", "cfg3", "special"):
        A = np.ascontiguousarray(inputs[f"{case}_A"], K.REAL)
        B = np.ascontiguousarray(inputs[f"{case}_B"], K.REAL)
        for pname, pkw in PARAM_SETS.items():
            p = K.KernelParams(**pkw)
            eps = np.full(A.shape[0], p.epsilon, K.REAL)
            cm = K.comparison_batch(A, B, eps)
            out.update(_cols(cm, f"{case}_{pname}_comparison"))
            out[f"{case}_{pname}_comparison_ids"] = comparison_ids(A, B, cm)
            it = K.iterative_batch(A, B, p, eps)
            out.update(_cols(it, f"{case}_{pname}_iterative"))
            counters = K.KernelCounters()
            try:
                hy = K.hybrid_batch(A, B, p, counters, eps)
                out.update(_cols(hy, f"{case}_{pname}_hybrid"))
                out[f"{case}_{pname}_hybrid_counters"] = np.array(
                    [counters.iterative_invocations, counters.comparison_invocations, counters.fallback_invocations])
            except K.DegenerateTriangle:
                out[f"{case}_{pname}_hybrid_raised"] = np.array(1)
    # per-pair eps and allow_fallback mask, as multiscale_contacts passes them (RK/stepping.py:338-339)
    A = np.ascontiguousarray(inputs["cfg0_A"][:1024], K.REAL)
    B = np.ascontiguousarray(inputs["cfg0_B"][:1024], K.REAL)
    p = K.KernelParams()
    eps = np.asarray(inputs["mask_eps"], K.REAL)
    allow = np.asarray(inputs["mask_allow"], bool)
    counters = K.KernelCounters()
    hy = K.hybrid_batch(A, B, p, counters, eps, allow_fallback=allow)
    out.update(_cols(hy, "masked_hybrid"))
    out["masked_hybrid_counters"] = np.array(
        [counters.iterative_invocations, counters.comparison_invocations, counters.fallback_invocations])
    # point-triangle and degenerate helpers
    P = np.asarray(inputs["cpt_P"], K.REAL)
    T = np.asarray(inputs["cpt_T"], K.REAL)
    cl, ba = K.closest_point_triangle_batch(P, T)
    out["cpt_closest"], out["cpt_bary"], out["cpt_region"] = cl, ba, _region_ids(P, T)
    out["degenerate_mask"] = degenerate_mask(np.asarray(inputs["degenerate_T"], K.REAL))
    return out


def make_inputs() -> dict:
    A0, B0 = workloads.random_pairs(**{k: workloads.CFG0[k] for k in ("n", "seed", "sep")})
    A3, B3 = workloads.adversarial_pairs(256)
    As, Bs = special_pairs()
    rng = np.random.default_rng(20260810)
    return {
        "cfg0_A": A0, "cfg0_B": B0,
        "cfg3_A": A3, "cfg3_B": B3,
        "special_A": As, "special_B": Bs,
        "mask_eps": rng.uniform(1e-3, 5e-2, 1024),
        "mask_allow": rng.random(1024) < 0.5,
        "cpt_P": rng.normal(size=(2000, 3)),
        "cpt_T": rng.normal(size=(2000, 3, 3)),
        "degenerate_T": degenerate_cases(rng),
    }


def main():
    if len(sys.argv) > 1 and sys.argv[1] == "--worker":
        # child interpreter: TRICONTACT_REAL is already set in the environment
        src, dst = sys.argv[2], sys.argv[3]
        inputs = dict(np.load(src))
        np.savez_compressed(dst, **run_reference(inputs))
        return
    inputs = make_inputs()
    np.savez_compressed(HERE / "inputs.npz", **inputs)
    for real in ("float64", "float32"):
        env = dict(os.environ, TRICONTACT_REAL=real, PYTHONPATH=f"{REF_SRC}:{REPO}")
        dst = HERE / f"ref_{real}.npz"
        subprocess.run([sys.executable, __file__, "--worker", str(HERE / "inputs.npz"), str(dst)],
                       env=env, check=True)
        print("wrote", dst, dst.stat().st_size, "bytes")


if __name__ == "__main__":
    main()
