"""Tolerance comparison of the fast (FMA-contracted) kernels against the oracle.

North-star tolerance: |x - x_ref| <= tau * max(|x_ref|, L) with
tau = 1e-9 (fp64) / 1e-4 (fp32) and L the pair's longest edge; discrete
outputs (kind, fallback path, feature id) must match except at ties.
"""

from __future__ import annotations

import numpy as np

TAU = {np.dtype(np.float64): 1e-9, np.dtype(np.float32): 1e-4}


def longest_edge(A, B):
    def sq(T):
        e = np.roll(T, -1, axis=1) - T
        return (e * e).sum(axis=2).max(axis=1)
    return np.sqrt(np.maximum(sq(A.astype(np.float64)), sq(B.astype(np.float64))))


def rel_err(x, ref, L):
    x = np.asarray(x, np.float64)
    ref = np.asarray(ref, np.float64)
    if x.ndim == 1:
        return np.abs(x - ref) / np.maximum(np.abs(ref), L)
    return (np.abs(x - ref).max(axis=1)) / np.maximum(np.abs(ref).max(axis=1), L)


def compare_fast(O, variant, A, B, pkw, got, dtype, max_tie_frac=None):
    """Compare one fast-mode result dict against the oracle; returns a report."""
    dtype = np.dtype(dtype)
    tau = TAU[dtype]
    p = O.make_params(**pkw)
    eps = np.full(len(A), p.epsilon, dtype)
    if variant == "comparison":
        ref = O.comparison(A, B, eps, dtype)
    elif variant == "iterative":
        ref = O.iterative(A, B, p, eps, dtype)
    else:
        ref, _, _ = O.hybrid(A, B, p, eps, dtype=dtype)
    L = longest_edge(A, B)
    path_ref = ref["ids"][:, 3] & 4
    path_got = got["ids"][:, 3] & 4 if "ids" in got else path_ref
    same = (ref["kind"] == got["kind"]) & (path_ref == path_got)
    if variant == "comparison":
        same &= ref["ids"][:, 0] == got["ids"][:, 0] if "ids" in got else True
    d_err = rel_err(got["distance"], ref["distance"], L)
    p_err = np.maximum(rel_err(got["point_a"], ref["point_a"], L), rel_err(got["point_b"], ref["point_b"], L))
    mism = int((~same).sum())
    if max_tie_frac is None:
        max_tie_frac = 1e-3 if dtype == np.float64 else 2e-2
    rep = {
        "variant": variant, "n": len(A), "discrete_mismatches": mism,
        "distance_max_rel": float(d_err[same].max()) if same.any() else 0.0,
        "point_max_rel": float(p_err[same].max()) if same.any() else 0.0,
        "point_over_tol": int((p_err[same] > tau).sum()),
    }
    rep["ok"] = (rep["distance_max_rel"] <= tau and mism <= max_tie_frac * len(A)
                 and rep["point_over_tol"] <= max_tie_frac * len(A))
    return rep
