"""ctypes front end of the CPU oracle (oracle/libtc_oracle.so).

TEST INFRASTRUCTURE ONLY: tests/, ``__graft_entry__.smoke()`` and bench.py's
``cpu_baseline`` / ``--impl reference`` legs are the only callers.  The
product path (paper_2105_12415_b200) never imports this module.

Every function restates the reference function of the same name in
/root/reference/pkg/src/tricontact/kernels.py (RK):
  comparison   -> RK/kernels.py:301 comparison_batch
  iterative    -> RK/kernels.py:447 iterative_batch
  hybrid       -> RK/kernels.py:568 hybrid_batch (degenerate pairs -> kind 3)
  closest_point_triangle -> RK/kernels.py:157
  degenerate   -> RK/geometry.py:68 degenerate_mask
Outputs are dicts of numpy columns named like BatchResult (RK/kernels.py:96)
plus ``ids`` (n, 4) uint8 (layout in oracle/README.md).
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
_LIB_PATH = _HERE / "libtc_oracle.so"
_lib = None


class OracleParams(ctypes.Structure):
    _fields_ = [
        ("epsilon", ctypes.c_double),
        ("c_factor", ctypes.c_double),
        ("alpha_iterative", ctypes.c_double),
        ("alpha_regulariser", ctypes.c_double),
        ("move_factor", ctypes.c_double),
        ("start_coord", ctypes.c_double),
        ("n_iterative", ctypes.c_int32),
        ("flags", ctypes.c_int32),
    ]


def build(force: bool = False) -> Path:
    """Compile the oracle with its Makefile (gcc, -ffp-contract=off)."""
    if force or not _LIB_PATH.exists() or not (_HERE / "libtc_oracle_fma.so").exists() or _LIB_PATH.stat().st_mtime < max(
            p.stat().st_mtime for p in _HERE.glob("tc_oracle*")):
        subprocess.run(["make", "-s", "-C", str(_HERE)], check=True)
    return _LIB_PATH


def fma_variant():
    """A second copy of this module bound to libtc_oracle_fma.so (FMA-contracted
    build of the same restatement; CPU stand-in for the GPU fast build)."""
    import importlib.util
    spec = importlib.util.spec_from_file_location("oracle_fma", __file__)
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    mod._LIB_PATH = _HERE / "libtc_oracle_fma.so"
    if not mod._LIB_PATH.exists():
        build(force=True)
    return mod


def lib():
    global _lib
    if _lib is None:
        if not _LIB_PATH.exists():
            build()
        _lib = ctypes.CDLL(str(_LIB_PATH))
        p = ctypes.c_void_p
        i64 = ctypes.c_int64
        i32 = ctypes.c_int
        for sfx in ("f64", "f32"):
            getattr(_lib, f"tco_comparison_{sfx}").argtypes = [p, p, i64, p] + [p] * 7 + [i32]
            getattr(_lib, f"tco_iterative_{sfx}").argtypes = [p, p, i64, p, p] + [p] * 7 + [i32]
            getattr(_lib, f"tco_hybrid_{sfx}").argtypes = [p, p, i64, p, p, p] + [p] * 8 + [i32]
            getattr(_lib, f"tco_closest_point_triangle_{sfx}").argtypes = [p, p, i64, p, p, i32]
            getattr(_lib, f"tco_degenerate_{sfx}").argtypes = [p, i64, ctypes.c_double, p, i32]
            getattr(_lib, f"tco_margins_{sfx}").argtypes = [p, p, i64, p, p, p, i32]
            getattr(_lib, f"tco_apply_motion_{sfx}").argtypes = [p, i64, p, p, p]
            for name in ("comparison", "iterative", "hybrid", "closest_point_triangle", "degenerate", "margins",
                         "apply_motion"):
                getattr(_lib, f"tco_{name}_{sfx}").restype = ctypes.c_int
    return _lib


def default_threads() -> int:
    return len(os.sched_getaffinity(0))


def _sfx(dtype) -> str:
    dtype = np.dtype(dtype)
    if dtype == np.float64:
        return "f64"
    if dtype == np.float32:
        return "f32"
    raise TypeError(f"unsupported dtype {dtype}")


def _tris(x, dtype):
    a = np.ascontiguousarray(x, dtype=dtype)
    if a.ndim == 2:
        a = a[None]
    if a.ndim != 3 or a.shape[1:] != (3, 3):
        raise ValueError(f"expected triangles of shape (n, 3, 3), got {a.shape}")
    return a


def _eps(eps, n, dtype):
    e = np.asarray(eps, dtype=dtype)
    if e.ndim == 0:
        e = np.full(n, e, dtype=dtype)
    if e.shape != (n,):
        raise ValueError("eps must be scalar or shape (n,)")
    return np.ascontiguousarray(e)


def _ptr(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _outputs(n, dtype):
    return {
        "distance": np.empty(n, dtype),
        "point_a": np.empty((n, 3), dtype),
        "point_b": np.empty((n, 3), dtype),
        "bary_a": np.empty((n, 2), dtype),
        "bary_b": np.empty((n, 2), dtype),
        "kind": np.empty(n, np.int8),
        "ids": np.empty((n, 4), np.uint8),
    }


def make_params(epsilon=1e-2, n_iterative=4, c_factor=1.0, alpha_iterative=10.0,
                alpha_regulariser=1e-4, move_factor=0.25, start_coord=1.0 / 3.0):
    return OracleParams(epsilon, c_factor, alpha_iterative, alpha_regulariser,
                        move_factor, start_coord, n_iterative, 0)


def _out_ptrs(o):
    return [_ptr(o[k]) for k in ("distance", "point_a", "point_b", "bary_a", "bary_b", "kind", "ids")]


def comparison(A, B, eps, dtype=np.float64, threads=1):
    A = _tris(A, dtype); B = _tris(B, dtype)
    n = A.shape[0]
    e = _eps(eps, n, dtype)
    o = _outputs(n, dtype)
    rc = getattr(lib(), f"tco_comparison_{_sfx(dtype)}")(_ptr(A), _ptr(B), n, _ptr(e), *_out_ptrs(o), threads)
    assert rc == 0
    return o


def iterative(A, B, params, eps, dtype=np.float64, threads=1):
    A = _tris(A, dtype); B = _tris(B, dtype)
    n = A.shape[0]
    e = _eps(eps, n, dtype)
    o = _outputs(n, dtype)
    rc = getattr(lib(), f"tco_iterative_{_sfx(dtype)}")(_ptr(A), _ptr(B), n, _ptr(e), ctypes.byref(params),
                                                       *_out_ptrs(o), threads)
    assert rc == 0
    return o


def hybrid(A, B, params, eps, allow_fallback=None, dtype=np.float64, threads=1):
    """Returns (columns, counts[iterative, comparison, fallback, degenerate], rc)."""
    A = _tris(A, dtype); B = _tris(B, dtype)
    n = A.shape[0]
    e = _eps(eps, n, dtype)
    allow = None
    if allow_fallback is not None:
        allow = np.ascontiguousarray(np.broadcast_to(np.asarray(allow_fallback, bool), (n,)), dtype=np.uint8)
    o = _outputs(n, dtype)
    counts = np.zeros(4, np.int64)
    rc = getattr(lib(), f"tco_hybrid_{_sfx(dtype)}")(_ptr(A), _ptr(B), n, _ptr(e), _ptr(allow), ctypes.byref(params),
                                                    *_out_ptrs(o), _ptr(counts), threads)
    return o, counts, rc


def closest_point_triangle(P, T, dtype=np.float64, threads=1):
    P = np.ascontiguousarray(P, dtype=dtype).reshape(-1, 3)
    T = _tris(T, dtype)
    n = T.shape[0]
    c = np.empty((n, 3), dtype)
    b = np.empty((n, 2), dtype)
    rc = getattr(lib(), f"tco_closest_point_triangle_{_sfx(dtype)}")(_ptr(P), _ptr(T), n, _ptr(c), _ptr(b), threads)
    assert rc == 0
    return c, b


def degenerate(T, dtype=np.float64, threads=1, rel_tol=1e-12):
    T = _tris(T, dtype)
    m = np.empty(T.shape[0], np.uint8)
    rc = getattr(lib(), f"tco_degenerate_{_sfx(dtype)}")(_ptr(T), T.shape[0], float(rel_tol), _ptr(m), threads)
    assert rc == 0
    return m.astype(bool)


def apply_motion(points, quat, t, dtype=np.float64):
    """RK/geometry.py:173-176 RigidMotion.apply_points (see tc_oracle_impl.h)."""
    P = np.ascontiguousarray(points, dtype=dtype).reshape(-1, 3)
    out = np.empty_like(P)
    q = np.ascontiguousarray(quat, np.float64).reshape(4)
    tt = np.ascontiguousarray(t, dtype).reshape(3)
    rc = getattr(lib(), f"tco_apply_motion_{_sfx(dtype)}")(_ptr(P), P.shape[0], _ptr(q), _ptr(tt), _ptr(out))
    assert rc == 0
    return out.reshape(np.shape(points))


def margins(A, B, params, eps, dtype=np.float64, threads=1):
    """(n, 10) float64 decision margins (layout in tc_oracle_impl.h, tco_margins_*)."""
    A = _tris(A, dtype); B = _tris(B, dtype)
    n = A.shape[0]
    e = _eps(eps, n, dtype)
    m = np.empty((n, 10), np.float64)
    rc = getattr(lib(), f"tco_margins_{_sfx(dtype)}")(_ptr(A), _ptr(B), n, _ptr(e), ctypes.byref(params), _ptr(m),
                                                     threads)
    assert rc == 0
    return m
