"""Drop-in replacement of the reference module ``tricontact.kernels``.

Same names, signatures, keyword defaults, result types and errors as
/root/reference/pkg/src/tricontact/kernels.py (RK), with every batch
computed by the sm_100a kernels of libtricontact_b200.so through its C ABI
(host entry points: the library pipelines H2D copy, kernel and D2H copy).
There is no CPU path: without the library or a CUDA device these functions
raise.

Rounding: by default the kernels run in TC_STRICT mode, which reproduces
the reference's IEEE operation order and is bit-identical to it (the
drop-in promise).  ``set_rounding("fast")`` (or TRICONTACT_B200_ROUNDING=fast)
selects the FMA-contracted throughput build, equal within the north-star
tolerance instead of bitwise.

To serve this module as ``tricontact.kernels`` for the reference's callers
(contact.py, stepping.py bind ``hybrid_batch`` by name at import), install
it in ``sys.modules`` before they import -- see INTEGRATION.md.
"""

from __future__ import annotations

import ctypes
import os
import weakref
from dataclasses import dataclass
from enum import IntEnum

import numpy as np

from . import _abi

# RK/geometry.py:23 -- scalar type fixed at import from the environment
REAL = np.float32 if os.environ.get("TRICONTACT_REAL") == "float32" else np.float64
_TINY = 1e-30

_ROUNDING = os.environ.get("TRICONTACT_B200_ROUNDING", "strict")


def set_rounding(mode: str) -> None:
    """'strict' (bit-identical to the reference) or 'fast' (FMA-contracted)."""
    global _ROUNDING
    if mode not in ("strict", "fast"):
        raise ValueError("rounding mode must be 'strict' or 'fast'")
    _ROUNDING = mode


def rounding() -> str:
    return _ROUNDING


def _flags() -> int:
    return _abi.TC_STRICT if _ROUNDING == "strict" else 0


class DegenerateTriangle(ValueError):
    """Raised when the comparison kernel receives a near-zero-area triangle."""


class Kind(IntEnum):
    NO_CONTACT = 0
    CONTACT = 1
    NOT_TERMINATED = 2


@dataclass
class KernelParams:
    """Tunables of the iterative/hybrid kernels (RK/kernels.py:42-72)."""

    epsilon: float = 1e-2
    n_iterative: int = 4
    c_factor: float = 1.0
    alpha_iterative: float = 10.0
    alpha_regulariser: float = 1e-4
    move_factor: float = 0.25
    start_coord: float = 1.0 / 3.0

    def __post_init__(self):
        if self.epsilon <= 0.0:
            raise ValueError("epsilon must be positive")
        if self.n_iterative < 1:
            raise ValueError("n_iterative must be at least 1")
        if self.c_factor <= 0.0:
            raise ValueError("c_factor must be positive")
        if self.alpha_iterative <= 0.0 or self.alpha_regulariser <= 0.0:
            raise ValueError("penalty weights must be positive")


@dataclass
class KernelCounters:
    """Monotone tallies of kernel work within a run (RK/kernels.py:75-93)."""

    iterative_invocations: int = 0
    comparison_invocations: int = 0
    fallback_invocations: int = 0

    def merge(self, other: "KernelCounters") -> None:
        self.iterative_invocations += other.iterative_invocations
        self.comparison_invocations += other.comparison_invocations
        self.fallback_invocations += other.fallback_invocations

    def as_dict(self) -> dict:
        return {
            "iterative_invocations": self.iterative_invocations,
            "comparison_invocations": self.comparison_invocations,
            "fallback_invocations": self.fallback_invocations,
        }


@dataclass
class BatchResult:
    """Column-wise kernel results (RK/kernels.py:96-117)."""

    kind: np.ndarray
    distance: np.ndarray
    point_a: np.ndarray
    point_b: np.ndarray
    bary_a: np.ndarray
    bary_b: np.ndarray

    def __len__(self) -> int:
        return self.kind.shape[0]

    def splice(self, mask: np.ndarray, other: "BatchResult") -> None:
        self.kind[mask] = other.kind
        self.distance[mask] = other.distance
        self.point_a[mask] = other.point_a
        self.point_b[mask] = other.point_b
        self.bary_a[mask] = other.bary_a
        self.bary_b[mask] = other.bary_b


@dataclass
class DistanceResult:
    """Scalar result for one pair (RK/kernels.py:120-129)."""

    kind: Kind
    distance: float
    point_a: np.ndarray
    point_b: np.ndarray
    bary_a: tuple[float, float]
    bary_b: tuple[float, float]


def _scalar(res: BatchResult, i: int = 0) -> DistanceResult:
    return DistanceResult(
        kind=Kind(int(res.kind[i])),
        distance=float(res.distance[i]),
        point_a=res.point_a[i].copy(),
        point_b=res.point_b[i].copy(),
        bary_a=(float(res.bary_a[i, 0]), float(res.bary_a[i, 1])),
        bary_b=(float(res.bary_b[i, 0]), float(res.bary_b[i, 1])),
    )


def as_triangles(obj) -> np.ndarray:
    """RK/geometry.py:35-42: coerce to (n, 3, 3) REAL."""
    arr = np.asarray(obj, dtype=REAL)
    if arr.ndim == 2:
        arr = arr[None]
    if arr.ndim != 3 or arr.shape[1:] != (3, 3):
        raise ValueError(f"expected triangles of shape (n, 3, 3), got {arr.shape}")
    return arr


def _as_eps(eps, n: int) -> np.ndarray:
    """RK/kernels.py:143-149."""
    eps = np.asarray(eps, dtype=REAL)
    if eps.ndim == 0:
        eps = np.full(n, float(eps), dtype=REAL)
    if eps.shape != (n,):
        raise ValueError("eps must be scalar or shape (n,)")
    return eps


def _ptr(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _sfx(dtype) -> str:
    return "f32" if np.dtype(dtype) == np.float32 else "f64"


_PINNED_MIN = 1 << 16  # pairs; smaller results are plain numpy arrays


def _result(n: int) -> BatchResult:
    """Result columns for n pairs.  Large results live in one pinned host
    block of the library (tc_host_alloc), which the DMA engines write directly
    (no staging copy); the block returns to the library's cache when the last
    column view is garbage-collected.  They are ordinary writeable numpy
    arrays for the caller."""
    cols = (("distance", (n,), REAL), ("point_a", (n, 3), REAL), ("point_b", (n, 3), REAL),
            ("bary_a", (n, 2), REAL), ("bary_b", (n, 2), REAL), ("kind", (n,), np.int8))
    if n >= _PINNED_MIN:
        offs, total = [], 0
        for _, shape, dt in cols:
            offs.append(total)
            total += (int(np.prod(shape)) * np.dtype(dt).itemsize + 255) & ~255
        lib = _abi.load()
        ptr = lib.tc_host_alloc(total)
        if ptr:
            buf = (ctypes.c_char * total).from_address(ptr)
            fin = weakref.finalize(buf, lib.tc_host_free, ptr)
            fin.atexit = False  # the process is ending: the OS reclaims the block
            raw = np.frombuffer(buf, np.uint8)
            arrs = {name: raw[o:o + int(np.prod(shape)) * np.dtype(dt).itemsize].view(dt).reshape(shape)
                    for (name, shape, dt), o in zip(cols, offs)}
            return BatchResult(**arrs)
    return BatchResult(**{name: np.empty(shape, dt) for name, shape, dt in cols})


def _run(variant: str, A, B, eps, params, allow=None):
    """One host-buffer C-ABI call; returns (BatchResult, TcStats, rc).

    ``eps`` is the reference's per-pair halo array, or a positive scalar,
    which travels as ``tc_params.epsilon`` instead of an (n,) array (the
    kernels read ``eps == NULL`` as "every pair uses params.epsilon", rounded
    to REAL exactly like ``np.asarray(eps, REAL)``).  ``allow``: an (n,) mask,
    already broadcast by the caller.  Pageable numpy buffers are staged through
    the library's pinned buffers (tc_run_host_*, include/tricontact_b200.h).
    """
    lib = _abi.load()
    A = np.ascontiguousarray(A, dtype=REAL)
    B = np.ascontiguousarray(B, dtype=REAL)
    n = A.shape[0]
    if B.shape[0] != n:
        raise ValueError("tri_a and tri_b must have the same length")
    res = _result(n)
    stats = _abi.TcStats(0, 0, 0, 0, 0, 0, float("inf"))
    if n == 0:
        return res, stats, _abi.TC_OK
    p = _abi.params_struct(params if params is not None else KernelParams(), _flags())
    eps_arr = None
    if np.ndim(eps) == 0 and float(eps) > 0.0:
        p.epsilon = float(eps)
    else:
        eps_arr = np.ascontiguousarray(np.broadcast_to(np.asarray(eps, dtype=REAL), (n,)))
    if allow is not None:
        allow = np.ascontiguousarray(allow, dtype=np.uint8)
        if allow.shape != (n,):
            raise ValueError("allow_fallback mask must have shape (n,)")
    fn = getattr(lib, f"tc_run_host_{_sfx(REAL)}")
    rc = fn(_abi.VARIANTS[variant], _ptr(A), _ptr(B), n, _ptr(eps_arr), _ptr(allow), ctypes.byref(p),
            _ptr(res.distance), _ptr(res.point_a), _ptr(res.point_b), _ptr(res.bary_a), _ptr(res.bary_b),
            _ptr(res.kind), None, ctypes.byref(stats))
    if rc not in (_abi.TC_OK, _abi.TC_EDEGENERATE):
        _abi.check(rc, f"tc_run_host ({variant})")
    return res, stats, rc


def _halo(eps, n: int):
    """RK/kernels.py:143-149 _as_eps, keeping a scalar halo scalar (same
    validation and rounding; the kernels broadcast it)."""
    e = np.asarray(eps, dtype=REAL)
    if e.ndim == 0:
        return e
    if e.shape != (n,):
        raise ValueError("eps must be scalar or shape (n,)")
    return e


# ---------------------------------------------------------------------------
# Batch API
# ---------------------------------------------------------------------------


def closest_point_triangle_batch(points: np.ndarray, tris: np.ndarray):
    """RK/kernels.py:157-221: ``(closest (n, 3), bary (n, 2))``."""
    p = np.ascontiguousarray(np.asarray(points, dtype=REAL).reshape(-1, 3))
    t = np.ascontiguousarray(as_triangles(tris))
    n = t.shape[0]
    if p.shape[0] != n:
        raise ValueError("points and triangles must have the same length")
    closest = np.empty((n, 3), REAL)
    bary = np.empty((n, 2), REAL)
    if n:
        lib = _abi.load()
        rc = getattr(lib, f"tc_closest_point_triangle_host_{_sfx(REAL)}")(_ptr(p), _ptr(t), n, _ptr(closest),
                                                                           _ptr(bary))
        _abi.check(rc, "tc_closest_point_triangle_host")
    return closest, bary


def degenerate_mask(tris: np.ndarray, rel_tol: float = 1e-12) -> np.ndarray:
    """RK/geometry.py:68-75: squared area below ``rel_tol * longest_edge**4``."""
    t = np.ascontiguousarray(as_triangles(tris))
    mask = np.zeros(t.shape[0], np.uint8)
    if t.shape[0]:
        rc = getattr(_abi.load(), f"tc_degenerate_mask_host_{_sfx(REAL)}")(_ptr(t), t.shape[0], float(rel_tol),
                                                                          _ptr(mask))
        _abi.check(rc, "tc_degenerate_mask_host")
    return mask.astype(bool)


def comparison_batch(tri_a: np.ndarray, tri_b: np.ndarray, eps) -> BatchResult:
    """RK/kernels.py:301-401.  Degenerate triangles must be filtered by the caller."""
    A = as_triangles(tri_a)
    B = as_triangles(tri_b)
    res, _, _ = _run("comparison", A, B, _halo(eps, A.shape[0]), None)
    return res


def iterative_batch(tri_a: np.ndarray, tri_b: np.ndarray, params: KernelParams, eps) -> BatchResult:
    """RK/kernels.py:447-565."""
    A = as_triangles(tri_a)
    B = as_triangles(tri_b)
    res, _, _ = _run("iterative", A, B, _halo(eps, A.shape[0]), params)
    return res


def hybrid_batch(
    tri_a: np.ndarray,
    tri_b: np.ndarray,
    params: KernelParams,
    counters: KernelCounters | None,
    eps,
    allow_fallback=True,
) -> BatchResult:
    """RK/kernels.py:568-605: iterative, then the in-kernel comparison fallback."""
    A = as_triangles(tri_a)
    B = as_triangles(tri_b)
    n = A.shape[0]
    eps = _halo(eps, n)
    if isinstance(allow_fallback, np.ndarray):
        # the reference ANDs the mask into the open pairs (RK/kernels.py:590-591):
        # numpy broadcasting, so a scalar / (1,) mask applies to every pair and
        # any other shape than (n,) raises ValueError
        allow = np.broadcast_to(np.asarray(allow_fallback).astype(bool), (n,))
        res, stats, rc = _run("hybrid", A, B, eps, params, allow=allow)
    elif not allow_fallback:
        res, _, _ = _run("iterative", A, B, eps, params)
        if counters is not None:
            counters.iterative_invocations += n
        return res
    else:
        res, stats, rc = _run("hybrid", A, B, eps, params)
    if counters is not None:
        counters.iterative_invocations += n
    if rc == _abi.TC_EDEGENERATE:
        raise DegenerateTriangle("degenerate triangle in comparison fallback")
    if counters is not None:
        counters.comparison_invocations += int(stats.comparison)
        counters.fallback_invocations += int(stats.fallback)
    return res


# ---------------------------------------------------------------------------
# Scalar API (RK/kernels.py:613-669)
# ---------------------------------------------------------------------------


def closest_comparison(t1, t2, params: KernelParams | None = None) -> DistanceResult:
    params = params or KernelParams()
    A = as_triangles(t1)
    B = as_triangles(t2)
    if degenerate_mask(A)[0] or degenerate_mask(B)[0]:
        raise DegenerateTriangle("degenerate triangle")
    return _scalar(comparison_batch(A, B, params.epsilon))


def closest_iterative(t1, t2, params: KernelParams | None = None) -> DistanceResult:
    params = params or KernelParams()
    return _scalar(iterative_batch(as_triangles(t1), as_triangles(t2), params, params.epsilon))


def closest_hybrid(t1, t2, params: KernelParams | None = None,
                   counters: KernelCounters | None = None) -> DistanceResult:
    params = params or KernelParams()
    return _scalar(hybrid_batch(as_triangles(t1), as_triangles(t2), params, counters, params.epsilon))


def batch_closest(pairs, params: KernelParams | None = None, counters: KernelCounters | None = None):
    """Hybrid over a sequence of pairs; degenerate failures reported positionally."""
    params = params or KernelParams()
    pairs = list(pairs)
    if not pairs:
        return []
    A = as_triangles(np.asarray([p[0] for p in pairs], dtype=REAL))
    B = as_triangles(np.asarray([p[1] for p in pairs], dtype=REAL))
    n = A.shape[0]
    res, stats, _ = _run("hybrid", A, B, np.asarray(params.epsilon, dtype=REAL), params)
    if counters is not None:
        counters.iterative_invocations += n
        counters.comparison_invocations += int(stats.comparison)
        counters.fallback_invocations += int(stats.fallback)
    out: list = []
    for i in range(n):
        if res.kind[i] == 3:
            out.append(DegenerateTriangle(f"degenerate triangle in pair {i}"))
        else:
            out.append(_scalar(res, i))
    return out


# ---------------------------------------------------------------------------
# Penalised functional and its gradient, for verification only
# (RK/kernels.py:417-444, 677-717).  Single pair, not on the hot path.
# ---------------------------------------------------------------------------


def _pair_max_sq_edge(A: np.ndarray, B: np.ndarray) -> np.ndarray:
    # 3-term sums through einsum: the reference's reduction order (RK:409-414)
    def longest(T):
        e = np.roll(T, -1, axis=1) - T
        return np.einsum("ijk,ijk->ij", e, e).max(axis=1)
    return np.maximum(longest(A), longest(B))


def _penalty_terms(x: np.ndarray):
    a1, b1, a2, b2 = x[:, 0], x[:, 1], x[:, 2], x[:, 3]
    return (a1 - 1.0, -a1, b1 - 1.0, -b1, a1 + b1 - 1.0, a2 - 1.0, -a2, b2 - 1.0, -b2, a2 + b2 - 1.0)


def _penalty_value(x: np.ndarray, alpha: np.ndarray) -> np.ndarray:
    return alpha * sum(np.maximum(0.0, t) for t in _penalty_terms(x))


def _penalty_gradient(x: np.ndarray, alpha: np.ndarray) -> np.ndarray:
    """Subgradient of the penalty sum; zero exactly on the kinks."""
    t = [(v > 0.0).astype(REAL) for v in _penalty_terms(x)]
    g = np.stack([t[0] - t[1] + t[4], t[2] - t[3] + t[4], t[5] - t[6] + t[9], t[7] - t[8] + t[9]], axis=1)
    return alpha[:, None] * g


def _diff(A, B, x):
    e1a, e2a = A[:, 1] - A[:, 0], A[:, 2] - A[:, 0]
    e1b, e2b = B[:, 1] - B[:, 0], B[:, 2] - B[:, 0]
    d = A[:, 0] - B[:, 0] + x[:, :1] * e1a + x[:, 1:2] * e2a - x[:, 2:3] * e1b - x[:, 3:4] * e2b
    return d, (e1a, e2a, e1b, e2b)


def _dot(u, v):
    return np.einsum("ij,ij->i", u, v)


def functional_value(t1, t2, a1, b1, a2, b2, params: KernelParams | None = None) -> float:
    params = params or KernelParams()
    A, B = as_triangles(t1), as_triangles(t2)
    x = np.array([[a1, b1, a2, b2]], dtype=REAL)
    d, _ = _diff(A, B, x)
    alpha = params.alpha_iterative * _pair_max_sq_edge(A, B)
    return 0.5 * float(_dot(d, d)[0]) + float(_penalty_value(x, alpha)[0])


def gradient_of_J(t1, t2, a1, b1, a2, b2, params: KernelParams | None = None) -> np.ndarray:
    params = params or KernelParams()
    A, B = as_triangles(t1), as_triangles(t2)
    x = np.array([[a1, b1, a2, b2]], dtype=REAL)
    d, (e1a, e2a, e1b, e2b) = _diff(A, B, x)
    grad_hat = np.stack([_dot(d, e1a), _dot(d, e2a), -_dot(d, e1b), -_dot(d, e2b)], axis=1)
    alpha = params.alpha_iterative * _pair_max_sq_edge(A, B)
    return (grad_hat + _penalty_gradient(x, alpha))[0]
