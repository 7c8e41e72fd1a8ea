"""Device-resident entry points on torch CUDA tensors.

PyTorch is plumbing here: it owns device memory and streams; the compute is
the C-ABI library (device entry points of include/tricontact_b200.h), called
with raw device pointers and the current torch stream.  Nothing in this
module computes on the host; every call fails loudly without the library.

Inputs are either the reference layout (two (n, 3, 3) tensors) or the
planar SoA layout (two [9][n] tensors, ``soa=True``).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import torch

from . import _abi

_DT = {torch.float64: "f64", torch.float32: "f32"}
STATS_WORDS = 7  # tc_stats = 6 x int64 + 1 x double


@dataclass
class Params:
    """KernelParams mirror (RK/kernels.py:42-72) for the device API."""

    epsilon: float = 1e-2
    n_iterative: int = 4
    c_factor: float = 1.0
    alpha_iterative: float = 10.0
    alpha_regulariser: float = 1e-4
    move_factor: float = 0.25
    start_coord: float = 1.0 / 3.0


def _p(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def new_stats(device="cuda") -> torch.Tensor:
    s = torch.zeros(STATS_WORDS, dtype=torch.int64, device=device)
    reset_stats(s)
    return s


def reset_stats(stats: torch.Tensor, stream=None) -> None:
    st = stream if stream is not None else torch.cuda.current_stream(stats.device)
    _abi.check(_abi.load().tc_stats_reset(_p(stats), ctypes.c_void_p(st.cuda_stream)), "tc_stats_reset")


def read_stats(stats: torch.Tensor) -> dict:
    h = stats.cpu()
    return {
        "iterative": int(h[0]), "comparison": int(h[1]), "fallback": int(h[2]),
        "degenerate": int(h[3]), "contacts": int(h[4]), "intersecting": int(h[5]),
        "min_distance": float(h[6:7].view(torch.float64)[0]),
    }


def alloc_outputs(n: int, dtype, device, soa: bool = False, ids: bool = False) -> dict:
    if soa:
        shp3, shp2 = (3, n), (2, n)
    else:
        shp3, shp2 = (n, 3), (n, 2)
    out = {
        "kind": torch.empty(n, dtype=torch.int8, device=device),
        "distance": torch.empty(n, dtype=dtype, device=device),
        "point_a": torch.empty(shp3, dtype=dtype, device=device),
        "point_b": torch.empty(shp3, dtype=dtype, device=device),
        "bary_a": torch.empty(shp2, dtype=dtype, device=device),
        "bary_b": torch.empty(shp2, dtype=dtype, device=device),
    }
    if ids:
        out["ids"] = torch.empty((n, 4), dtype=torch.uint8, device=device)
    return out


def run(variant: str, tri_a: torch.Tensor, tri_b: torch.Tensor, params=None, *, eps=None, allow=None,
        soa: bool = False, strict: bool = False, out: dict | None = None, ids: bool = False,
        stats: torch.Tensor | None = None, stream=None, n: int | None = None) -> dict | None:
    """Enqueue one kernel launch; returns the output dict (or None if out == {}).

    ``out``: None allocates the full result record; ``{}`` is reduce-only
    (only ``stats`` is written); a dict of preallocated tensors is filled.
    """
    if tri_a.dtype not in _DT or tri_b.dtype != tri_a.dtype:
        raise TypeError("tri_a / tri_b must both be float64 or float32")
    if not (tri_a.is_cuda and tri_b.is_cuda):
        raise ValueError("device entry points take CUDA tensors")
    if not (tri_a.is_contiguous() and tri_b.is_contiguous()):
        raise ValueError("inputs must be contiguous")
    if n is None:
        n = tri_a.shape[-1] if soa else tri_a.shape[0]
    params = params or Params()
    flags = (_abi.TC_SOA if soa else 0) | (_abi.TC_STRICT if strict else 0) | (_abi.TC_EMIT_IDS if ids else 0)
    p = _abi.params_struct(params, flags)
    if out is None:
        out = alloc_outputs(n, tri_a.dtype, tri_a.device, soa=soa, ids=ids)
    st = stream if stream is not None else torch.cuda.current_stream(tri_a.device)
    if eps is not None:
        eps = eps.to(device=tri_a.device, dtype=tri_a.dtype).contiguous()
    if allow is not None:
        allow = allow.to(device=tri_a.device, dtype=torch.uint8).contiguous()
    g = out.get
    cols = [_p(g("distance")), _p(g("point_a")), _p(g("point_b")), _p(g("bary_a")), _p(g("bary_b")),
            _p(g("kind")), _p(g("ids"))]
    lib = _abi.load()
    sfx = _DT[tri_a.dtype]
    s = ctypes.c_void_p(st.cuda_stream)
    if variant == "hybrid":
        rc = getattr(lib, f"tc_hybrid_{sfx}")(_p(tri_a), _p(tri_b), n, _p(eps), _p(allow), ctypes.byref(p),
                                               *cols, _p(stats), s)
    elif variant in ("iterative", "comparison"):
        if allow is not None:
            raise ValueError("allow_fallback applies to the hybrid variant only")
        rc = getattr(lib, f"tc_{variant}_{sfx}")(_p(tri_a), _p(tri_b), n, _p(eps), ctypes.byref(p), *cols,
                                                  _p(stats), s)
    else:
        raise ValueError(f"unknown variant {variant!r}")
    _abi.check(rc, f"tc_{variant}_{sfx}")
    return out


def closest_point_triangle(points: torch.Tensor, tris: torch.Tensor, stream=None):
    n = tris.shape[0]
    closest = torch.empty((n, 3), dtype=tris.dtype, device=tris.device)
    bary = torch.empty((n, 2), dtype=tris.dtype, device=tris.device)
    st = stream if stream is not None else torch.cuda.current_stream(tris.device)
    rc = getattr(_abi.load(), f"tc_closest_point_triangle_{_DT[tris.dtype]}")(
        _p(points.contiguous()), _p(tris.contiguous()), n, _p(closest), _p(bary), ctypes.c_void_p(st.cuda_stream))
    _abi.check(rc, "tc_closest_point_triangle")
    return closest, bary


def degenerate_mask(tris: torch.Tensor, stream=None) -> torch.Tensor:
    n = tris.shape[0]
    mask = torch.empty(n, dtype=torch.uint8, device=tris.device)
    st = stream if stream is not None else torch.cuda.current_stream(tris.device)
    rc = getattr(_abi.load(), f"tc_degenerate_mask_{_DT[tris.dtype]}")(
        _p(tris.contiguous()), n, _p(mask), ctypes.c_void_p(st.cuda_stream))
    _abi.check(rc, "tc_degenerate_mask")
    return mask.bool()


def launch_count() -> int:
    return int(_abi.load().tc_launch_count())
