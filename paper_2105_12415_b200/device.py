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


def _on_stream(t: torch.Tensor | None, st) -> torch.Tensor | None:
    """Mark a tensor used on stream ``st`` (a caller-supplied stream may still
    read it after this function returns and the caching allocator reuses it)."""
    if t is not None and st != torch.cuda.current_stream(t.device):
        t.record_stream(st)
    return t


def _per_pair(x, n: int, dtype, device, what: str) -> torch.Tensor | None:
    """A per-pair column: a scalar (or 1-element tensor) broadcasts to n, any
    other shape must hold exactly n elements."""
    if x is None:
        return None
    x = torch.as_tensor(x)
    if x.numel() == 1 and n != 1:
        x = x.reshape(1).expand(n)
    if x.numel() != n:
        raise ValueError(f"{what} must be a scalar or hold n = {n} elements, got shape {tuple(x.shape)}")
    return x.reshape(n).to(device=device, dtype=dtype).contiguous()


def _check_out(out: dict, n: int, dtype, device, soa: bool) -> None:
    shapes = {"kind": (n,), "distance": (n,), "point_a": (3, n) if soa else (n, 3),
              "point_b": (3, n) if soa else (n, 3), "bary_a": (2, n) if soa else (n, 2),
              "bary_b": (2, n) if soa else (n, 2), "ids": (n, 4)}
    dts = {"kind": torch.int8, "ids": torch.uint8}
    for k, t in out.items():
        if k not in shapes:
            raise ValueError(f"unknown output column {k!r}")
        want = dts.get(k, dtype)
        if t.dtype != want or t.device != device or tuple(t.shape) != shapes[k] or not t.is_contiguous():
            raise ValueError(f"output {k!r} must be a contiguous {want} tensor of shape {shapes[k]} on {device}")


def run(variant: str, tri_a: torch.Tensor, tri_b: torch.Tensor, params=None, *, eps=None, allow=None,
        soa: bool = False, strict: bool = False, out: dict | None = None, ids: bool = False,
        stats: torch.Tensor | None = None, stream=None, n: int | None = None) -> dict | None:
    """Enqueue one kernel launch; returns the output dict (or None if out == {}).

    ``out``: None allocates the full result record; ``{}`` is reduce-only
    (only ``stats`` is written); a dict of preallocated tensors is filled.
    ``eps`` / ``allow``: per-pair halo / fallback mask, a scalar or n values.
    """
    if tri_a.dtype not in _DT or tri_b.dtype != tri_a.dtype:
        raise TypeError("tri_a / tri_b must both be float64 or float32")
    if not (tri_a.is_cuda and tri_b.is_cuda) or tri_a.device != tri_b.device:
        raise ValueError("device entry points take CUDA tensors on one device")
    if not (tri_a.is_contiguous() and tri_b.is_contiguous()):
        raise ValueError("inputs must be contiguous")
    dev = tri_a.device
    if n is None:
        n = tri_a.shape[-1] if soa else tri_a.shape[0]
    cap = min(tri_a.numel(), tri_b.numel()) // 9
    if soa:
        if tri_a.shape[0] != 9 or tri_b.shape[0] != 9 or n > tri_a.shape[-1] or n > tri_b.shape[-1]:
            raise ValueError("SoA inputs must be [9][m] planes with m >= n")
    elif n > cap:
        raise ValueError(f"n = {n} exceeds the inputs' {cap} triangle pairs")
    params = params or Params()
    flags = (_abi.TC_SOA if soa else 0) | (_abi.TC_STRICT if strict else 0) | (_abi.TC_EMIT_IDS if ids else 0)
    p = _abi.params_struct(params, flags)
    if out is None:
        out = alloc_outputs(n, tri_a.dtype, dev, soa=soa, ids=ids)
    else:
        _check_out(out, n, tri_a.dtype, dev, soa)
    if stats is not None and (stats.device != dev or stats.dtype != torch.int64 or stats.numel() != STATS_WORDS):
        raise ValueError("stats must be the 7-word int64 tensor of new_stats() on the inputs' device")
    st = stream if stream is not None else torch.cuda.current_stream(dev)
    eps = _on_stream(_per_pair(eps, n, tri_a.dtype, dev, "eps"), st)
    allow = _on_stream(_per_pair(allow, n, torch.uint8, dev, "allow"), st)
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
    for t in out.values():
        _on_stream(t, st)
    return out


def closest_point_triangle(points: torch.Tensor, tris: torch.Tensor, stream=None):
    if points.dtype != tris.dtype or tris.dtype not in _DT or not (points.is_cuda and tris.is_cuda):
        raise TypeError("points and tris must be CUDA tensors of one dtype (float64 or float32)")
    n = tris.shape[0]
    if tris.numel() != 9 * n or points.numel() != 3 * n:
        raise ValueError("expected points (n, 3) and tris (n, 3, 3)")
    closest = torch.empty((n, 3), dtype=tris.dtype, device=tris.device)
    bary = torch.empty((n, 2), dtype=tris.dtype, device=tris.device)
    st = stream if stream is not None else torch.cuda.current_stream(tris.device)
    pc, tc_ = _on_stream(points.contiguous(), st), _on_stream(tris.contiguous(), st)
    rc = getattr(_abi.load(), f"tc_closest_point_triangle_{_DT[tris.dtype]}")(
        _p(pc), _p(tc_), n, _p(closest), _p(bary), ctypes.c_void_p(st.cuda_stream))
    _abi.check(rc, "tc_closest_point_triangle")
    _on_stream(closest, st)
    _on_stream(bary, st)
    return closest, bary


def degenerate_mask(tris: torch.Tensor, rel_tol: float = 1e-12, stream=None) -> torch.Tensor:
    """RK/geometry.py:68-75 on a CUDA (n, 3, 3) tensor."""
    if tris.dtype not in _DT or not tris.is_cuda:
        raise TypeError("tris must be a float64/float32 CUDA tensor")
    n = tris.shape[0]
    if tris.numel() != 9 * n:
        raise ValueError("expected tris (n, 3, 3)")
    mask = torch.empty(n, dtype=torch.uint8, device=tris.device)
    st = stream if stream is not None else torch.cuda.current_stream(tris.device)
    tc_ = _on_stream(tris.contiguous(), st)
    rc = getattr(_abi.load(), f"tc_degenerate_mask_{_DT[tris.dtype]}")(
        _p(tc_), n, float(rel_tol), _p(mask), ctypes.c_void_p(st.cuda_stream))
    _abi.check(rc, "tc_degenerate_mask")
    with torch.cuda.stream(st):
        return mask.bool()


def launch_count() -> int:
    return int(_abi.load().tc_launch_count())
