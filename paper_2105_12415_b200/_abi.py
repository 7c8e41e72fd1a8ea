"""ctypes binding of include/tricontact_b200.h (libtricontact_b200.so).

This is the reference-side binding a maintainer would add: every symbol the
header declares is bound here with its exact C signature.  There is no CPU
fallback -- if the library is missing or no CUDA device is present, the
product entry points raise.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

LIB_PATH = Path(__file__).resolve().parent / "libtricontact_b200.so"

TC_ABI_VERSION = 2  # include/tricontact_b200.h
TC_OK, TC_EINVAL, TC_EDEGENERATE, TC_ECUDA, TC_ENODEVICE = 0, 1, 2, 3, 4
TC_SOA, TC_STRICT, TC_EMIT_IDS = 1, 2, 4
VARIANTS = {"comparison": 0, "iterative": 1, "hybrid": 2}


class TcParams(ctypes.Structure):
    _fields_ = [
        ("epsilon", ctypes.c_double),
        ("c_factor", ctypes.c_double),
        ("alpha_iterative", ctypes.c_double),
        ("alpha_regulariser", ctypes.c_double),
        ("move_factor", ctypes.c_double),
        ("start_coord", ctypes.c_double),
        ("n_iterative", ctypes.c_int32),
        ("flags", ctypes.c_uint32),
    ]


class TcStats(ctypes.Structure):
    _fields_ = [
        ("iterative", ctypes.c_int64),
        ("comparison", ctypes.c_int64),
        ("fallback", ctypes.c_int64),
        ("degenerate", ctypes.c_int64),
        ("contacts", ctypes.c_int64),
        ("intersecting", ctypes.c_int64),
        ("min_distance", ctypes.c_double),
    ]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_INT = ctypes.c_int

# symbol -> (restype, argtypes); mirrors include/tricontact_b200.h one to one
SIGNATURES = {
    "tc_params_default": (None, [_P]),
    "tc_abi_version": (_INT, []),
    "tc_last_error": (ctypes.c_char_p, []),
    "tc_launch_count": (_I64, []),
    "tc_allreduce_stats": (_INT, [_P, _P, _P]),
    "tc_stats_reset": (_INT, [_P, _P]),
    "tc_fma_probe": (_I64, [_INT, _I64, _INT, _P, _P]),
    "tc_host_alloc": (_P, [_I64]),
    "tc_debug_set_max_ctas": (None, [_I64]),
    "tc_debug_fallback_rate_high": (_INT, []),
    "tc_debug_hybrid_mode": (_INT, []),
    "tc_debug_fallback_history": (None, [_P]),
    "tc_host_free": (_INT, [_P]),
    "tc_random_pairs_soa_f64": (_INT, [ctypes.c_uint64, _I64, _I64, ctypes.c_double, ctypes.c_double, _P, _P]),
    "tc_closest_point_triangle_f64": (_INT, [_P, _P, _I64, _P, _P, _P]),
    "tc_closest_point_triangle_f32": (_INT, [_P, _P, _I64, _P, _P, _P]),
    "tc_point_triangle_distance_f64": (_INT, [_P, _P, _I64, _P, _I64, _P, _P, _P]),
    "tc_point_triangle_distance_f32": (_INT, [_P, _P, _I64, _P, _I64, _P, _P, _P]),
    "tc_degenerate_mask_f64": (_INT, [_P, _I64, ctypes.c_double, _P, _P]),
    "tc_degenerate_mask_f32": (_INT, [_P, _I64, ctypes.c_double, _P, _P]),
    "tc_closest_point_triangle_host_f64": (_INT, [_P, _P, _I64, _P, _P]),
    "tc_closest_point_triangle_host_f32": (_INT, [_P, _P, _I64, _P, _P]),
    "tc_degenerate_mask_host_f64": (_INT, [_P, _I64, ctypes.c_double, _P]),
    "tc_degenerate_mask_host_f32": (_INT, [_P, _I64, ctypes.c_double, _P]),
    "tc_run_host_f64": (_INT, [_INT, _P, _P, _I64, _P, _P, _P] + [_P] * 7 + [_P]),
    "tc_run_host_f32": (_INT, [_INT, _P, _P, _I64, _P, _P, _P] + [_P] * 7 + [_P]),
}
for _v in ("comparison", "iterative"):
    for _s in ("f64", "f32"):
        # tri_a, tri_b, n, eps, p, distance, point_a, point_b, bary_a, bary_b, kind, ids, stats, stream
        SIGNATURES[f"tc_{_v}_{_s}"] = (_INT, [_P, _P, _I64, _P, _P] + [_P] * 7 + [_P, _P])
for _s in ("f64", "f32"):
    # tri_a, tri_b, n, eps, allow_fb, p, distance, ..., ids, stats, stream
    SIGNATURES[f"tc_hybrid_{_s}"] = (_INT, [_P, _P, _I64, _P, _P, _P] + [_P] * 7 + [_P, _P])

for _s in ("f64", "f32"):
    # meshes, tris, n_meshes, mesh_tris, motions, blocks, n_blocks, block_eps, p, max_contacts, idx, dist, pa, pb,
    # n_contacts, stats, stream
    SIGNATURES[f"tc_blocks_hybrid_{_s}"] = (_INT, [_P, ctypes.c_int32, _I64, _P, _P, _P, _I64, _P, _P, _I64] + [_P] * 7)

for _s in ("f64", "f32"):
    # tris, node_owner, motions, node_eps, child_off, child_ids, is_fine, height, max_height, roots, n_pairs, p,
    # max_contacts, idx, pa, pb, n_contacts, checks, stats, stream
    SIGNATURES[f"tc_multiscale_{_s}"] = (_INT, [_P] * 8 + [ctypes.c_int32, _P, _I64, _P, _I64] + [_P] * 7)

_lib = None


class TricontactError(RuntimeError):
    pass


def load(path: Path | str | None = None):
    """Load the library and bind every header symbol (raises if absent)."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    p = Path(path) if path else Path(os.environ.get("TC_LIB_PATH", LIB_PATH))
    if not p.exists():
        raise TricontactError(
            f"{p} is missing: build it with `python -m paper_2105_12415_b200._build` "
            "(there is no CPU fallback)")
    lib = ctypes.CDLL(str(p))
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.tc_abi_version() != TC_ABI_VERSION:
        raise TricontactError(f"{p} implements ABI {lib.tc_abi_version()}, this binding expects {TC_ABI_VERSION}: "
                              "rebuild it with `python -m paper_2105_12415_b200._build`")
    if path is None:
        _lib = lib
    return lib


def check(rc: int, what: str = "tricontact call"):
    if rc != TC_OK:
        msg = load().tc_last_error()
        raise TricontactError(f"{what} failed with code {rc}: {msg.decode() if msg else ''}")


def params_struct(params, flags: int = 0) -> TcParams:
    """KernelParams-like object -> TcParams."""
    return TcParams(float(params.epsilon), float(params.c_factor), float(params.alpha_iterative),
                    float(params.alpha_regulariser), float(params.move_factor), float(params.start_coord),
                    int(params.n_iterative), int(flags))

