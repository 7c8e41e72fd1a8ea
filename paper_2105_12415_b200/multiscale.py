"""Device multiscale traversal.

RK/stepping.py:311-368 ``multiscale_contacts`` for many particle pairs in one
call: the surrogate trees of all particles (RK/stepping.py:78-129 FlatTree)
are concatenated into one global id space on the device, the frontier of
every particle pair is advanced together -- one hybrid launch and one
unfolding per round -- and the mesh-level contacts come back as
(pair, source_i, source_j, point_a, point_b).  ``contact_points`` then places
them on their segments like RK/contact.py:75-94 ``contact_from_segment`` and
orders them like RK/stepping.py:281 ``_sorted_contacts``.

The tree arrays here are plain arrays (world coordinates under each
particle's motion, halos, CSR children, heights); ``FlatTreeArrays.from_reference``
builds them from a reference ``FlatTree`` when one is at hand.
"""

from __future__ import annotations

import ctypes
import time
from dataclasses import dataclass, field

import numpy as np

from . import _abi
from .contact import contact_from_segment_batch


@dataclass
class FlatTreeArrays:
    """One particle's FlatTree in array form (ids: nodes in preorder, then mesh triangles)."""

    tris: np.ndarray        # (n_total, 3, 3) world coordinates (local ones when the forest has motions)
    eps: np.ndarray         # (n_total,)
    child_off: np.ndarray   # (n_total + 1,) CSR offsets
    child_ids: np.ndarray   # children ids (local)
    height: np.ndarray      # (n_total,) 0 = mesh level
    n_nodes: int            # surrogate nodes; ids >= n_nodes are mesh triangles

    @classmethod
    def from_reference(cls, flat, world_tris):
        """From a reference FlatTree (RK/stepping.py:78) and its world triangles."""
        off = np.zeros(flat.tri.shape[0] + 1, np.int32)
        off[1:] = np.cumsum([c.size for c in flat.children])
        ids = np.concatenate([c for c in flat.children if c.size]).astype(np.int32)
        return cls(np.asarray(world_tris), np.asarray(flat.eps), off, ids, np.asarray(flat.height, np.int32),
                   int(flat.n_nodes))

    @property
    def n_total(self) -> int:
        return int(self.eps.shape[0])


@dataclass
class Forest:
    """All particles' trees concatenated on the device (global ids)."""

    tris: object
    eps: object
    child_off: object
    child_ids: object
    is_fine: object
    height: object
    base: np.ndarray        # (n_particles,) global id of each root
    n_nodes: np.ndarray     # (n_particles,)
    max_height: int
    host_eps: np.ndarray = field(repr=False, default=None)
    owner: object = None    # (n_total,) int32 particle of each node (with motions)
    motions: object = None  # (n_particles, 7) quaternion (w, x, y, z) + translation, or None

    def set_motions(self, motions) -> None:
        """Rigid motions of every particle (the trees then hold local coordinates)."""
        import torch
        m = torch.as_tensor(np.asarray(motions), dtype=self.tris.dtype).to(self.tris.device).contiguous()
        if m.shape != (self.base.shape[0], 7):
            raise ValueError("motions must be (n_particles, 7)")
        if self.owner is None:
            sizes = np.diff(np.append(self.base, self.tris.shape[0]))
            own = np.repeat(np.arange(self.base.shape[0], dtype=np.int32), sizes)
            self.owner = torch.from_numpy(own).to(self.tris.device)
        self.motions = m


def build_forest(trees: list[FlatTreeArrays], device="cuda", dtype=None, motions=None) -> Forest:
    """Concatenate trees into one device-resident global id space.  With
    ``motions`` (n_particles, 7) the trees hold local coordinates and every
    node is transformed by its particle's motion as the kernel loads it."""
    import torch

    dtype = dtype or trees[0].tris.dtype
    sizes = np.array([t.n_total for t in trees], np.int64)
    base = np.zeros(len(trees), np.int64)
    base[1:] = np.cumsum(sizes)[:-1]
    tris = np.concatenate([np.asarray(t.tris, dtype).reshape(-1, 9) for t in trees])
    eps = np.concatenate([np.asarray(t.eps, dtype) for t in trees])
    off = [np.zeros(1, np.int64)]
    ids, acc = [], 0
    for t, b in zip(trees, base):
        off.append(np.asarray(t.child_off[1:], np.int64) + acc)
        acc += int(t.child_off[-1])
        ids.append(np.asarray(t.child_ids, np.int64) + b)
    child_off = np.concatenate(off)
    child_ids = np.concatenate(ids) if ids else np.zeros(0, np.int64)
    if acc >= 2 ** 31 or tris.shape[0] >= 2 ** 31:
        raise ValueError("forest exceeds int32 ids")
    is_fine = np.concatenate([np.arange(t.n_total) >= t.n_nodes for t in trees]).astype(np.uint8)
    height = np.concatenate([np.asarray(t.height, np.int32) for t in trees])
    tt = lambda a, dt: torch.as_tensor(np.ascontiguousarray(a), dtype=dt, device=device)  # noqa: E731
    fdt = torch.float64 if np.dtype(dtype) == np.float64 else torch.float32
    forest = Forest(tt(tris, fdt), tt(eps, fdt), tt(child_off, torch.int32), tt(child_ids, torch.int32),
                    tt(is_fine, torch.uint8), tt(height, torch.int32), base,
                    np.array([t.n_nodes for t in trees], np.int64), int(height.max()), eps)
    if motions is not None:
        forest.set_motions(motions)
    return forest


@dataclass
class MultiscaleResult:
    n_contacts: int
    pair: np.ndarray        # (n,) particle-pair index
    id_i: np.ndarray        # (n,) global ids
    id_j: np.ndarray
    point_a: np.ndarray     # (n, 3)
    point_b: np.ndarray
    checks: np.ndarray      # (max_height + 1,) pairings per max height
    stats: dict
    call_ms: float = 0.0    # wall time of the library call (synchronous)


def multiscale_contacts(forest: Forest, pairs, params, *, strict=True, max_contacts=1 << 20,
                        stream=None) -> MultiscaleResult:
    """Traverse every (particle_i, particle_j) of ``pairs`` (n, 2) on the device.

    ``max_contacts`` sizes the first attempt's contact list; when the traversal
    finds more (the count is exact), it is re-run with room for all of them, so
    the result never depends on which contacts won the atomic slots."""
    import torch
    from .device import _DT, _p

    pairs = np.asarray(pairs, np.int64).reshape(-1, 2)
    roots = np.ascontiguousarray(forest.base[pairs].astype(np.int32))
    dev, dt = forest.tris.device, forest.tris.dtype
    p = _abi.params_struct(params, _abi.TC_STRICT if strict else 0)
    s = stream if stream is not None else torch.cuda.current_stream(dev)
    fn = getattr(_abi.load(), f"tc_multiscale_{_DT[dt]}")
    cap = max(int(max_contacts), 1)
    while True:
        idx = torch.empty((cap, 3), dtype=torch.int32, device=dev)
        pa = torch.empty((cap, 3), dtype=dt, device=dev)
        pb = torch.empty((cap, 3), dtype=dt, device=dev)
        n_contacts = ctypes.c_int64(0)
        checks = np.zeros(forest.max_height + 1, np.int64)
        st = _abi.TcStats()
        st.min_distance = float("inf")
        t0 = time.perf_counter()
        rc = fn(_p(forest.tris), _p(forest.owner), _p(forest.motions), _p(forest.eps), _p(forest.child_off),
                _p(forest.child_ids), _p(forest.is_fine), _p(forest.height), int(forest.max_height),
                roots.ctypes.data, int(roots.shape[0]), ctypes.byref(p), int(cap), _p(idx), _p(pa), _p(pb),
                ctypes.byref(n_contacts), checks.ctypes.data, ctypes.byref(st), ctypes.c_void_p(s.cuda_stream))
        call_ms = (time.perf_counter() - t0) * 1e3
        if rc == _abi.TC_EDEGENERATE:
            from .kernels import DegenerateTriangle
            raise DegenerateTriangle("degenerate triangle in comparison fallback")
        _abi.check(rc, "tc_multiscale")
        n = int(n_contacts.value)
        if n <= cap:
            break
        cap = n  # the list overflowed: traverse again with room for every contact
    # order by (pair, id_i, id_j) on the device: three stable sorts, last key first
    with torch.cuda.stream(s):
        d_idx = idx[:n]
        perm = torch.arange(n, device=dev)
        for col in (2, 1, 0):
            perm = perm[torch.sort(d_idx[perm, col], stable=True).indices]
        ih = d_idx[perm].cpu().numpy()
        pa_h = pa[:n][perm].cpu().numpy()
        pb_h = pb[:n][perm].cpu().numpy()
    stats = {k: getattr(st, k) for k in ("iterative", "comparison", "fallback", "degenerate", "contacts",
                                         "intersecting", "min_distance")}
    return MultiscaleResult(n, ih[:, 0], ih[:, 1], ih[:, 2], pa_h, pb_h, checks, stats, call_ms)


def contact_points(forest: Forest, res: MultiscaleResult, pairs):
    """RK/contact.py:75-94 contact_from_segment on every contact, ordered by
    (pair, source) (RK/stepping.py:281).  Returns a dict of arrays:
    pair (n, 2) particle ids, source (n, 2) mesh triangle indices, position,
    normal (n, 3), eps (n, 2)."""
    pairs = np.asarray(pairs, np.int64).reshape(-1, 2)
    owner = np.searchsorted(forest.base, np.concatenate([res.id_i, res.id_j]), side="right") - 1
    oi, oj = owner[: res.id_i.size], owner[res.id_i.size:]
    src_i = res.id_i - forest.base[oi] - forest.n_nodes[oi]
    src_j = res.id_j - forest.base[oj] - forest.n_nodes[oj]
    eps_a = forest.host_eps[res.id_i].astype(np.float64)
    eps_b = forest.host_eps[res.id_j].astype(np.float64)
    position, normal = contact_from_segment_batch(res.point_a, res.point_b, eps_a, eps_b)
    order = np.lexsort((src_j, src_i, pairs[res.pair, 1], pairs[res.pair, 0]))
    return dict(pair=pairs[res.pair][order], source=np.stack([src_i, src_j], 1)[order], position=position[order],
                normal=normal[order], eps=np.stack([eps_a, eps_b], 1)[order])
