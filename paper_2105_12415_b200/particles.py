"""All-pairs particle blocks (BASELINE.json config 2) and their device entry.

A "block" is a pair of particle meshes whose every triangle pair goes through
the hybrid kernel -- the all-pairs meshgrid of the reference's flat detection
(RK/stepping.py:285-308 single_level_contacts, RK/contact.py:97-140
find_contacts_single_level).  The device kernel stages both meshes of a block
in shared memory and never materialises the pair list
(``tc_blocks_hybrid_*``, include/tricontact_b200.h).

cfg2 scene (synthetic, seeded): 2,048 icosphere(2) particles
(320 triangles, 162 vertices, radius 1) with a per-vertex radial jitter
x(1 + U(-0.05, 0.05)) and a random rotation each, on a 16 x 16 x 8 lattice of
spacing 2 * 1.05 + 0.025 with a per-particle jitter U(+-0.0125)^3, so the
bounding-sphere gaps fall in [0, 0.05]; blocks are the 6-neighbour pairs with
gap <= 0.1 (5,632 blocks x 102,400 pairs).  The mesh is built here (the
reference's scenes.icosphere is not available on the GPU box); its vertex
order may differ from the reference's, which does not matter for the
benchmark.  The reference's own particles use outward-only value noise
(RK/scenes.py:196-217); the symmetric jitter is BASELINE.json's.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _abi
from .workloads import rotation_matrices


def icosahedron():
    t = (1.0 + 5.0 ** 0.5) / 2.0
    v = np.array([[-1, t, 0], [1, t, 0], [-1, -t, 0], [1, -t, 0],
                  [0, -1, t], [0, 1, t], [0, -1, -t], [0, 1, -t],
                  [t, 0, -1], [t, 0, 1], [-t, 0, -1], [-t, 0, 1]], float)
    v /= np.linalg.norm(v, axis=1, keepdims=True)
    f = np.array([[0, 11, 5], [0, 5, 1], [0, 1, 7], [0, 7, 10], [0, 10, 11],
                  [1, 5, 9], [5, 11, 4], [11, 10, 2], [10, 7, 6], [7, 1, 8],
                  [3, 9, 4], [3, 4, 2], [3, 2, 6], [3, 6, 8], [3, 8, 9],
                  [4, 9, 5], [2, 4, 11], [6, 2, 10], [8, 6, 7], [9, 8, 1]], np.int64)
    return v, f


def icosphere(level: int):
    """Unit icosphere: 10*4^level + 2 vertices, 20*4^level outward-facing triangles."""
    v, f = icosahedron()
    verts = [tuple(x) for x in v]
    for _ in range(level):
        cache = {}

        def mid(a, b):
            key = (min(a, b), max(a, b))
            if key not in cache:
                m = (np.asarray(verts[a]) + np.asarray(verts[b])) / 2.0
                verts.append(tuple(m / np.linalg.norm(m)))
                cache[key] = len(verts) - 1
            return cache[key]

        nf = []
        for a, b, c in f:
            ab, bc, ca = mid(a, b), mid(b, c), mid(c, a)
            nf += [[a, ab, ca], [b, bc, ab], [c, ca, bc], [ab, bc, ca]]
        f = np.array(nf, np.int64)
    return np.array(verts), f


SPACING = 2 * 1.05 + 0.025


def cfg2_scene(grid=(16, 16, 8), level: int = 2, seed: int = 2, jitter: float = 0.05,
               pos_jitter: float = 0.0125, cutoff: float = 0.1):
    """(meshes (N, T, 3, 3) world triangles, blocks (nb, 2) int32, gaps (nb,))."""
    rng = np.random.default_rng(seed)
    v0, faces = icosphere(level)
    nx, ny, nz = grid
    N = nx * ny * nz
    radial = 1.0 + rng.uniform(-jitter, jitter, (N, v0.shape[0]))
    q = rng.normal(size=(N, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    R = rotation_matrices(q)
    ijk = np.stack(np.meshgrid(np.arange(nx), np.arange(ny), np.arange(nz), indexing="ij"), -1).reshape(-1, 3)
    centers = ijk * SPACING + rng.uniform(-pos_jitter, pos_jitter, (N, 3))
    local = v0[None] * radial[..., None]                               # (N, V, 3)
    world = np.einsum("nij,nvj->nvi", R, local) + centers[:, None, :]
    meshes = world[:, faces]                                           # (N, T, 3, 3)
    rmax = np.linalg.norm(local, axis=2).max(axis=1)
    idx = np.arange(N).reshape(nx, ny, nz)
    pairs = []
    for axis in range(3):
        a = np.take(idx, np.arange(idx.shape[axis] - 1), axis=axis).ravel()
        b = np.take(idx, np.arange(1, idx.shape[axis]), axis=axis).ravel()
        pairs.append(np.stack([a, b], 1))
    pairs = np.concatenate(pairs)
    gaps = np.linalg.norm(centers[pairs[:, 0]] - centers[pairs[:, 1]], axis=1) - rmax[pairs[:, 0]] - rmax[pairs[:, 1]]
    keep = gaps <= cutoff
    return np.ascontiguousarray(meshes), pairs[keep].astype(np.int32), gaps[keep]


def cfg2_scene_local(**kw):
    """cfg2 as local-space meshes + rigid motions (N, 7): each particle's
    jittered mesh centred at the origin, rotated and translated by its motion."""
    rng = np.random.default_rng(kw.pop("seed", 2))
    meshes, blocks, gaps = cfg2_scene(seed=int(rng.integers(1 << 30)), **kw)
    N = meshes.shape[0]
    centers = meshes.reshape(N, -1, 3).mean(axis=1)
    local = meshes - centers[:, None, None, :]
    q = rng.normal(size=(N, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    Rt = rotation_matrices(q)
    # local = R^T (world - c): the motion (q, c) maps it back near the world pose
    local = np.einsum("nji,ntvj->ntvi", Rt, local)
    motions = np.concatenate([q, centers], axis=1)
    return np.ascontiguousarray(local), motions, blocks, gaps


def block_pairs(meshes: np.ndarray, blocks: np.ndarray, which):
    """Materialise the (A, B) triangle pairs of the listed blocks (oracle checks):
    pair (i, j) of block b is at row b_pos * T * T + i * T + j."""
    T = meshes.shape[1]
    As, Bs = [], []
    for b in which:
        ma, mb = meshes[blocks[b, 0]], meshes[blocks[b, 1]]
        As.append(np.repeat(ma, T, axis=0))
        Bs.append(np.tile(mb, (T, 1, 1)))
    return np.concatenate(As), np.concatenate(Bs)


def blocks_hybrid(meshes, blocks, params, *, motions=None, block_eps=None, mesh_tris=None, strict=False,
                  max_contacts=1 << 20, stats=None, stream=None):
    """Hybrid kernel over every triangle pair of every block (device tensors).

    ``meshes``: (N, T, 3, 3) CUDA tensor (world space, or local space with
    ``motions`` (N, 7) = quaternion (w, x, y, z) + translation, applied while
    the meshes are staged); ``blocks``: (nb, 2) int32 CUDA tensor;
    ``mesh_tris``: (N,) triangles per mesh for ragged meshes padded to T.
    A block (m, m) skips the diagonal (a triangle is never tested against itself).
    Returns a dict: n_contacts (device int64 scalar tensor) and the contact
    arrays idx (max, 3) int32 [block, tri_a, tri_b], distance, point_a, point_b
    (unordered; ``sort_contacts`` orders them like the reference).
    """
    import torch
    from .device import _DT, _on_stream, _p

    if meshes.dtype not in _DT or not meshes.is_cuda or not meshes.is_contiguous():
        raise ValueError("meshes must be a contiguous CUDA float64/float32 tensor (N, T, 3, 3)")
    blocks = torch.as_tensor(blocks).to(device=meshes.device, dtype=torch.int32).contiguous()
    if blocks.dim() != 2 or blocks.shape[1] != 2:
        raise ValueError("blocks must be (nb, 2) mesh indices")
    dev, dt = meshes.device, meshes.dtype
    out = {
        "n_contacts": torch.zeros(1, dtype=torch.int64, device=dev),
        "idx": torch.empty((max_contacts, 3), dtype=torch.int32, device=dev),
        "distance": torch.empty(max_contacts, dtype=dt, device=dev),
        "point_a": torch.empty((max_contacts, 3), dtype=dt, device=dev),
        "point_b": torch.empty((max_contacts, 3), dtype=dt, device=dev),
    }
    p = _abi.params_struct(params, _abi.TC_STRICT if strict else 0)
    st = stream if stream is not None else torch.cuda.current_stream(dev)
    if block_eps is not None:
        block_eps = block_eps.to(device=dev, dtype=dt).contiguous()
    if motions is not None:
        motions = motions.to(device=dev, dtype=dt).contiguous()
    if mesh_tris is not None:
        mesh_tris = torch.as_tensor(mesh_tris, dtype=torch.int32).to(dev).contiguous()
        if mesh_tris.numel() != meshes.shape[0]:
            raise ValueError("mesh_tris must hold one count per mesh")
    if block_eps is not None and block_eps.numel() != blocks.shape[0]:
        raise ValueError("block_eps must hold one halo per block")
    if motions is not None and tuple(motions.shape) != (meshes.shape[0], 7):
        raise ValueError("motions must be (N, 7): quaternion (w, x, y, z) + translation")
    if stats is not None and (stats.device != dev or stats.dtype != torch.int64 or stats.numel() != 7):
        raise ValueError("stats must be the 7-word int64 tensor of device.new_stats() on the meshes' device")
    for t in (blocks, block_eps, motions, mesh_tris, *out.values()):
        _on_stream(t, st)
    fn = getattr(_abi.load(), f"tc_blocks_hybrid_{_DT[dt]}")
    rc = fn(_p(meshes), int(meshes.shape[1]), int(meshes.shape[0]), _p(mesh_tris), _p(motions), _p(blocks),
            int(blocks.shape[0]),
            _p(block_eps), ctypes.byref(p), int(max_contacts), _p(out["idx"]), _p(out["distance"]),
            _p(out["point_a"]), _p(out["point_b"]), _p(out["n_contacts"]), _p(stats),
            ctypes.c_void_p(st.cuda_stream))
    _abi.check(rc, "tc_blocks_hybrid")
    return out


def sort_contacts(out: dict) -> dict:
    """Host copy of the contact list ordered by (block, tri_a, tri_b).

    Raises if the launch found more contacts than ``max_contacts`` slots:
    the stored subset would depend on atomic slot order (rerun with
    ``max_contacts >= n_contacts``; the count is exact)."""
    n = int(out["n_contacts"].item())
    if n > out["idx"].shape[0]:
        raise RuntimeError(f"{n} contacts found but only max_contacts = {out['idx'].shape[0]} stored; "
                           "rerun blocks_hybrid with max_contacts >= n_contacts")
    m = n
    idx = out["idx"][:m].cpu().numpy()
    order = np.lexsort((idx[:, 2], idx[:, 1], idx[:, 0]))
    res = {"n_contacts": n, "idx": idx[order]}
    for k in ("distance", "point_a", "point_b"):
        res[k] = out[k][:m].cpu().numpy()[order]
    return res
