"""Contact emission on the device kernels.

Mirrors the detection half of the reference's ``tricontact.contact``
(RK/contact.py): ``ContactPoint`` (:31-42), ``contact_from_segment``
(:75-94) and ``find_contacts_single_level`` (:97-140), plus
``contact_from_segment_batch``, the same placement for whole contact
arrays, which the device callers (particle blocks, multiscale traversal)
use.  Force models, mass properties and ``merge_contacts`` (greedy,
order-dependent) stay with the reference.

``find_contacts_single_level`` runs the all-pairs meshgrid as one block of
the particle-block kernel (both soups staged in shared memory, the pair
list never materialised, diagonal skipped for a soup against itself);
soups too large for the staging go through ``kernels.hybrid_batch`` in
chunks, like the reference.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import kernels as K

# largest soup the block kernel stages in shared memory (per dtype)
_STAGE_LIMIT = {np.dtype(np.float64): 1200, np.dtype(np.float32): 2400}


@dataclass
class ContactPoint:
    """RK/contact.py:31-42."""

    position: np.ndarray
    normal: np.ndarray
    pair: tuple
    source: tuple = (-1, -1)
    level: tuple = (0, 0)
    eps: tuple = (1e-2, 1e-2)

    @property
    def depth(self) -> float:
        """Spring engagement in [0, 1]: 0 at halo touch, 1 at surface touch."""
        return 1.0 - float(np.linalg.norm(self.normal)) / self.eps[0]


def contact_from_segment(point_a, point_b, eps_a: float, eps_b: float, pair=(0, 1), source=(-1, -1),
                         level=(0, 0), fallback_dir=None) -> ContactPoint:
    """RK/contact.py:75-94: the contact divides the segment a->b in the ratio
    eps_a : eps_b; coincident points take ``fallback_dir`` with zero magnitude."""
    point_a = np.asarray(point_a, dtype=K.REAL)
    point_b = np.asarray(point_b, dtype=K.REAL)
    w = eps_a / (eps_a + eps_b)
    position = point_a + w * (point_b - point_a)
    normal = point_a - position
    if np.linalg.norm(normal) < 1e-12:
        direction = np.zeros(3, dtype=K.REAL) if fallback_dir is None else np.asarray(fallback_dir, dtype=K.REAL)
        normal = 0.0 * direction
    return ContactPoint(position, normal, tuple(pair), tuple(source), tuple(level), (eps_a, eps_b))


def contact_from_segment_batch(point_a: np.ndarray, point_b: np.ndarray, eps_a, eps_b):
    """``contact_from_segment`` over (n, 3) arrays with per-contact halos:
    (position, normal), rounded exactly like n scalar calls (the halo weight
    is formed in double, as the reference's Python floats, then cast to the
    array type as NumPy 2 casts a Python scalar)."""
    real = point_a.dtype
    ea = np.asarray(eps_a, np.float64)
    eb = np.asarray(eps_b, np.float64)
    w = np.broadcast_to(ea / (ea + eb), (point_a.shape[0],)).astype(real)
    position = point_a + w[:, None] * (point_b - point_a)
    normal = point_a - position
    # |normal| < 1e-12, decided like the reference's per-contact
    # np.linalg.norm; only rows within rounding of the threshold need it
    n2 = np.einsum("ij,ij->i", normal.astype(np.float64), normal.astype(np.float64))
    small = n2 < 1e-24
    near = np.nonzero(np.abs(n2 - 1e-24) <= 1e-30)[0]
    for k in near:
        small[k] = np.linalg.norm(normal[k]) < 1e-12
    normal[small] = 0.0
    return position, normal


def _triangles(soup) -> np.ndarray:
    t = soup.triangles() if hasattr(soup, "triangles") else soup
    return np.ascontiguousarray(np.asarray(t, dtype=K.REAL).reshape(-1, 3, 3))


def _same(soup_i, soup_j, ti, tj) -> bool:
    if soup_i is soup_j:
        return True
    return ti.shape == tj.shape and np.array_equal(ti, tj)


def _device_block(ti, tj, same, eps_pair, params):
    """All pairs of one block on the device: (ii, jj, point_a, point_b, stats)."""
    import torch

    from . import particles as PT
    from .device import Params, new_stats, read_stats

    dev = torch.device("cuda")
    ni, nj = ti.shape[0], tj.shape[0]
    T = max(ni, nj)
    meshes = np.zeros((1 if same else 2, T, 3, 3), K.REAL)
    meshes[0, :ni] = ti
    if not same:
        meshes[1, :nj] = tj
    counts = np.array([ni] if same else [ni, nj], np.int32)
    blocks = torch.tensor([[0, 0] if same else [0, 1]], dtype=torch.int32, device=dev)
    p = params or K.KernelParams()
    P = Params(epsilon=p.epsilon, n_iterative=p.n_iterative, c_factor=p.c_factor,
               alpha_iterative=p.alpha_iterative, alpha_regulariser=p.alpha_regulariser,
               move_factor=p.move_factor, start_coord=p.start_coord)
    st = new_stats(dev)
    cap = ni * nj
    out = PT.blocks_hybrid(torch.from_numpy(meshes).to(dev), blocks, P,
                           block_eps=torch.tensor([eps_pair], dtype=torch.from_numpy(meshes).dtype, device=dev),
                           mesh_tris=counts, strict=K.rounding() == "strict", max_contacts=max(cap, 1), stats=st)
    res = PT.sort_contacts(out)
    return res["idx"][:, 1], res["idx"][:, 2], res["point_a"], res["point_b"], read_stats(st)


def find_contacts_single_level(soup_i, soup_j, params: K.KernelParams | None = None,
                               counters: K.KernelCounters | None = None, pair=(0, 1), eps_i: float | None = None,
                               eps_j: float | None = None, chunk: int = 262144) -> list[ContactPoint]:
    """RK/contact.py:97-140: all-pairs hybrid detection between two soups;
    the same soup twice skips the diagonal; output ordered by (i, j)."""
    params = params or K.KernelParams()
    eps_i = params.epsilon if eps_i is None else eps_i
    eps_j = params.epsilon if eps_j is None else eps_j
    ti, tj = _triangles(soup_i), _triangles(soup_j)
    ni, nj = ti.shape[0], tj.shape[0]
    if ni == 0 or nj == 0:
        return []
    same = _same(soup_i, soup_j, ti, tj)
    eps_pair = 0.5 * (eps_i + eps_j)
    if max(ni, nj) <= _STAGE_LIMIT[np.dtype(K.REAL)]:
        ii, jj, pa, pb, st = _device_block(ti, tj, same, eps_pair, params)
        if st["degenerate"]:
            raise K.DegenerateTriangle("degenerate triangle in comparison fallback")
        if counters is not None:
            counters.iterative_invocations += st["iterative"]
            counters.comparison_invocations += st["comparison"]
            counters.fallback_invocations += st["fallback"]
    else:
        ii, jj = np.meshgrid(np.arange(ni), np.arange(nj), indexing="ij")
        ii, jj = ii.ravel(), jj.ravel()
        if same:
            keep = ii != jj
            ii, jj = ii[keep], jj[keep]
        hits_i, hits_j, pas, pbs = [], [], [], []
        for start in range(0, ii.size, chunk):
            si, sj = ii[start:start + chunk], jj[start:start + chunk]
            res = K.hybrid_batch(ti[si], tj[sj], params, counters, eps_pair)
            hit = np.nonzero(res.kind == np.int8(K.Kind.CONTACT))[0]
            hits_i.append(si[hit])
            hits_j.append(sj[hit])
            pas.append(res.point_a[hit])
            pbs.append(res.point_b[hit])
        ii, jj = np.concatenate(hits_i), np.concatenate(hits_j)
        pa, pb = np.concatenate(pas), np.concatenate(pbs)
    if ii.size == 0:
        return []
    position, normal = contact_from_segment_batch(pa, pb, eps_i, eps_j)
    return [ContactPoint(position[k], normal[k], tuple(pair), (int(ii[k]), int(jj[k])), (0, 0), (eps_i, eps_j))
            for k in range(ii.size)]


__all__ = ["ContactPoint", "contact_from_segment", "contact_from_segment_batch", "find_contacts_single_level"]
