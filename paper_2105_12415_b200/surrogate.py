"""Surrogate halo checks on the point-triangle kernel.

Mirrors the point-triangle consumers of the reference's
``tricontact.surrogate`` (RK/surrogate.py): ``conservative_epsilon``
(:237-257) and ``validate_conservative`` (:463-505), with every
point-to-triangle distance computed by ``tc_point_triangle_distance_*``
(strict IEEE, bit-identical to ``closest_point_triangle_batch`` + the
reference's norm).  ``validate_conservative`` gathers the sample points and
conservative-halo vertices of every node of the tree into ONE launch (the
reference loops over nodes with one small batch each) and reduces per node
on the host in the reference's order.  Tree construction and fitting stay
with the reference (offline).

``tree`` arguments are duck-typed like the reference's SurrogateTree:
``nodes()``, ``finest_epsilon``; nodes with ``triangle``, ``epsilon``,
``is_leaf``, ``children`` and ``leaf_indices()``.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _abi
from . import kernels as K


class EmptyInput(ValueError):
    """RK/surrogate.py:27."""


def point_triangle_distance(points, tris, tri_index=None, stream=None):
    """Device distance of every point to its triangle (torch CUDA tensors):
    points (n, 3), tris (m, 3, 3), tri_index (n,) int32 or None (tris[i])."""
    import torch

    from .device import _DT, _p

    if points.dtype not in _DT or not points.is_cuda:
        raise ValueError("points must be a CUDA float64/float32 tensor")
    points = points.contiguous()
    tris = tris.to(points.dtype).contiguous()
    n = int(points.shape[0])
    if tri_index is not None:
        tri_index = tri_index.to(device=points.device, dtype=torch.int32).contiguous()
    dist = torch.empty(n, dtype=points.dtype, device=points.device)
    st = stream if stream is not None else torch.cuda.current_stream(points.device)
    fn = getattr(_abi.load(), f"tc_point_triangle_distance_{_DT[points.dtype]}")
    _abi.check(fn(_p(points), _p(tris), int(tris.shape[0]), _p(tri_index), n, _p(dist), None,
                  ctypes.c_void_p(st.cuda_stream)), "tc_point_triangle_distance")
    return dist


def _distances(points: np.ndarray, tris: np.ndarray, tri_index: np.ndarray) -> np.ndarray:
    """Host arrays in, host distances out (one launch)."""
    import torch

    if points.shape[0] == 0:
        return np.empty(0, K.REAL)
    dev = torch.device("cuda")
    d = point_triangle_distance(torch.from_numpy(np.ascontiguousarray(points, K.REAL)).to(dev),
                                torch.from_numpy(np.ascontiguousarray(tris, K.REAL)).to(dev),
                                torch.from_numpy(np.ascontiguousarray(tri_index, np.int32)).to(dev))
    return d.cpu().numpy()


def _child_eps(children: np.ndarray, child_epsilons) -> np.ndarray:
    eps = np.asarray(child_epsilons, dtype=K.REAL)
    if eps.ndim == 0:
        eps = np.full(children.shape[0], float(eps), dtype=K.REAL)
    return eps


def conservative_epsilon(surrogate: np.ndarray, children: np.ndarray, child_epsilons) -> float:
    """RK/surrogate.py:237-257: max over child vertices of dist(v, surrogate) + eps_child."""
    children = K.as_triangles(children)
    if children.shape[0] == 0:
        raise EmptyInput("no child triangles")
    surrogate = np.asarray(surrogate, dtype=K.REAL).reshape(1, 3, 3)
    eps = _child_eps(children, child_epsilons)
    pts = children.reshape(-1, 3)
    dist = _distances(pts, surrogate, np.zeros(pts.shape[0], np.int32)).reshape(-1, 3)
    return float((dist + eps[:, None]).max())


def _bary_samples(count: int) -> np.ndarray:
    """RK/surrogate.py:450-458: corners, edges and interior rows."""
    rows = max(int(np.ceil((np.sqrt(8.0 * count + 1.0) - 1.0) / 2.0)) + 1, 2)
    return np.asarray([(i / (rows - 1), j / (rows - 1)) for i in range(rows) for j in range(rows - i)],
                      dtype=K.REAL)


def validate_conservative(tree, triangles: np.ndarray, samples_per_triangle: int = 10) -> dict:
    """RK/surrogate.py:463-505: sampled descendant surface points (padded by
    the finest halo) inside every node's halo, and the chain condition over
    each node's immediate children.  Returns {"ok", "worst_slack", "checked_nodes"}."""
    triangles = K.as_triangles(triangles)
    bary = _bary_samples(samples_per_triangle)
    nodes = list(tree.nodes())
    surr = np.stack([np.asarray(nd.triangle, K.REAL).reshape(3, 3) for nd in nodes]).astype(K.REAL)
    pts_all, idx_all, plan = [], [], []
    off = 0
    for k, nd in enumerate(nodes):
        tris = triangles[nd.leaf_indices()]
        v0 = tris[:, 0]
        e1 = tris[:, 1] - tris[:, 0]
        e2 = tris[:, 2] - tris[:, 0]
        pts = (v0[:, None, :] + bary[None, :, 0, None] * e1[:, None, :]
               + bary[None, :, 1, None] * e2[:, None, :]).reshape(-1, 3)
        if nd.is_leaf:
            ch, ch_eps = tris, _child_eps(tris, tree.finest_epsilon)
        else:
            ch = np.stack([c.triangle for c in nd.children]).astype(K.REAL)
            ch_eps = _child_eps(ch, [c.epsilon for c in nd.children])
        if ch.shape[0] == 0:
            raise EmptyInput("no child triangles")
        vtx = ch.reshape(-1, 3)
        pts_all += [pts, vtx]
        idx_all.append(np.full(pts.shape[0] + vtx.shape[0], k, np.int32))
        plan.append((off, pts.shape[0], vtx.shape[0], ch_eps))
        off += pts.shape[0] + vtx.shape[0]
    dist = _distances(np.concatenate(pts_all), surr, np.concatenate(idx_all))
    worst = np.inf
    for nd, (o, n_s, n_v, ch_eps) in zip(nodes, plan):
        slack = nd.epsilon - (dist[o:o + n_s] + tree.finest_epsilon)
        worst = min(worst, float(slack.min()))
        need = float((dist[o + n_s:o + n_s + n_v].reshape(-1, 3) + ch_eps[:, None]).max())
        worst = min(worst, float(nd.epsilon - need))
    return {"ok": worst >= -1e-6, "worst_slack": worst, "checked_nodes": len(nodes)}
