"""CPU restatement of the reference's multiscale traversal -- TEST INFRASTRUCTURE.

Only tests/ (and bench.py's CPU legs) may call this.  It restates, per
particle pair and in the reference's own order:
  multiscale_contacts  -> RK/stepping.py:311-368 (frontier loop, halo
                          0.5 (eps_i + eps_j), fallback on mesh-level pairs
                          only, meshgrid unfolding, per-height check counts)
  contact_from_segment -> RK/contact.py:75-94
  _sorted_contacts     -> RK/stepping.py:281
on top of the C oracle's hybrid (oracle.py), with a tree given as plain
arrays (RK/stepping.py:78-129 FlatTree: tris (n_total, 3, 3), eps, CSR
children, height, n_nodes).  Pinned against tests/golden/ms_float*.npz,
which the reference itself produced (tests/golden/make_multiscale_golden.py).
"""

from __future__ import annotations

import numpy as np

import oracle


def _children(tree, k):
    return np.asarray(tree["child_ids"][tree["child_off"][k]:tree["child_off"][k + 1]], np.int64)


def contact_from_segment(point_a, point_b, eps_a: float, eps_b: float):
    """RK/contact.py:75-94 (no fallback direction): (position, normal)."""
    w = eps_a / (eps_a + eps_b)
    position = point_a + w * (point_b - point_a)
    normal = point_a - position
    if np.linalg.norm(normal) < 1e-12:
        normal = 0.0 * np.zeros(3, dtype=point_a.dtype)
    return position, normal


def multiscale_pair(ti, tj, params, dtype=np.float64, threads=1):
    """One particle pair: (contacts, checks {height: count}, counts[4], rc).

    contacts: list of (source_i, source_j, point_a, point_b, eps_i, eps_j)
    sorted by source."""
    ids_i = np.array([0], np.int64)
    ids_j = np.array([0], np.int64)
    checks: dict[int, int] = {}
    counts = np.zeros(4, np.int64)
    out = []
    while ids_i.size:
        A = np.asarray(ti["tris"], dtype).reshape(-1, 3, 3)[ids_i]
        B = np.asarray(tj["tris"], dtype).reshape(-1, 3, 3)[ids_j]
        eps_i = np.asarray(ti["eps"], dtype)[ids_i]
        eps_j = np.asarray(tj["eps"], dtype)[ids_j]
        fine_i = ids_i >= ti["n_nodes"]
        fine_j = ids_j >= tj["n_nodes"]
        both = fine_i & fine_j
        hgt = np.maximum(np.asarray(ti["height"])[ids_i], np.asarray(tj["height"])[ids_j])
        for lvl in np.unique(hgt):
            checks[int(lvl)] = checks.get(int(lvl), 0) + int((hgt == lvl).sum())
        res, c, rc = oracle.hybrid(A, B, params, (0.5 * (eps_i + eps_j)).astype(dtype), allow_fallback=both,
                                   dtype=dtype, threads=threads)
        counts += c
        if rc != 0:
            return out, checks, counts, rc
        kind = res["kind"]
        for h in np.nonzero(both & (kind == 1))[0]:
            out.append((int(ids_i[h] - ti["n_nodes"]), int(ids_j[h] - tj["n_nodes"]), res["point_a"][h],
                        res["point_b"][h], float(eps_i[h]), float(eps_j[h])))
        expand = np.nonzero(((kind == 1) | (kind == 2)) & ~both)[0]
        ni, nj = [], []
        for k in expand:
            ci = _children(ti, ids_i[k]) if not fine_i[k] else ids_i[k:k + 1]
            cj = _children(tj, ids_j[k]) if not fine_j[k] else ids_j[k:k + 1]
            gi, gj = np.meshgrid(ci, cj, indexing="ij")
            ni.append(gi.ravel())
            nj.append(gj.ravel())
        ids_i = np.concatenate(ni) if ni else np.empty(0, np.int64)
        ids_j = np.concatenate(nj) if nj else np.empty(0, np.int64)
    out.sort(key=lambda c: (c[0], c[1]))
    return out, checks, counts, 0


def multiscale(trees, pairs, params, dtype=np.float64, threads=1):
    """Every particle pair of ``pairs`` in order; returns dict of arrays:
    pair (n, 2), source (n, 2), point_a/b, position, normal (n, 3), eps (n, 2),
    checks (max_height + 1,), counts[4] (iterative, comparison, fallback, degenerate), rc."""
    rows = []
    checks: dict[int, int] = {}
    counts = np.zeros(4, np.int64)
    rc = 0
    for pi, pj in np.asarray(pairs, np.int64).reshape(-1, 2):
        cs, ch, c, rc = multiscale_pair(trees[pi], trees[pj], params, dtype, threads)
        counts += c
        for h, v in ch.items():
            checks[h] = checks.get(h, 0) + v
        for s_i, s_j, pa, pb, ea, eb in cs:
            pos, nrm = contact_from_segment(pa, pb, ea, eb)
            rows.append(((int(pi), int(pj)), (s_i, s_j), pa, pb, pos, nrm, (ea, eb)))
        if rc != 0:
            break
    rows.sort(key=lambda r: (r[0], r[1]))
    hmax = max(max(int(np.max(t["height"])) for t in trees), 0)
    n = len(rows)
    return dict(pair=np.array([r[0] for r in rows], np.int64).reshape(n, 2),
                source=np.array([r[1] for r in rows], np.int64).reshape(n, 2),
                point_a=np.array([r[2] for r in rows], dtype).reshape(n, 3),
                point_b=np.array([r[3] for r in rows], dtype).reshape(n, 3),
                position=np.array([r[4] for r in rows], dtype).reshape(n, 3),
                normal=np.array([r[5] for r in rows], dtype).reshape(n, 3),
                eps=np.array([r[6] for r in rows], np.float64).reshape(n, 2),
                checks=np.array([checks.get(h, 0) for h in range(hmax + 1)], np.int64), counts=counts, rc=rc)
