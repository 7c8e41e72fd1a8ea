"""Device multiscale traversal (tc_multiscale_*) against
the reference's multiscale_contacts (tests/golden/ms_float*.npz) and the
multiscale oracle (oracle/ms_oracle.py) on batched, re-posed scenes."""

import numpy as np
import pytest

from conftest import DTYPES
from ms_common import load, moved, scenes, tree

pytestmark = pytest.mark.gpu


def _run(trees, pairs, dt, strict=True, max_contacts=1 << 16):
    from paper_2105_12415_b200 import kernels, multiscale as ms

    arrs = [ms.FlatTreeArrays(t["tris"].reshape(-1, 3, 3), t["eps"], t["child_off"], t["child_ids"], t["height"],
                              t["n_nodes"]) for t in trees]
    forest = ms.build_forest(arrs, dtype=dt)
    res = ms.multiscale_contacts(forest, pairs, kernels.KernelParams(), strict=strict, max_contacts=max_contacts)
    return res, ms.contact_points(forest, res, pairs)


@pytest.mark.parametrize("real", list(DTYPES))
def test_reference_scenes_bitwise(real):
    g = load(real)
    dt = DTYPES[real]
    for sc in scenes(g):
        res, cp = _run([tree(g, sc, "i"), tree(g, sc, "j")], [(0, 1)], dt)
        assert res.n_contacts == g[f"{sc}_source"].shape[0], sc
        assert np.array_equal(cp["source"], g[f"{sc}_source"]), sc
        assert cp["position"].tobytes() == g[f"{sc}_position"].astype(dt).tobytes(), sc
        assert cp["normal"].tobytes() == g[f"{sc}_normal"].astype(dt).tobytes(), sc
        assert np.array_equal(cp["eps"], g[f"{sc}_eps"]), sc
        ref = g[f"{sc}_checks"]
        assert np.array_equal(res.checks[: ref.size], ref), sc
        assert not res.checks[ref.size:].any()
        c = g[f"{sc}_counters"]
        assert (res.stats["iterative"], res.stats["comparison"], res.stats["fallback"]) == tuple(c), sc


def _batched_scene(g, dt, poses, seed):
    """Every golden scene re-posed `poses` times (one extra rigid motion applied
    to both particles), all trees in one forest, pair k = (2k, 2k+1)."""
    rng = np.random.default_rng(seed)
    trees = []
    for sc in scenes(g):
        ti, tj = tree(g, sc, "i"), tree(g, sc, "j")
        for _ in range(poses):
            q = rng.normal(size=4)
            q /= np.linalg.norm(q)
            w, x, y, z = q
            R = np.array([[1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)],
                          [2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)],
                          [2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)]])
            shift = rng.uniform(-3, 3, 3)
            trees += [moved(ti, R, shift), moved(tj, R, shift)]
    pairs = np.arange(len(trees)).reshape(-1, 2)
    return trees, pairs


@pytest.mark.parametrize("real", list(DTYPES))
def test_batched_reposed_vs_oracle_bitwise(oracle_lib, real):
    import ms_oracle

    g = load(real)
    dt = DTYPES[real]
    trees, pairs = _batched_scene(g, dt, poses=6, seed=7)
    # add cross pairs that share particles with the main ones
    pairs = np.concatenate([pairs, pairs[:: 3, ::-1]])
    res, cp = _run(trees, pairs, dt)
    o = ms_oracle.multiscale(trees, pairs, oracle_lib.make_params(), dtype=dt)
    assert o["rc"] == 0
    assert o["source"].shape[0] > 100
    assert np.array_equal(cp["pair"], o["pair"])
    assert np.array_equal(cp["source"], o["source"])
    assert cp["position"].tobytes() == o["position"].tobytes()
    assert cp["normal"].tobytes() == o["normal"].tobytes()
    assert np.array_equal(res.checks[: o["checks"].size], o["checks"])
    assert (res.stats["iterative"], res.stats["comparison"], res.stats["fallback"]) == tuple(o["counts"][:3])


def _replay_fast(oracle_lib, trees, pairs, dt):
    """RK/stepping.py:311-368 replayed round by round in Python over the fast
    device hybrid (device entry point, per-pair halos 0.5 (eps_i + eps_j),
    fallback only where both sides are mesh triangles).  Every round's results
    go through the tie-aware checker against the oracle on the same pairings
    (tests/parity.py: kinds / paths / ids equal except at ties within the
    north-star tolerance, values within it).  Returns the mesh-level contacts
    {(pair, src_i, src_j): (point_a, point_b)} and the per-round reports."""
    import torch
    import parity
    from paper_2105_12415_b200 import device as D

    tt = {np.float64: torch.float64, np.float32: torch.float32}[dt]
    front = [(k, 0, 0) for k in range(len(pairs))]
    contacts, reports = {}, []
    while front:
        f = np.array(front, np.int64)
        ti = [trees[pairs[k][0]] for k in f[:, 0]]
        tj = [trees[pairs[k][1]] for k in f[:, 0]]
        A = np.stack([t["tris"].reshape(-1, 3, 3)[i] for t, i in zip(ti, f[:, 1])]).astype(dt)
        B = np.stack([t["tris"].reshape(-1, 3, 3)[j] for t, j in zip(tj, f[:, 2])]).astype(dt)
        ei = np.array([t["eps"][i] for t, i in zip(ti, f[:, 1])], dt)
        ej = np.array([t["eps"][j] for t, j in zip(tj, f[:, 2])], dt)
        halo = (dt(0.5) * (ei + ej)).astype(dt)
        fine_i = np.array([i >= t["n_nodes"] for t, i in zip(ti, f[:, 1])])
        fine_j = np.array([j >= t["n_nodes"] for t, j in zip(tj, f[:, 2])])
        both = fine_i & fine_j
        out = D.run("hybrid", torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda(), D.Params(),
                    eps=torch.from_numpy(halo).cuda(), allow=torch.from_numpy(both.astype(np.uint8)).cuda(),
                    strict=False, ids=True)
        got = {k: v.cpu().numpy() for k, v in out.items()}
        # (measured excused rates: 0.013 % fp64, 0.043 % fp32)
        rep = parity.compare_fast(oracle_lib, "hybrid", A, B, {}, got, dt, eps=halo, allow=both,
                                  max_excused=1e-3 if dt == np.float64 else 5e-3)
        reports.append(rep)
        nxt = []
        for r, (k, i, j) in enumerate(front):
            kd = got["kind"][r]
            if both[r]:
                if kd == 1:
                    contacts[(k, i - ti[r]["n_nodes"], j - tj[r]["n_nodes"])] = (got["point_a"][r], got["point_b"][r])
                continue
            if kd in (1, 2):
                ci = [i] if fine_i[r] else list(ti[r]["child_ids"][ti[r]["child_off"][i]:ti[r]["child_off"][i + 1]])
                cj = [j] if fine_j[r] else list(tj[r]["child_ids"][tj[r]["child_off"][j]:tj[r]["child_off"][j + 1]])
                nxt += [(k, a, b) for a in ci for b in cj]
        front = nxt
    return contacts, reports


@pytest.mark.parametrize("real", list(DTYPES))
def test_fast_traversal_tie_aware(oracle_lib, real):
    """Fast (FMA-contracted) traversal: every decision of every round checked
    against the oracle with the tie classifier (no contact-set slack), and the
    fused device traversal equal, bit for bit, to the round-by-round replay
    over the device hybrid."""
    g = load(real)
    dt = DTYPES[real]
    trees, pairs = _batched_scene(g, dt, poses=3, seed=11)
    contacts, reports = _replay_fast(oracle_lib, trees, [tuple(p) for p in pairs], dt)
    for rep in reports:
        assert rep["ok"], rep
    assert sum(r["n"] for r in reports) > 1000 and len(contacts) > 50
    res, cp = _run(trees, pairs, dt, strict=False)
    got = {(int(np.nonzero((pairs == p).all(1))[0][0]), int(s[0]), int(s[1])): n
           for n, (p, s) in enumerate(zip(cp["pair"], cp["source"]))}
    assert set(got) == set(contacts)
    order = [got[k] for k in contacts]
    pa = np.array([contacts[k][0] for k in contacts])
    pb = np.array([contacts[k][1] for k in contacts])
    assert np.array_equal(np.sort(order), np.arange(len(order)))
    keys = list(contacts)
    # positions from the replay's points, rounded like contact_points
    from paper_2105_12415_b200.contact import contact_from_segment_batch
    ea = np.array([cp["eps"][got[k]][0] for k in keys])
    eb = np.array([cp["eps"][got[k]][1] for k in keys])
    pos, nrm = contact_from_segment_batch(pa, pb, ea, eb)
    assert pos.astype(dt).tobytes() == cp["position"][order].tobytes()
    assert nrm.astype(dt).tobytes() == cp["normal"][order].tobytes()


def test_capacity_and_empty():
    g = load("float64")
    sc = "s320_rest"
    trees = [tree(g, sc, "i"), tree(g, sc, "j")]
    res, _ = _run(trees, np.zeros((0, 2), np.int64), np.float64)
    assert res.n_contacts == 0 and not res.checks.any()
    # a contact list sized below the count is re-run with room for every
    # contact: never a truncated (atomic-order dependent) subset
    res, cp = _run(trees, [(0, 1)], np.float64, max_contacts=3)
    assert res.n_contacts == g[f"{sc}_source"].shape[0] == res.pair.size
    assert np.array_equal(cp["source"], g[f"{sc}_source"])


@pytest.mark.parametrize("real", list(DTYPES))
def test_fused_motion_matches_reference(real):
    # local node coordinates + per-particle rigid motions, transformed as the
    # frontier loads them (8f row 2), reproduce the reference's world-space run
    from paper_2105_12415_b200 import kernels, multiscale as ms

    g = load(real)
    dt = DTYPES[real]
    trees, motions, pairs, scs = [], [], [], []
    for sc in scenes(g):
        for side in ("i", "j"):
            t = tree(g, sc, side)
            trees.append(ms.FlatTreeArrays(g[f"{sc}_{side}_local"].reshape(-1, 3, 3), t["eps"], t["child_off"],
                                           t["child_ids"], t["height"], t["n_nodes"]))
            motions.append(g[f"{sc}_{side}_motion"])
        pairs.append((len(trees) - 2, len(trees) - 1))
        scs.append(sc)
    forest = ms.build_forest(trees, dtype=dt, motions=np.stack(motions))
    for strict in (True, False):
        res = ms.multiscale_contacts(forest, pairs, kernels.KernelParams(), strict=strict)
        cp = ms.contact_points(forest, res, pairs)
        for k, sc in enumerate(scs):
            sel = cp["pair"][:, 0] == pairs[k][0]
            if strict:
                assert np.array_equal(cp["source"][sel], g[f"{sc}_source"]), sc
                assert cp["position"][sel].tobytes() == g[f"{sc}_position"].astype(dt).tobytes(), sc
                assert cp["normal"][sel].tobytes() == g[f"{sc}_normal"].astype(dt).tobytes(), sc
        if not strict:
            # fused fast == world-space fast, bitwise (the transform rounds like the reference)
            wt = [tree(g, sc, side) for sc in scs for side in ("i", "j")]
            res_w, cp_w = _run(wt, pairs, dt, strict=False)
            assert np.array_equal(cp["source"], cp_w["source"])
            assert cp["position"].tobytes() == cp_w["position"].tobytes()


def test_degenerate_mesh_triangle_raises():
    # a mesh-level fallback pair with a degenerate triangle: the reference
    # raises DegenerateTriangle (RK/kernels.py:598-600); the traversal returns
    # TC_EDEGENERATE, which the wrapper raises
    from paper_2105_12415_b200 import kernels

    g = load("float64")
    sc = "s80_rest"
    ti, tj = tree(g, sc, "i"), tree(g, sc, "j")
    tris = ti["tris"].reshape(-1, 3, 3).copy()
    # collapse every mesh triangle of particle i onto a line
    fine = np.arange(ti["n_nodes"], tris.shape[0])
    tris[fine, 2] = tris[fine, 0] + 2.0 * (tris[fine, 1] - tris[fine, 0])
    ti = dict(ti, tris=tris.reshape(-1, 9))
    with pytest.raises(kernels.DegenerateTriangle):
        _run([ti, tj], [(0, 1)], np.float64)
