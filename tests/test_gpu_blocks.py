"""All-pairs particle blocks (cfg2): tc_blocks_hybrid against the oracle
(strict: bitwise) and against the flat hybrid kernel on the materialised
pairs (fast: the same arithmetic, bitwise)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2105_12415_b200 import device as D  # noqa: E402
from paper_2105_12415_b200 import particles as PT  # noqa: E402


@pytest.fixture(scope="module")
def scene():
    meshes, blocks, gaps = PT.cfg2_scene(grid=(4, 4, 2))
    return meshes, blocks, gaps


def _contacts_from_flat(kind, dist, pa, pb, which, T):
    rows = np.nonzero(kind == 1)[0]
    blk = np.asarray(which)[rows // (T * T)]
    i = (rows % (T * T)) // T
    j = rows % T
    idx = np.stack([blk, i, j], 1).astype(np.int32)
    order = np.lexsort((idx[:, 2], idx[:, 1], idx[:, 0]))
    return idx[order], dist[rows][order], pa[rows][order], pb[rows][order]


@pytest.mark.parametrize("pkw", [dict(), dict(n_iterative=16, epsilon=1e-6), dict(epsilon=5e-2),
                                 dict(n_iterative=16, epsilon=4e-2)])
def test_blocks_strict_bitwise_vs_oracle(oracle_lib, scene, pkw):
    meshes, blocks, gaps = scene
    which = [int(np.argmin(gaps)), 0, 7]
    T = meshes.shape[1]
    st = D.new_stats()
    out = PT.blocks_hybrid(torch.from_numpy(meshes).cuda(), torch.from_numpy(blocks[which]).cuda(),
                           D.Params(**pkw), strict=True, stats=st)
    torch.cuda.synchronize()
    got = PT.sort_contacts(out)
    # block ids in the device result are positions in `which`
    A, B = PT.block_pairs(meshes, blocks, which)
    p = oracle_lib.make_params(**pkw)
    ref, counts, rc = oracle_lib.hybrid(A, B, p, p.epsilon, threads=oracle_lib.default_threads())
    assert rc == 0
    idx, dist, pa, pb = _contacts_from_flat(ref["kind"], ref["distance"], ref["point_a"], ref["point_b"],
                                            range(len(which)), T)
    assert got["n_contacts"] == len(idx)
    if pkw.get("epsilon", 1e-2) >= 4e-2:
        assert len(idx) > 0   # the facets of icosphere(2) sit ~0.07 apart at the closest blocks
    assert np.array_equal(got["idx"], idx)
    assert np.array_equal(got["distance"], dist)
    assert np.array_equal(got["point_a"], pa) and np.array_equal(got["point_b"], pb)
    s = D.read_stats(st)
    assert [s["iterative"], s["comparison"], s["fallback"]] == list(counts[:3])
    assert s["contacts"] == len(idx)
    assert s["min_distance"] == float(ref["distance"].min())


def test_blocks_fast_equals_flat_fast(scene):
    meshes, blocks, gaps = scene
    which = [int(b) for b in np.argsort(gaps)[:12]]
    T = meshes.shape[1]
    pk = dict(epsilon=5e-2)
    st = D.new_stats()
    out = PT.blocks_hybrid(torch.from_numpy(meshes).cuda(), torch.from_numpy(blocks[which]).cuda(),
                           D.Params(**pk), strict=False, stats=st)
    A, B = PT.block_pairs(meshes, blocks, which)
    st2 = D.new_stats()
    flat = D.run("hybrid", torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda(), D.Params(**pk), stats=st2)
    torch.cuda.synchronize()
    got = PT.sort_contacts(out)
    idx, dist, pa, pb = _contacts_from_flat(flat["kind"].cpu().numpy(), flat["distance"].cpu().numpy(),
                                            flat["point_a"].cpu().numpy(), flat["point_b"].cpu().numpy(),
                                            range(len(which)), T)
    assert got["n_contacts"] == len(idx) > 0
    assert np.array_equal(got["idx"], idx) and np.array_equal(got["distance"], dist)
    s1, s2 = D.read_stats(st), D.read_stats(st2)
    for k in ("iterative", "comparison", "fallback", "contacts", "intersecting", "min_distance"):
        assert s1[k] == s2[k], k


def test_blocks_contact_capacity_and_empty(scene):
    meshes, blocks, gaps = scene
    which = np.argsort(gaps)[:4]
    out = PT.blocks_hybrid(torch.from_numpy(meshes).cuda(), torch.from_numpy(blocks[which]).cuda(),
                           D.Params(epsilon=6e-2), max_contacts=3)
    torch.cuda.synchronize()
    n = int(out["n_contacts"].item())
    assert n > 3                                       # all counted ...
    with pytest.raises(RuntimeError):                  # ... never a truncated, slot-order dependent subset
        PT.sort_contacts(out)
    full = PT.blocks_hybrid(torch.from_numpy(meshes).cuda(), torch.from_numpy(blocks[which]).cuda(),
                            D.Params(epsilon=6e-2), max_contacts=n)
    assert PT.sort_contacts(full)["idx"].shape == (n, 3)
    empty = PT.blocks_hybrid(torch.from_numpy(meshes).cuda(), torch.zeros((0, 2), dtype=torch.int32).cuda(),
                             D.Params())
    assert int(empty["n_contacts"].item()) == 0


@pytest.mark.parametrize("strict", [True, False])
def test_blocks_fused_rigid_motion(oracle_lib, strict):
    """Local-space meshes + per-particle rigid motions, transformed while the
    meshes are staged, equal the world-space run."""
    local, motions, blocks, gaps = PT.cfg2_scene_local(grid=(4, 4, 2))
    # RK/geometry.py:173-176 apply_points, as the oracle restates NumPy's matmul rounding
    world = np.stack([oracle_lib.apply_motion(local[k], motions[k, :4], motions[k, 4:]) for k in range(local.shape[0])])
    which = [int(b) for b in np.argsort(gaps)[:3]]
    pk = dict(epsilon=5e-2)
    st1, st2 = D.new_stats(), D.new_stats()
    fused = PT.blocks_hybrid(torch.from_numpy(local).cuda(), torch.from_numpy(blocks[which]).cuda(), D.Params(**pk),
                             motions=torch.from_numpy(motions).cuda(), strict=strict, stats=st1)
    plain = PT.blocks_hybrid(torch.from_numpy(world).cuda(), torch.from_numpy(blocks[which]).cuda(), D.Params(**pk),
                             strict=strict, stats=st2)
    torch.cuda.synchronize()
    a, b = PT.sort_contacts(fused), PT.sort_contacts(plain)
    assert a["n_contacts"] == b["n_contacts"] > 0
    assert np.array_equal(a["idx"], b["idx"])
    # the fused transform rounds exactly like the reference's apply_points in both policies
    for k in ("distance", "point_a", "point_b"):
        assert np.array_equal(a[k], b[k]), k
    assert D.read_stats(st1) == D.read_stats(st2)
    if strict:
        A, B = PT.block_pairs(world, blocks, which)
        p = oracle_lib.make_params(**pk)
        ref, _, _ = oracle_lib.hybrid(A, B, p, p.epsilon, threads=oracle_lib.default_threads())
        assert a["n_contacts"] == int((ref["kind"] == 1).sum())


@pytest.mark.parametrize("strict", [True, False])
def test_blocks_degenerate_screen(oracle_lib, scene, strict):
    """Degenerate triangles among the open (fallback) pairs of a block are
    counted, never compared or emitted (RK/kernels.py:596-600); the screen
    runs in the fallback batches.  Strict: counts equal the oracle's."""
    meshes, blocks, gaps = scene
    which = [int(np.argmin(gaps))]
    a_mesh = int(blocks[which[0], 0])
    bad = meshes.copy()
    tri = bad[a_mesh]
    sel = np.arange(0, tri.shape[0], 5)
    tri[sel, 2] = tri[sel, 0] + 0.5 * (tri[sel, 1] - tri[sel, 0])   # collinear: zero area
    pkw = dict(n_iterative=4, epsilon=5e-2)   # halo wide enough for open pairs
    st = D.new_stats()
    out = PT.blocks_hybrid(torch.from_numpy(bad).cuda(), torch.from_numpy(blocks[which]).cuda(),
                           D.Params(**pkw), strict=strict, stats=st)
    torch.cuda.synchronize()
    got = PT.sort_contacts(out)
    s = D.read_stats(st)
    A, B = PT.block_pairs(bad, blocks, which)
    p = oracle_lib.make_params(**pkw)
    ref, counts, rc = oracle_lib.hybrid(A, B, p, p.epsilon, threads=oracle_lib.default_threads())
    assert counts[3] > 0 and rc != 0          # the oracle marks them (and would raise)
    assert s["degenerate"] > 0
    if strict:
        T = bad.shape[1]
        idx, dist, _, _ = _contacts_from_flat(ref["kind"], ref["distance"], ref["point_a"], ref["point_b"],
                                              range(len(which)), T)
        assert [s["iterative"], s["comparison"], s["fallback"], s["degenerate"]] == list(counts[:4])
        assert np.array_equal(got["idx"], idx) and np.array_equal(got["distance"], dist)


# ---------------------------------------------------------------------------
# BASELINE.json config 2 at its full size (16 x 16 x 8 particles of 320
# triangles, 5,632 neighbour blocks, 576.7M triangle pairs) through
# size-independent properties; tools/parity_cfg2.py compares every pair with
# the oracle (profiles/r02_parity_cfg2.txt, two CPU-minutes) and stays a tool.
# ---------------------------------------------------------------------------

@pytest.fixture(scope="module")
def cfg2_full():
    meshes, blocks, gaps = PT.cfg2_scene()
    return meshes, blocks, gaps, torch.from_numpy(meshes).cuda()


@pytest.mark.slow
@pytest.mark.parametrize("strict", [True, False])
def test_cfg2_full_size_whole_equals_block_groups(cfg2_full, strict):
    """One launch over all blocks == the launches over 8 contiguous groups of blocks:
    summed counters, minimum distance and the (block, i, j)-ordered contact list, bit for bit."""
    meshes, blocks, gaps, dmesh = cfg2_full
    nb, T = blocks.shape[0], meshes.shape[1]
    assert nb * T * T == 576_716_800
    p = D.Params(n_iterative=16, epsilon=5e-2)
    st = D.new_stats()
    whole = PT.sort_contacts(PT.blocks_hybrid(dmesh, torch.from_numpy(blocks).cuda(), p, strict=strict, stats=st))
    ws = D.read_stats(st)
    assert ws["iterative"] == nb * T * T and ws["fallback"] == ws["comparison"] and ws["degenerate"] == 0
    assert whole["n_contacts"] == ws["contacts"] > 10_000
    assert ws["min_distance"] == float(whole["distance"].min())
    assert np.all(whole["distance"] <= 2 * 5e-2)
    parts, pstats = [], []
    edges = np.linspace(0, nb, 9).astype(int)
    for lo, hi in zip(edges[:-1], edges[1:]):
        s = D.new_stats()
        got = PT.sort_contacts(PT.blocks_hybrid(dmesh, torch.from_numpy(blocks[lo:hi]).cuda(), p, strict=strict,
                                                stats=s))
        got["idx"][:, 0] += lo
        parts.append(got)
        pstats.append(D.read_stats(s))
    for k in ("iterative", "comparison", "fallback", "degenerate", "contacts", "intersecting"):
        assert ws[k] == sum(s[k] for s in pstats), k
    assert ws["min_distance"] == min(s["min_distance"] for s in pstats)
    for k in ("idx", "distance", "point_a", "point_b"):
        assert np.array_equal(whole[k], np.concatenate([q[k] for q in parts])), k


@pytest.mark.slow
def test_cfg2_full_size_sampled_blocks_bitwise(oracle_lib, cfg2_full):
    """Blocks sampled from the whole list (the ones with the most contacts among them): the
    strict contacts of the full-scene launch, restricted to them, equal the oracle's."""
    meshes, blocks, gaps, dmesh = cfg2_full
    nb, T = blocks.shape[0], meshes.shape[1]
    pkw = dict(n_iterative=16, epsilon=5e-2)
    whole = PT.sort_contacts(PT.blocks_hybrid(dmesh, torch.from_numpy(blocks).cuda(), D.Params(**pkw), strict=True))
    rng = np.random.default_rng(2)
    # the three blocks with the most contacts, the first and last block, five random ones
    blk, cnt = np.unique(whole["idx"][:, 0], return_counts=True)
    busiest = blk[np.argsort(cnt)[-3:]]
    which = sorted({*map(int, busiest), 0, nb - 1, *map(int, rng.integers(0, nb, 5))})
    A, B = PT.block_pairs(meshes, blocks, which)
    po = oracle_lib.make_params(**pkw)
    ref, _, rc = oracle_lib.hybrid(A, B, po, po.epsilon, threads=oracle_lib.default_threads())
    assert rc == 0
    idx, dist, pa, pb = _contacts_from_flat(ref["kind"], ref["distance"], ref["point_a"], ref["point_b"], which, T)
    sel = np.isin(whole["idx"][:, 0], which)
    assert sel.sum() == len(idx) > 0
    assert np.array_equal(whole["idx"][sel], idx)
    assert np.array_equal(whole["distance"][sel], dist)
    assert np.array_equal(whole["point_a"][sel], pa) and np.array_equal(whole["point_b"][sel], pb)
