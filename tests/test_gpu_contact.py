"""Contact emission against the reference's own
outputs (tests/golden/ms_float*.npz): find_contacts_single_level
(RK/contact.py:97-140: unequal halos, a soup against itself, ragged soups)
and single_level_contacts (RK/stepping.py:285-308) through the particle-block
kernel with the rigid motions fused into the staging."""

import numpy as np
import pytest
import torch

from conftest import DTYPES
from ms_common import load, scenes

from paper_2105_12415_b200 import contact as C
from paper_2105_12415_b200 import kernels as K
from paper_2105_12415_b200 import particles as PT

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("real", list(DTYPES))
def test_find_contacts_single_level_bitwise(monkeypatch, real):
    monkeypatch.setattr(K, "REAL", DTYPES[real])
    dt = DTYPES[real]
    g = load(real)
    for case in [str(c) for c in g["fc_cases"]]:
        pre = f"fc_{case}"
        ti = g[f"{pre}_tris_i"].reshape(-1, 3, 3)
        tj = ti if bool(g[f"{pre}_same"]) else g[f"{pre}_tris_j"].reshape(-1, 3, 3)
        ei, ej = (None if np.isnan(e) else float(e) for e in g[f"{pre}_eps"])
        counters = K.KernelCounters()
        got = C.find_contacts_single_level(ti, tj, K.KernelParams(), counters, pair=(3, 7), eps_i=ei, eps_j=ej)
        src = np.array([c.source for c in got], np.int64).reshape(-1, 2)
        assert np.array_equal(src, g[f"{pre}_source"]), case
        pos = np.array([c.position for c in got], dt).reshape(-1, 3)
        nrm = np.array([c.normal for c in got], dt).reshape(-1, 3)
        assert pos.tobytes() == g[f"{pre}_position"].astype(dt).tobytes(), case
        assert nrm.tobytes() == g[f"{pre}_normal"].astype(dt).tobytes(), case
        assert all(c.pair == (3, 7) for c in got)
        c = g[f"{pre}_counters"]
        assert (counters.iterative_invocations, counters.comparison_invocations,
                counters.fallback_invocations) == tuple(c), case
        if case == "self":
            assert all(s0 != s1 for s0, s1 in src)


@pytest.mark.parametrize("real", list(DTYPES))
def test_single_level_fused_motion_bitwise(real):
    # every golden two-particle scene: local mesh triangles + (quaternion,
    # translation) per particle, one block, transform fused into the staging
    dt = DTYPES[real]
    tdt = torch.float64 if dt == np.float64 else torch.float32
    g = load(real)
    for sc in scenes(g):
        loc, mot, cnt = [], [], []
        for side in ("i", "j"):
            n_nodes = int(g[f"{sc}_{side}_n_nodes"])
            loc.append(g[f"{sc}_{side}_local"][n_nodes:].reshape(-1, 3, 3))
            mot.append(g[f"{sc}_{side}_motion"])
            cnt.append(loc[-1].shape[0])
        T = max(cnt)
        meshes = np.zeros((2, T, 3, 3), dt)
        for k in range(2):
            meshes[k, :cnt[k]] = loc[k]
        eps_i, eps_j = (float(e) for e in g[f"{sc}_single_eps"])
        out = PT.blocks_hybrid(torch.from_numpy(meshes).cuda(), torch.tensor([[0, 1]], dtype=torch.int32).cuda(),
                               K.KernelParams(), motions=torch.tensor(np.stack(mot), dtype=tdt).cuda(),
                               block_eps=torch.tensor([0.5 * (eps_i + eps_j)], dtype=tdt).cuda(),
                               mesh_tris=np.array(cnt, np.int32), strict=True)
        res = PT.sort_contacts(out)
        pos, nrm = C.contact_from_segment_batch(res["point_a"], res["point_b"], eps_i, eps_j)
        assert np.array_equal(res["idx"][:, 1:], g[f"{sc}_single_source"]), sc
        assert pos.tobytes() == g[f"{sc}_single_position"].astype(dt).tobytes(), sc
        assert nrm.tobytes() == g[f"{sc}_single_normal"].astype(dt).tobytes(), sc


def test_ragged_and_self_blocks_counts():
    # pair counts of ragged and self blocks: n_a * n_b, and n (n - 1) on the diagonal block
    from paper_2105_12415_b200 import device as D
    rng = np.random.default_rng(0)
    meshes = rng.uniform(0, 1, (3, 50, 3, 3))
    cnt = np.array([50, 17, 33], np.int32)
    blocks = torch.tensor([[0, 1], [1, 2], [2, 2], [1, 1]], dtype=torch.int32).cuda()
    st = D.new_stats()
    PT.blocks_hybrid(torch.from_numpy(meshes).cuda(), blocks, D.Params(), mesh_tris=cnt, stats=st)
    s = D.read_stats(st)
    assert s["iterative"] == 50 * 17 + 17 * 33 + 33 * 32 + 17 * 16


@pytest.mark.parametrize("same", [False, True])
def test_find_contacts_chunked_path_equals_block_path(monkeypatch, same):
    # soups beyond the shared-memory staging limit go through kernels.hybrid_batch
    # in chunks (like the reference); both paths must give the same contacts
    g = load("float64")
    ti = g["fc_two_tris_i"].reshape(-1, 3, 3)
    tj = ti if same else g["fc_two_tris_j"].reshape(-1, 3, 3)
    c1 = K.KernelCounters()
    block = C.find_contacts_single_level(ti, tj, K.KernelParams(), c1)
    monkeypatch.setitem(C._STAGE_LIMIT, np.dtype(np.float64), 8)
    c2 = K.KernelCounters()
    chunked = C.find_contacts_single_level(ti, tj, K.KernelParams(), c2, chunk=1000)
    assert [c.source for c in block] == [c.source for c in chunked]
    assert all(a.position.tobytes() == b.position.tobytes() for a, b in zip(block, chunked))
    assert c1.as_dict() == c2.as_dict()
    if same:
        assert all(s0 != s1 for s0, s1 in (c.source for c in chunked))


def test_find_contacts_empty_soup():
    assert C.find_contacts_single_level(np.zeros((0, 3, 3)), np.ones((3, 3, 3))) == []
