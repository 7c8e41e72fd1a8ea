"""Surrogate halo checks on the point-triangle kernel
against the reference's own conservative_epsilon / validate_conservative
outputs (tests/golden/ms_float*.npz, RK/surrogate.py:237-257, 463-505)."""

from dataclasses import dataclass, field

import numpy as np
import pytest
import torch

from conftest import DTYPES
from ms_common import load

from paper_2105_12415_b200 import kernels as K
from paper_2105_12415_b200 import surrogate as S

pytestmark = pytest.mark.gpu


@dataclass
class _Node:
    triangle: np.ndarray
    epsilon: float
    is_leaf: bool
    payload: np.ndarray
    children: list = field(default_factory=list)

    def leaf_indices(self):
        if self.is_leaf:
            return self.payload
        return np.concatenate([c.leaf_indices() for c in self.children])


@dataclass
class _Tree:
    nodes_: list
    finest_epsilon: float

    def nodes(self):
        return iter(self.nodes_)


def _tree(g, pre, real):
    dt = DTYPES[real]
    n = g[f"{pre}_node_eps"].shape[0]
    ko, kk = g[f"{pre}_kids_off"], g[f"{pre}_kids"]
    lo, ll = g[f"{pre}_leafidx_off"], g[f"{pre}_leafidx"]
    nodes = [_Node(g[f"{pre}_node_tri"][k].astype(dt), float(g[f"{pre}_node_eps"][k]), bool(g[f"{pre}_node_leaf"][k]),
                   ll[lo[k]:lo[k + 1]]) for k in range(n)]
    for k in range(n):
        nodes[k].children = [nodes[c] for c in kk[ko[k]:ko[k + 1]]]
    return _Tree(nodes, float(g[f"{pre}_finest"]))


@pytest.mark.parametrize("real", list(DTYPES))
def test_validate_conservative_matches_reference(monkeypatch, real):
    monkeypatch.setattr(K, "REAL", DTYPES[real])
    g = load(real)
    for pre in ("sg80", "sg320"):
        tree = _tree(g, pre, real)
        mesh = g[f"{pre}_mesh"].reshape(-1, 3, 3)
        for spt in (10, 3):
            r = S.validate_conservative(tree, mesh, samples_per_triangle=spt)
            ref = g[f"{pre}_valid_{spt}"]
            assert r["worst_slack"] == ref[0] and r["ok"] == bool(ref[1]) and r["checked_nodes"] == ref[2], (pre, spt)
        tree.nodes_[0].epsilon *= 0.5
        r = S.validate_conservative(tree, mesh)
        ref = g[f"{pre}_halved_valid"]
        assert r["worst_slack"] == ref[0] and not r["ok"] and not ref[1]


@pytest.mark.parametrize("real", list(DTYPES))
def test_conservative_epsilon_matches_reference(monkeypatch, real):
    monkeypatch.setattr(K, "REAL", DTYPES[real])
    g = load(real)
    for k, ref in enumerate(g["ce_values"]):
        e = g[f"ce{k}_eps"]
        got = S.conservative_epsilon(g[f"ce{k}_surrogate"], g[f"ce{k}_children"].reshape(-1, 3, 3),
                                     float(e) if e.ndim == 0 else e)
        assert got == ref, k
    with pytest.raises(S.EmptyInput):
        S.conservative_epsilon(g["ce0_surrogate"], np.empty((0, 3, 3)), 0.0)


@pytest.mark.parametrize("dt", [np.float64, np.float32])
def test_point_triangle_distance_vs_oracle(oracle_lib, dt):
    rng = np.random.default_rng(4)
    n, m = 100_000, 777
    P = rng.normal(size=(n, 3)).astype(dt)
    T = rng.normal(size=(m, 3, 3)).astype(dt)
    idx = rng.integers(0, m, n).astype(np.int32)
    c, _ = oracle_lib.closest_point_triangle(P, T[idx], dtype=dt)
    ref = np.linalg.norm(P - c, axis=1)
    got = S.point_triangle_distance(torch.from_numpy(P).cuda(), torch.from_numpy(T).cuda(),
                                    torch.from_numpy(idx).cuda()).cpu().numpy()
    assert got.tobytes() == ref.astype(dt).tobytes()
