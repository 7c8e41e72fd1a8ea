"""The multiscale oracle (oracle/ms_oracle.py) against the reference's own
multiscale_contacts outputs (tests/golden/ms_float*.npz, RK/stepping.py:311-368)."""

import numpy as np
import pytest

from conftest import DTYPES
from ms_common import load, scenes, tree


@pytest.mark.parametrize("real", list(DTYPES))
def test_oracle_matches_reference_multiscale(oracle_lib, real):
    import ms_oracle

    g = load(real)
    dt = DTYPES[real]
    p = oracle_lib.make_params()
    for sc in scenes(g):
        trees = [tree(g, sc, "i"), tree(g, sc, "j")]
        o = ms_oracle.multiscale(trees, [(0, 1)], p, dtype=dt)
        assert o["rc"] == 0
        assert np.array_equal(o["source"], g[f"{sc}_source"]), sc
        assert o["position"].tobytes() == g[f"{sc}_position"].astype(dt).tobytes(), sc
        assert o["normal"].tobytes() == g[f"{sc}_normal"].astype(dt).tobytes(), sc
        assert np.array_equal(o["eps"], g[f"{sc}_eps"]), sc
        ref_checks = g[f"{sc}_checks"]
        assert np.array_equal(o["checks"][: ref_checks.size], ref_checks), sc
        assert not o["checks"][ref_checks.size:].any()
        assert np.array_equal(o["counts"][:3], g[f"{sc}_counters"]), sc


@pytest.mark.parametrize("real", list(DTYPES))
def test_golden_equivalence_lemma(real):
    # the reference's own multiscale and single-level contacts agree on every scene
    g = load(real)
    for sc in scenes(g):
        assert np.array_equal(g[f"{sc}_source"], g[f"{sc}_single_source"]), sc
    assert sum(g[f"{sc}_source"].shape[0] for sc in scenes(g)) > 50


@pytest.mark.parametrize("real", list(DTYPES))
def test_oracle_apply_motion_matches_reference(oracle_lib, real):
    # RK/geometry.py:173-176 apply_points (the reference's world_tris) == the
    # oracle's FMA-chain restatement, bitwise, on every golden particle
    g = load(real)
    dt = DTYPES[real]
    for sc in scenes(g):
        for side in ("i", "j"):
            m = g[f"{sc}_{side}_motion"]
            w = oracle_lib.apply_motion(g[f"{sc}_{side}_local"].reshape(-1, 3), m[:4], m[4:].astype(dt), dtype=dt)
            assert w.tobytes() == g[f"{sc}_{side}_tris"].astype(dt).reshape(-1, 3).tobytes(), (sc, side)
