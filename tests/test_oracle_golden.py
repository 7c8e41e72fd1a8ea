"""The CPU oracle (oracle/tc_oracle.c) is bit-identical to the reference.

Fixtures come from the reference itself (tests/golden/make_golden.py).
Equality is IEEE ``==`` per element (so +0 == -0), exact for kind, ids and
counters.
"""

import numpy as np
import pytest

from conftest import DTYPES, PARAM_SETS

COLS = ("kind", "distance", "point_a", "point_b", "bary_a", "bary_b")


def _assert_cols(ref, pre, got):
    for col in COLS:
        r = ref[f"{pre}_{col}"]
        g = got[col]
        assert r.shape == g.shape, (pre, col)
        neq = ~((r == g) | (np.isnan(r) & np.isnan(g)))
        assert not neq.any(), f"{pre}.{col}: {int(neq.sum())} elements differ, first rows {np.nonzero(neq)[0][:5]}"


@pytest.mark.parametrize("real", list(DTYPES))
@pytest.mark.parametrize("pname", list(PARAM_SETS))
@pytest.mark.parametrize("case", ["cfg0", "cfg3", "special"])
def test_oracle_matches_reference(oracle_lib, golden_inputs, golden_ref, real, pname, case):
    O = oracle_lib
    dt = DTYPES[real]
    ref = golden_ref[real]
    A = golden_inputs[f"{case}_A"].astype(dt)
    B = golden_inputs[f"{case}_B"].astype(dt)
    p = O.make_params(**PARAM_SETS[pname])
    eps = np.full(len(A), p.epsilon, dt)
    pre = f"{case}_{pname}"
    cm = O.comparison(A, B, eps, dt)
    _assert_cols(ref, f"{pre}_comparison", cm)
    assert np.array_equal(ref[f"{pre}_comparison_ids"], cm["ids"])
    _assert_cols(ref, f"{pre}_iterative", O.iterative(A, B, p, eps, dt))
    hy, counts, rc = O.hybrid(A, B, p, eps, dtype=dt)
    if f"{pre}_hybrid_raised" in ref:
        assert rc == 2
    else:
        assert rc == 0
        _assert_cols(ref, f"{pre}_hybrid", hy)
        assert np.array_equal(ref[f"{pre}_hybrid_counters"], counts[:3])


@pytest.mark.parametrize("real", list(DTYPES))
def test_oracle_masked_hybrid(oracle_lib, golden_inputs, golden_ref, real):
    """Per-pair eps + allow_fallback mask (RK/kernels.py:589-593)."""
    O = oracle_lib
    dt = DTYPES[real]
    ref = golden_ref[real]
    A = golden_inputs["cfg0_A"][:1024].astype(dt)
    B = golden_inputs["cfg0_B"][:1024].astype(dt)
    eps = golden_inputs["mask_eps"].astype(dt)
    hy, counts, rc = O.hybrid(A, B, O.make_params(), eps, golden_inputs["mask_allow"], dtype=dt)
    assert rc == 0
    _assert_cols(ref, "masked_hybrid", hy)
    assert np.array_equal(ref["masked_hybrid_counters"], counts[:3])


@pytest.mark.parametrize("real", list(DTYPES))
def test_oracle_point_triangle_and_degenerate(oracle_lib, golden_inputs, golden_ref, real):
    O = oracle_lib
    dt = DTYPES[real]
    ref = golden_ref[real]
    cl, ba = O.closest_point_triangle(golden_inputs["cpt_P"], golden_inputs["cpt_T"], dt)
    assert np.array_equal(cl, ref["cpt_closest"])
    assert np.array_equal(ba, ref["cpt_bary"])
    m = O.degenerate(golden_inputs["degenerate_T"], dt)
    assert np.array_equal(m, ref["degenerate_mask"])
    assert m.any() and not m.all()


def test_oracle_threads_invariant(oracle_lib, golden_inputs):
    """Tiling invariance (SPEC: results equal the element-wise map for any tiling)."""
    O = oracle_lib
    A = np.concatenate([golden_inputs["cfg0_A"]] * 3)
    B = np.concatenate([golden_inputs["cfg0_B"]] * 3)
    p = O.make_params(n_iterative=16, epsilon=1e-6)
    eps = np.full(len(A), 1e-6)
    h1, c1, _ = O.hybrid(A, B, p, eps, threads=1)
    h8, c8, _ = O.hybrid(A, B, p, eps, threads=7)
    for k in h1:
        assert np.array_equal(h1[k], h8[k])
    assert np.array_equal(c1, c8)


@pytest.mark.parametrize("real", list(DTYPES))
def test_oracle_degenerate_rel_tol(oracle_lib, golden_inputs, golden_r2, real):
    """degenerate_mask(T, rel_tol) at non-default tolerances (RK/geometry.py:68-75)."""
    ref = golden_r2[real]
    for i, tol in enumerate(ref["degtol_rel_tols"]):
        m = oracle_lib.degenerate(golden_inputs["degenerate_T"], DTYPES[real], rel_tol=float(tol))
        assert np.array_equal(m, ref[f"degtol_{i}"]), tol


def test_oracle_acceptance_criterion_1(oracle_lib, golden_r2):
    """The 10,000 scene-drawn pairs of RT/test_acceptance.py:69-87: the oracle's
    comparison (incl. ids) and hybrid are bit-identical to the reference's."""
    O = oracle_lib
    ref = golden_r2["float64"]
    A, B = ref["crit1_A"], ref["crit1_B"]
    p = O.make_params()
    eps = np.full(len(A), p.epsilon)
    cm = O.comparison(A, B, eps, threads=O.default_threads())
    _assert_cols(ref, "crit1_comparison", cm)
    assert np.array_equal(ref["crit1_comparison_ids"], cm["ids"])
    hy, counts, rc = O.hybrid(A, B, p, eps, threads=O.default_threads())
    assert rc == 0
    _assert_cols(ref, "crit1_hybrid", hy)
