"""The tie-aware tolerance checker (tests/parity.py) on CPU.

The FMA-contracted build of the oracle (oracle/libtc_oracle_fma.so) stands
in for the GPU's fast build: it must pass, and corrupted results must fail.
"""

import numpy as np
import pytest

import parity
from conftest import DTYPES, PARAM_SETS


@pytest.fixture(scope="module")
def fma(oracle_lib):
    return oracle_lib.fma_variant()


def _run(O, variant, A, B, pkw, dt):
    p = O.make_params(**pkw)
    eps = np.full(len(A), p.epsilon, dt)
    if variant == "comparison":
        return O.comparison(A, B, eps, dt)
    if variant == "iterative":
        return O.iterative(A, B, p, eps, dt)
    return O.hybrid(A, B, p, eps, dtype=dt)[0]


@pytest.mark.parametrize("real", list(DTYPES))
@pytest.mark.parametrize("pname", list(PARAM_SETS))
@pytest.mark.parametrize("case", ["cfg0", "cfg3"])
@pytest.mark.parametrize("variant", ["comparison", "iterative", "hybrid"])
def test_fma_build_within_tolerance(oracle_lib, fma, golden_inputs, variant, case, pname, real):
    dt = DTYPES[real]
    A = golden_inputs[f"{case}_A"].astype(dt)
    B = golden_inputs[f"{case}_B"].astype(dt)
    got = _run(fma, variant, A, B, PARAM_SETS[pname], dt)
    rep = parity.compare_fast(oracle_lib, variant, A, B, PARAM_SETS[pname], got, dt)
    assert rep["ok"], str(rep)


def test_strict_oracle_against_itself_is_exact(oracle_lib, golden_inputs):
    A, B = golden_inputs["cfg0_A"], golden_inputs["cfg0_B"]
    got = _run(oracle_lib, "hybrid", A, B, PARAM_SETS["bl"], np.float64)
    rep = parity.compare_fast(oracle_lib, "hybrid", A, B, PARAM_SETS["bl"], got, np.float64)
    assert rep["ok"] and rep["excused"] == 0 and rep["distance_max_rel"] == 0.0


@pytest.mark.parametrize("col,delta", [("distance", 1e-7), ("point_a", 1e-6), ("bary_a", 1e-6), ("bary_b", 1e-6)])
def test_checker_rejects_corruption(oracle_lib, golden_inputs, col, delta):
    A, B = golden_inputs["cfg0_A"][:512], golden_inputs["cfg0_B"][:512]
    got = _run(oracle_lib, "hybrid", A, B, PARAM_SETS["def"], np.float64)
    got[col] = got[col] + delta
    assert not parity.compare_fast(oracle_lib, "hybrid", A, B, PARAM_SETS["def"], got, np.float64)["ok"]


def test_checker_rejects_flipped_kind(oracle_lib, golden_inputs):
    A, B = golden_inputs["cfg0_A"][:512], golden_inputs["cfg0_B"][:512]
    got = _run(oracle_lib, "comparison", A, B, PARAM_SETS["def"], np.float64)
    far = np.nonzero(got["distance"] > 0.1)[0][:3]
    got["kind"][far] = 1
    assert not parity.compare_fast(oracle_lib, "comparison", A, B, PARAM_SETS["def"], got, np.float64)["ok"]


def test_bary_err_is_in_point_units():
    """Weights along a sliver's two nearly parallel long edges are
    ill-conditioned; the checker judges them by the point they name
    (tests/parity.py bary_err): a weight change of 1e-4 that moves the point
    by 1e-10 passes at tau = 1e-9, one that moves it by 1e-4 does not."""
    T = np.array([[[0.0, 0, 0], [1.0, 0, 0], [0.5, 1e-6, 0]]])   # ab ~ 2 ac: height 5e-7
    ref = {"bary_a": np.array([[0.25, 0.5]]), "bary_b": np.array([[0.25, 0.5]])}
    L = parity.longest_edge(T, T)
    d = 1e-4
    along = {"bary_a": np.array([[0.25 - 0.5 * d, 0.5 + d]]), "bary_b": ref["bary_b"]}   # moves the point by 1e-10
    across = {"bary_a": np.array([[0.25 + d, 0.5]]), "bary_b": ref["bary_b"]}           # moves it by 1e-4
    assert parity.bary_err(T, T, along, ref, L)[0] < 1e-9
    assert parity.bary_err(T, T, across, ref, L)[0] > 1e-5
    assert np.allclose(parity.bary_point(T, ref["bary_a"]), [[0.5, 5e-7, 0.0]])
