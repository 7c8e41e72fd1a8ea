"""BASELINE.json config 4 at its full size (2^28 pairs, reduce-only hybrid),
checked inside the GPU suite through size-independent properties:

* one launch over all 2^28 pairs and the 16 contiguous shards of a 16-way
  split (each regenerated independently by the counter-based device generator,
  as ``bench.py`` ranks do) give the same summed counters and the same minimum
  distance -- strict and fast builds (no data-path collective, one
  SUM/MIN of the stats record);
* the invariants of the hybrid's counters (RK/kernels.py:568-605);
* windows drawn from the whole index range (including the last pairs, whose
  plane offsets pass 2^31 elements): the strict build's full records and ids
  are bit-identical to the oracle's, and the window's counters equal its.

tools/parity_cfg4.py compares the counters of all 2^28 pairs with the oracle's
(profiles/r02_parity_cfg4.txt); that takes the CPU two minutes and stays a tool.
"""

import ctypes

import numpy as np
import pytest

from conftest import PARAM_SETS

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2105_12415_b200 import _abi  # noqa: E402
from paper_2105_12415_b200 import device as D  # noqa: E402

N = 1 << 28
SHARDS = 16
SEP = (-0.05, 0.2)
COUNTERS = ("iterative", "comparison", "fallback", "degenerate", "contacts", "intersecting")


def _generate(start, n):
    planes = torch.empty((18, n), dtype=torch.float64, device="cuda")
    lib = _abi.load()
    _abi.check(lib.tc_random_pairs_soa_f64(4, start, n, SEP[0], SEP[1], ctypes.c_void_p(planes.data_ptr()), None),
               "tc_random_pairs_soa_f64")
    return planes


@pytest.fixture(scope="module")
def cfg4():
    free, _ = torch.cuda.mem_get_info()
    if free < 60 << 30:
        pytest.skip("cfg4 at full size needs 39 GB of inputs plus shard copies")
    planes = _generate(0, N)
    torch.cuda.synchronize()
    yield planes
    del planes
    torch.cuda.empty_cache()


def _reduce_only(planes, n, strict):
    st = D.new_stats()
    D.run("hybrid", planes[:9], planes[9:], D.Params(**PARAM_SETS["bl"]), soa=True, strict=strict, out={},
          stats=st, n=n)
    torch.cuda.synchronize()
    return D.read_stats(st)


@pytest.mark.slow
@pytest.mark.parametrize("strict", [True, False])
def test_cfg4_whole_equals_sum_of_shards(cfg4, strict):
    whole = _reduce_only(cfg4, N, strict)
    assert whole["iterative"] == N
    assert whole["fallback"] == whole["comparison"]
    assert whole["degenerate"] == 0
    assert whole["intersecting"] <= whole["contacts"] <= N
    assert 0.3 < whole["fallback"] / N < 0.6     # BASELINE.json config 4: ~43 % fallbacks
    parts = []
    for r in range(SHARDS):
        lo, hi = r * N // SHARDS, (r + 1) * N // SHARDS
        shard = _generate(lo, hi - lo)
        if r in (0, SHARDS - 1):  # any shard is generated independently of the others
            assert torch.equal(shard, cfg4[:, lo:hi])
        parts.append(_reduce_only(shard, hi - lo, strict))
        del shard
    for k in COUNTERS:
        assert whole[k] == sum(p[k] for p in parts), k
    assert whole["min_distance"] == min(p["min_distance"] for p in parts)


@pytest.mark.slow
def test_cfg4_windows_strict_bitwise(oracle_lib, cfg4):
    w = 1 << 14
    rng = np.random.default_rng(4)
    starts = [0, N - w] + [int(s) for s in rng.integers(0, N - w, 4)]
    p = D.Params(**PARAM_SETS["bl"])
    po = oracle_lib.make_params(**PARAM_SETS["bl"])
    for lo in starts:
        win = cfg4[:, lo:lo + w]
        host = win.cpu().numpy()
        A = np.ascontiguousarray(host[:9].T).reshape(w, 3, 3)
        B = np.ascontiguousarray(host[9:].T).reshape(w, 3, 3)
        sub = win.contiguous()
        st = D.new_stats()
        out = D.run("hybrid", sub[:9], sub[9:], p, soa=True, strict=True, ids=True, stats=st, n=w)
        torch.cuda.synchronize()
        ref, counts, rc = oracle_lib.hybrid(A, B, po, PARAM_SETS["bl"]["epsilon"])
        assert rc == 0
        got = {k: v.cpu().numpy() for k, v in out.items()}
        for k in ("point_a", "point_b", "bary_a", "bary_b"):
            got[k] = got[k].T
        for k in ("kind", "distance", "point_a", "point_b", "bary_a", "bary_b", "ids"):
            assert np.array_equal(got[k], ref[k]), (lo, k)
        s = D.read_stats(st)
        assert [s["iterative"], s["comparison"], s["fallback"], s["degenerate"]] == list(counts[:4]), lo
        assert s["contacts"] == int((ref["kind"] == 1).sum())


@pytest.mark.slow
def test_cfg4_tail_of_the_single_launch(oracle_lib, cfg4):
    """The last pairs of the one 2^28-pair launch (element offsets beyond 2^31): full
    records of a strict launch over the whole batch, compared on its tail."""
    w = 1 << 12
    p = D.Params(**PARAM_SETS["bl"])
    out = {"kind": torch.empty(N, dtype=torch.int8, device="cuda"),
           "distance": torch.empty(N, dtype=torch.float64, device="cuda")}
    res = D.run("hybrid", cfg4[:9], cfg4[9:], p, soa=True, strict=True, out=out, n=N)
    torch.cuda.synchronize()
    host = cfg4[:, N - w:].cpu().numpy()
    A = np.ascontiguousarray(host[:9].T).reshape(w, 3, 3)
    B = np.ascontiguousarray(host[9:].T).reshape(w, 3, 3)
    ref, _, rc = oracle_lib.hybrid(A, B, oracle_lib.make_params(**PARAM_SETS["bl"]), PARAM_SETS["bl"]["epsilon"])
    assert rc == 0
    assert np.array_equal(res["kind"][N - w:].cpu().numpy(), ref["kind"])
    assert np.array_equal(res["distance"][N - w:].cpu().numpy(), ref["distance"])
