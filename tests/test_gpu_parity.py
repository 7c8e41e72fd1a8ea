"""GPU parity: the sm_100a kernels against the reference's golden vectors and
the CPU oracle, through the C ABI.

* TC_STRICT (device entry points and the drop-in host path): bit-identical
  to the reference -- every column, kind, ids and counters.
* fast (FMA-contracted) build: within the north-star tolerance
  |x - x_ref| <= tau * max(|x_ref|, L), tau = 1e-9 (fp64) / 1e-4 (fp32),
  L = the pair's longest edge, with kind mismatches allowed only at ties
  (tests/parity.py).
"""

import numpy as np
import pytest

from conftest import DTYPES, PARAM_SETS

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2105_12415_b200 import device as D  # noqa: E402
from paper_2105_12415_b200 import workloads as W  # noqa: E402

import parity  # noqa: E402

COLS = ("kind", "distance", "point_a", "point_b", "bary_a", "bary_b")
TDT = {"float64": torch.float64, "float32": torch.float32}


def run_dev(variant, A, B, real, pname, strict, soa=False, eps=None, allow=None, ids=True):
    dt = TDT[real]
    p = D.Params(**PARAM_SETS[pname])
    if soa:
        planes = torch.from_numpy(W.to_soa(A, B)).to("cuda", dt)
        ta, tb = planes[:9].contiguous(), planes[9:].contiguous()
    else:
        ta = torch.from_numpy(np.ascontiguousarray(A)).to("cuda", dt)
        tb = torch.from_numpy(np.ascontiguousarray(B)).to("cuda", dt)
    stats = D.new_stats()
    e = None if eps is None else torch.from_numpy(np.asarray(eps)).to("cuda", dt)
    al = None if allow is None else torch.from_numpy(np.asarray(allow, np.uint8)).cuda()
    out = D.run(variant, ta, tb, p, eps=e, allow=al, soa=soa, strict=strict, ids=ids, stats=stats)
    torch.cuda.synchronize()
    res = {k: v.cpu().numpy() for k, v in out.items()}
    if soa:
        for k in ("point_a", "point_b", "bary_a", "bary_b"):
            res[k] = np.ascontiguousarray(res[k].T)
    return res, D.read_stats(stats)


def assert_bitwise(ref, pre, got):
    for col in COLS:
        r = ref[f"{pre}_{col}"]
        g = got[col]
        neq = ~((r == g) | (np.isnan(r) & np.isnan(g)))
        assert not neq.any(), f"{pre}.{col}: {int(neq.sum())} differ, rows {np.nonzero(neq)[0][:8]}"


@pytest.mark.parametrize("soa", [False, True])
@pytest.mark.parametrize("real", list(DTYPES))
@pytest.mark.parametrize("pname", list(PARAM_SETS))
@pytest.mark.parametrize("case", ["cfg0", "cfg3", "special"])
def test_strict_bitwise_vs_reference(golden_inputs, golden_ref, case, pname, real, soa):
    ref = golden_ref[real]
    dt = DTYPES[real]
    A = golden_inputs[f"{case}_A"].astype(dt)
    B = golden_inputs[f"{case}_B"].astype(dt)
    pre = f"{case}_{pname}"
    cm, st = run_dev("comparison", A, B, real, pname, True, soa)
    assert_bitwise(ref, f"{pre}_comparison", cm)
    assert np.array_equal(cm["ids"], ref[f"{pre}_comparison_ids"])
    assert st["comparison"] == len(A) and st["fallback"] == 0
    it, st = run_dev("iterative", A, B, real, pname, True, soa)
    assert_bitwise(ref, f"{pre}_iterative", it)
    assert st["iterative"] == len(A)
    hy, st = run_dev("hybrid", A, B, real, pname, True, soa)
    if f"{pre}_hybrid_raised" in ref:
        assert st["degenerate"] > 0
    else:
        assert_bitwise(ref, f"{pre}_hybrid", hy)
        assert [st["iterative"], st["comparison"], st["fallback"]] == list(ref[f"{pre}_hybrid_counters"])
        assert st["contacts"] == int((hy["kind"] == 1).sum())
        assert st["min_distance"] == float(hy["distance"].min())


@pytest.mark.parametrize("real", list(DTYPES))
def test_strict_masked_hybrid(golden_inputs, golden_ref, real):
    dt = DTYPES[real]
    A = golden_inputs["cfg0_A"][:1024].astype(dt)
    B = golden_inputs["cfg0_B"][:1024].astype(dt)
    hy, st = run_dev("hybrid", A, B, real, "def", True, eps=golden_inputs["mask_eps"].astype(dt),
                     allow=golden_inputs["mask_allow"])
    assert_bitwise(golden_ref[real], "masked_hybrid", hy)
    assert [st["iterative"], st["comparison"], st["fallback"]] == list(golden_ref[real]["masked_hybrid_counters"])


@pytest.mark.parametrize("real", list(DTYPES))
def test_point_triangle_and_degenerate(golden_inputs, golden_ref, real):
    dt = TDT[real]
    P = torch.from_numpy(golden_inputs["cpt_P"]).to("cuda", dt)
    T = torch.from_numpy(golden_inputs["cpt_T"]).to("cuda", dt)
    cl, ba = D.closest_point_triangle(P, T)
    assert np.array_equal(cl.cpu().numpy(), golden_ref[real]["cpt_closest"])
    assert np.array_equal(ba.cpu().numpy(), golden_ref[real]["cpt_bary"])
    m = D.degenerate_mask(torch.from_numpy(golden_inputs["degenerate_T"]).to("cuda", dt))
    assert np.array_equal(m.cpu().numpy(), golden_ref[real]["degenerate_mask"])


@pytest.mark.parametrize("real", list(DTYPES))
@pytest.mark.parametrize("pname", list(PARAM_SETS))
@pytest.mark.parametrize("case", ["cfg0", "cfg3"])
def test_fast_within_tolerance(oracle_lib, golden_inputs, case, pname, real):
    dt = DTYPES[real]
    A = golden_inputs[f"{case}_A"].astype(dt)
    B = golden_inputs[f"{case}_B"].astype(dt)
    for variant in ("comparison", "iterative", "hybrid"):
        got, _ = run_dev(variant, A, B, real, pname, False)
        rep = parity.compare_fast(oracle_lib, variant, A, B, PARAM_SETS[pname], got, dt)
        assert rep["ok"], str(rep)


@pytest.mark.parametrize("n", [1, 31, 255, 256, 257, 4097])
def test_ragged_sizes_strict(oracle_lib, golden_inputs, n):
    A = golden_inputs["cfg0_A"][:n]
    B = golden_inputs["cfg0_B"][:n]
    p = PARAM_SETS["bl"]
    hy, st = run_dev("hybrid", A, B, "float64", "bl", True)
    o, counts, _ = oracle_lib.hybrid(A, B, oracle_lib.make_params(**p), p["epsilon"])
    for col in COLS:
        assert np.array_equal(hy[col], o[col]), col
    assert np.array_equal(hy["ids"], o["ids"])
    assert [st["iterative"], st["comparison"], st["fallback"]] == list(counts[:3])


def test_empty_batch():
    t = torch.empty((0, 3, 3), dtype=torch.float64, device="cuda")
    out = D.run("hybrid", t, t, D.Params())
    assert out["kind"].numel() == 0


def test_degenerate_fallback_marks_pairs():
    """RK/kernels.py:598-600: degenerate triangles only matter on fallback."""
    U = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0]], float)
    bad = np.array([[0, 0, 0], [1, 0, 0], [2, 0, 0]], float)
    # NOT_TERMINATED after the default 4 sweeps against `bad` (oracle-checked
    # below), so this pair reaches the fallback and its screen
    open_b = np.array([[0.206, 0.02, 0.383], [-0.516, -0.114, -0.337], [0.419, 0.028, -0.205]])
    far = U + [0, 0, 1.0]
    A = np.stack([bad, bad, U])
    B = np.stack([far, open_b, far])
    hy, st = run_dev("hybrid", A, B, "float64", "def", True)
    assert hy["kind"][0] == 0                     # settled: never consults the comparison kernel
    assert hy["kind"][2] == 0
    assert hy["kind"][1] == 3 and st["degenerate"] == 1 and st["fallback"] == 0
    assert (hy["ids"][1, 3] & 8) > 0
    assert not (hy["kind"] == 2).any()


# ---------------------------------------------------------------------------
# BASELINE.json config 1 scale (2^24 pairs): size-independent properties,
# sampled bit-exact parity, and the fast build against the oracle on 2^20
# pairs with the tie classifier.
# ---------------------------------------------------------------------------

@pytest.fixture(scope="module")
def cfg1():
    A, B = W.random_pairs(1 << 24, seed=0, sep=(-0.1, 0.5))
    planes = torch.from_numpy(W.to_soa(A, B)).cuda()
    return A, B, planes


@pytest.mark.slow
def test_cfg1_strict_sampled_bitwise_and_stats(oracle_lib, cfg1):
    A, B, planes = cfg1
    n = A.shape[0]
    p = D.Params(**PARAM_SETS["bl"])
    stats = D.new_stats()
    out = D.run("hybrid", planes[:9], planes[9:], p, soa=True, strict=True, ids=True, stats=stats, n=n)
    torch.cuda.synchronize()
    st = D.read_stats(stats)
    kind = out["kind"].cpu().numpy()
    ids = out["ids"].cpu().numpy()
    dist = out["distance"].cpu().numpy()
    # size-independent properties of the hybrid (RK/kernels.py:568-605)
    assert not (kind == 2).any()
    assert st["iterative"] == n
    assert st["fallback"] == st["comparison"] == int(((ids[:, 3] & 4) > 0).sum())
    assert st["contacts"] == int((kind == 1).sum())
    assert st["intersecting"] == int(((ids[:, 3] & 16) > 0).sum())
    assert st["min_distance"] == float(dist.min())
    assert np.all(dist[(ids[:, 3] & 16) > 0] == 0)   # proper crossings report distance 0
    # bit-exact on a random sample against the oracle
    rng = np.random.default_rng(7)
    idx = np.sort(rng.choice(n, 20000, replace=False))
    ref, _, rc = oracle_lib.hybrid(A[idx], B[idx], oracle_lib.make_params(**PARAM_SETS["bl"]), 1e-6)
    assert rc == 0
    cols = {"distance": dist, "kind": kind}
    for k in ("point_a", "point_b", "bary_a", "bary_b"):
        cols[k] = out[k].cpu().numpy().T
    for k, v in cols.items():
        assert np.array_equal(v[idx], ref[k]), k
    assert np.array_equal(ids[idx], ref["ids"])


@pytest.mark.slow
@pytest.mark.parametrize("strict", [True, False])
def test_cfg1_shard_invariance(cfg1, strict):
    """Contiguous shards give bit-identical results and summed stats."""
    A, B, planes = cfg1
    n = A.shape[0]
    p = D.Params(**PARAM_SETS["bl"])
    whole = D.new_stats()
    full = D.run("hybrid", planes[:9].contiguous(), planes[9:].contiguous(), p, soa=True, strict=strict,
                 stats=whole, n=n)
    parts = []
    part_stats = []
    for w in range(4):
        lo, hi = w * n // 4, (w + 1) * n // 4
        sub = planes[:, lo:hi].contiguous()
        s = D.new_stats()
        parts.append(D.run("hybrid", sub[:9], sub[9:], p, soa=True, strict=strict, stats=s, n=hi - lo))
        part_stats.append(D.read_stats(s))
    torch.cuda.synchronize()
    for k in ("kind", "distance"):
        assert torch.equal(full[k], torch.cat([q[k] for q in parts], dim=-1)), k
    for k in ("point_a", "bary_b"):
        assert torch.equal(full[k], torch.cat([q[k] for q in parts], dim=1)), k
    ws = D.read_stats(whole)
    for k in ("iterative", "comparison", "fallback", "contacts", "intersecting"):
        assert ws[k] == sum(s[k] for s in part_stats), k
    assert ws["min_distance"] == min(s["min_distance"] for s in part_stats)


@pytest.mark.slow
@pytest.mark.parametrize("real", list(DTYPES))
def test_fast_vs_oracle_one_million(oracle_lib, real):
    """The fast build on 2^20 fresh pairs (chunks 256..511 of cfg1) within tolerance."""
    dt = DTYPES[real]
    A, B = W.random_pairs(1 << 20, seed=0, sep=(-0.1, 0.5), start=1 << 20)
    A = A.astype(dt)
    B = B.astype(dt)
    got, _ = run_dev("hybrid", A, B, real, "bl", False)
    # excused-tie budget ~2x the measured rate (fp64: 0 of 2^20, fp32: 0.29 %)
    rep = parity.compare_fast(oracle_lib, "hybrid", A, B, PARAM_SETS["bl"], got, dt,
                              max_excused=1e-4 if dt == np.float64 else 6e-3)
    assert rep["ok"], str(rep)


# ---------------------------------------------------------------------------
# start_coord outside [0, 1] (KernelParams allows any value): the fast build
# then runs the general clips (no box shortcut) and the full penalty; strict
# stays bit-identical.
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("start", [-0.25, 0.0, 1.0, 1.5])
@pytest.mark.parametrize("real", list(DTYPES))
def test_start_coord_general(oracle_lib, real, start):
    dt = DTYPES[real]
    A, B = W.random_pairs(1 << 13, seed=0, sep=(-0.1, 0.5), start=1 << 16)
    A = A.astype(dt)
    B = B.astype(dt)
    pk = dict(n_iterative=16, epsilon=1e-6, start_coord=start)
    ta, tb = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    ref, counts, rc = oracle_lib.hybrid(A, B, oracle_lib.make_params(**pk), pk["epsilon"], dtype=dt)
    assert rc == 0
    for variant in ("iterative", "hybrid"):
        strict = D.run(variant, ta, tb, D.Params(**pk), strict=True, ids=True)
        fast = D.run(variant, ta, tb, D.Params(**pk), strict=False, ids=True)
        torch.cuda.synchronize()
        got = {k: v.cpu().numpy() for k, v in fast.items()}
        rep = parity.compare_fast(oracle_lib, variant, A, B, pk, got, dt)
        assert rep["ok"], (variant, str(rep))
        if variant == "hybrid":
            for k in COLS:
                assert np.array_equal(strict[k].cpu().numpy(), ref[k]), k


@pytest.mark.parametrize("soa", [False, True])
@pytest.mark.parametrize("real", list(DTYPES))
def test_degenerate_screen_random(oracle_lib, real, soa):
    """Degenerate triangles injected into random pairs, with a per-pair
    fallback mask and per-pair halos: the fallback batches screen them
    (kind 3, DEGENERATE flag, counted, not compared) exactly like the
    oracle's hybrid (strict: bitwise incl. ids and counters)."""
    dt = DTYPES[real]
    A, B = W.random_pairs(3 * 4096 + 5, seed=21, sep=(-0.1, 0.5))
    rng = np.random.default_rng(9)
    for T in (A, B):
        sel = rng.random(len(T)) < 0.05
        T[sel, 2] = T[sel, 0] + 0.25 * (T[sel, 1] - T[sel, 0])
    A = A.astype(dt)
    B = B.astype(dt)
    eps = rng.uniform(1e-7, 1e-5, len(A)).astype(dt)
    allow = (rng.random(len(A)) < 0.9).astype(np.uint8)
    pk = PARAM_SETS["bl"]
    got, st = run_dev("hybrid", A, B, real, "bl", True, soa=soa, eps=eps, allow=allow)
    ref, counts, rc = oracle_lib.hybrid(A, B, oracle_lib.make_params(**pk), eps, allow_fallback=allow, dtype=dt)
    assert rc != 0 and counts[3] > 0
    for k in COLS:
        assert np.array_equal(got[k], ref[k]), k
    assert np.array_equal(got["ids"], ref["ids"])
    assert [st["iterative"], st["comparison"], st["fallback"], st["degenerate"]] == list(counts[:4])
    fast, fst = run_dev("hybrid", A, B, real, "bl", False, soa=soa, eps=eps, allow=allow)
    assert fst["degenerate"] > 0
    assert np.all((fast["ids"][fast["kind"] == 3, 3] & 8) > 0)


@pytest.mark.parametrize("real", list(DTYPES))
@pytest.mark.parametrize("strict", [True, False])
def test_host_pipeline_equals_device(strict, real):
    """tc_run_host_f64 (pinned staging, 1M-pair chunks over 3 streams: the
    drop-in's path) gives the device entry point's results bit for bit on a
    batch of several chunks with a ragged tail, and the same counters."""
    import ctypes
    from paper_2105_12415_b200 import _abi
    n = (5 << 19) + 123   # 2.5 chunks of 2^20
    dt = DTYPES[real]
    A, B = W.random_pairs(n, seed=4, sep=(-0.1, 0.5))
    A, B = A.astype(dt), B.astype(dt)
    p = D.Params(**PARAM_SETS["bl"])
    st = D.new_stats()
    dev = D.run("hybrid", torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda(), p, strict=strict, stats=st)
    torch.cuda.synchronize()
    ds = D.read_stats(st)
    out = {"distance": np.empty(n, dt), "point_a": np.empty((n, 3), dt), "point_b": np.empty((n, 3), dt),
           "bary_a": np.empty((n, 2), dt), "bary_b": np.empty((n, 2), dt), "kind": np.empty(n, np.int8)}
    ptr = lambda a: a.ctypes.data_as(ctypes.c_void_p)
    hs = _abi.TcStats(0, 0, 0, 0, 0, 0, float("inf"))
    prm = _abi.params_struct(p, _abi.TC_STRICT if strict else 0)
    host = getattr(_abi.load(), "tc_run_host_f64" if real == "float64" else "tc_run_host_f32")
    rc = host(2, ptr(A), ptr(B), n, None, None, ctypes.byref(prm),
                                     *(ptr(out[k]) for k in ("distance", "point_a", "point_b", "bary_a", "bary_b")),
                                     ptr(out["kind"]), None, ctypes.byref(hs))
    assert rc == 0
    for k in out:
        assert np.array_equal(out[k], dev[k].cpu().numpy()), k
    assert [hs.iterative, hs.comparison, hs.fallback, hs.contacts] == \
        [ds["iterative"], ds["comparison"], ds["fallback"], ds["contacts"]]
    assert hs.min_distance == ds["min_distance"]
