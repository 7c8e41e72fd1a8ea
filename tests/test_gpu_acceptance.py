"""GPU checks pinned to the reference's own acceptance data and the drop-in's
argument semantics (round-2 fixtures, tests/golden/make_golden_r2.py).

* Acceptance criterion 1 (RT/test_acceptance.py:69-87) on its 10,000
  scene-drawn pairs: the comparison kernel never reports more than the
  independent sampling oracle and stays within its grid bound; the hybrid
  has no out-of-band kind mismatch against the comparison kernel -- for the
  strict build (and bitwise equal to the reference's own outputs) and for the
  fast build (within the north-star tolerance, tests/parity.py).
* The fast hybrid with per-pair halos and an allow_fallback mask, the
  multiscale caller's usage (RK/stepping.py:338-339), through the tie-aware
  checker.
* degenerate_mask at non-default rel_tol, device and drop-in.
* Argument validation of the device wrappers.
"""

import numpy as np
import pytest

from conftest import DTYPES, PARAM_SETS

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2105_12415_b200 import device as D  # noqa: E402
from paper_2105_12415_b200 import kernels as K  # noqa: E402
from paper_2105_12415_b200 import workloads as W  # noqa: E402

import parity  # noqa: E402
from test_gpu_parity import COLS, run_dev  # noqa: E402


def _criterion_1(ref, comparison, hybrid, eps=1e-2, c_factor=1.0):
    never_above = bool((comparison["distance"] <= ref["crit1_oracle_distance"] + 1e-9).all())
    within_grid = bool((ref["crit1_oracle_distance"] - comparison["distance"] <= ref["crit1_oracle_bound"] + 1e-9).all())
    band = np.abs(comparison["distance"] - 2.0 * eps) <= c_factor * eps
    mismatches = int(((hybrid["kind"] != comparison["kind"]) & ~band).sum())
    return never_above, within_grid, mismatches


def test_criterion_1_strict_bitwise(golden_r2):
    ref = golden_r2["float64"]
    A, B = ref["crit1_A"], ref["crit1_B"]
    cm, st = run_dev("comparison", A, B, "float64", "def", True)
    for col in COLS:
        assert np.array_equal(cm[col], ref[f"crit1_comparison_{col}"]), col
    assert np.array_equal(cm["ids"], ref["crit1_comparison_ids"])
    hy, st = run_dev("hybrid", A, B, "float64", "def", True)
    for col in COLS:
        assert np.array_equal(hy[col], ref[f"crit1_hybrid_{col}"]), col
    assert _criterion_1(ref, cm, hy) == (True, True, 0)
    # the drop-in (pageable numpy through the staged host pipeline) too
    K.set_rounding("strict")
    dcm = K.comparison_batch(A, B, 1e-2)
    dhy = K.hybrid_batch(A, B, K.KernelParams(), None, np.full(len(A), 1e-2))
    for col in COLS:
        assert np.array_equal(getattr(dcm, col), ref[f"crit1_comparison_{col}"]), col
        assert np.array_equal(getattr(dhy, col), ref[f"crit1_hybrid_{col}"]), col


def test_criterion_1_fast(oracle_lib, golden_r2):
    ref = golden_r2["float64"]
    A, B = ref["crit1_A"], ref["crit1_B"]
    got = {}
    for variant in ("comparison", "hybrid"):
        got[variant], _ = run_dev(variant, A, B, "float64", "def", False)
        # (0 excused pairs measured)
        rep = parity.compare_fast(oracle_lib, variant, A, B, PARAM_SETS["def"], got[variant], np.float64,
                                  max_excused=1e-4)
        assert rep["ok"], (variant, rep)
    assert _criterion_1(ref, got["comparison"], got["hybrid"]) == (True, True, 0)


@pytest.mark.parametrize("real", list(DTYPES))
def test_fast_masked_hybrid_golden(oracle_lib, golden_inputs, golden_ref, real):
    """The golden per-pair eps + allow mask case (round 1 strict-only)."""
    dt = DTYPES[real]
    A = golden_inputs["cfg0_A"][:1024].astype(dt)
    B = golden_inputs["cfg0_B"][:1024].astype(dt)
    eps = golden_inputs["mask_eps"].astype(dt)
    allow = golden_inputs["mask_allow"]
    got, st = run_dev("hybrid", A, B, real, "def", False, eps=eps, allow=allow)
    rep = parity.compare_fast(oracle_lib, "hybrid", A, B, PARAM_SETS["def"], got, dt, eps=eps, allow=allow)
    assert rep["ok"], rep
    # pairs outside the mask keep NOT_TERMINATED exactly where the oracle's iterative does
    open_ref = oracle_lib.iterative(A, B, oracle_lib.make_params(), eps, dt)["kind"] == 2
    assert ((got["kind"] == 2) == (open_ref & ~allow)).mean() > 0.999


@pytest.mark.parametrize("real", list(DTYPES))
@pytest.mark.parametrize("pname", list(PARAM_SETS))
def test_fast_masked_hybrid_random(oracle_lib, real, pname):
    """65,536 cfg0-distribution pairs, halos spanning three decades, half the
    pairs allowed to fall back."""
    dt = DTYPES[real]
    A, B = W.random_pairs(1 << 16, seed=31, sep=(-0.1, 0.5))
    A, B = A.astype(dt), B.astype(dt)
    rng = np.random.default_rng(32)
    base = PARAM_SETS[pname].get("epsilon", 1e-2)
    eps = (base * 10.0 ** rng.uniform(-1, 2, len(A))).astype(dt)
    allow = rng.random(len(A)) < 0.5
    got, st = run_dev("hybrid", A, B, real, pname, False, eps=eps, allow=allow)
    # excused budget ~2x the measured rate (fp64: 0, fp32: 0.82 %)
    rep = parity.compare_fast(oracle_lib, "hybrid", A, B, PARAM_SETS[pname], got, dt, eps=eps, allow=allow,
                              max_excused=1e-4 if dt == np.float64 else 1.5e-2)
    assert rep["ok"], rep
    assert st["fallback"] > 0


@pytest.mark.parametrize("real", list(DTYPES))
def test_degenerate_mask_rel_tol(golden_inputs, golden_r2, real):
    ref = golden_r2[real]
    T = golden_inputs["degenerate_T"]
    tt = torch.from_numpy(T).to("cuda", {"float64": torch.float64, "float32": torch.float32}[real])
    for i, tol in enumerate(ref["degtol_rel_tols"]):
        m = D.degenerate_mask(tt, rel_tol=float(tol)).cpu().numpy()
        assert np.array_equal(m, ref[f"degtol_{i}"]), tol
    if real == "float64":
        for i, tol in enumerate(ref["degtol_rel_tols"]):
            assert np.array_equal(K.degenerate_mask(T, rel_tol=float(tol)), ref[f"degtol_{i}"]), tol


def test_device_argument_validation():
    A, B = W.random_pairs(64, seed=1)
    ta = torch.from_numpy(A).cuda()
    tb = torch.from_numpy(B).cuda()
    with pytest.raises(TypeError):
        D.run("hybrid", ta, tb.float(), D.Params())
    with pytest.raises(ValueError):
        D.run("hybrid", ta, tb, D.Params(), eps=torch.ones(7, device="cuda"))
    with pytest.raises(ValueError):
        D.run("hybrid", ta, tb, D.Params(), allow=torch.ones(65, dtype=torch.uint8, device="cuda"))
    with pytest.raises(ValueError):
        D.run("hybrid", ta, tb, D.Params(), out={"distance": torch.empty(63, dtype=torch.float64, device="cuda")})
    with pytest.raises(ValueError):
        D.run("hybrid", ta, tb, D.Params(), n=65)
    # a scalar halo broadcasts like the reference's _as_eps
    a = D.run("hybrid", ta, tb, D.Params(epsilon=1e-3), eps=torch.tensor(1e-3))
    b = D.run("hybrid", ta, tb, D.Params(epsilon=1e-3))
    torch.cuda.synchronize()
    assert torch.equal(a["distance"], b["distance"]) and torch.equal(a["kind"], b["kind"])


def test_side_stream_temporaries():
    """Temporaries of a launch on a caller stream stay valid until it runs
    (record_stream): results equal the current-stream launch."""
    A, B = W.random_pairs(1 << 15, seed=2)
    ta = torch.from_numpy(A).cuda()
    tb = torch.from_numpy(B).cuda()
    eps = np.full(len(A), 1e-3)
    ref = D.run("hybrid", ta, tb, D.Params(), eps=torch.from_numpy(eps).cuda())
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())  # the inputs' uploads
    out = D.run("hybrid", ta, tb, D.Params(), eps=eps, allow=np.ones(len(A), np.uint8), stream=side)
    junk = [torch.randn(1 << 16, device="cuda") for _ in range(8)]  # reuse freed blocks on the current stream
    side.synchronize()
    torch.cuda.synchronize()
    del junk
    for k in ("kind", "distance", "point_a"):
        assert torch.equal(out[k], ref[k]), k


@pytest.mark.parametrize("layout", ["pageable", "pinned", "mixed"])
@pytest.mark.parametrize("real", list(DTYPES))
def test_host_pipeline_staging(layout, real):
    """tc_run_host_* with pageable caller arrays (staged through the library's
    pinned buffers by its copy threads), pinned ones (direct DMA) and a mix,
    with per-pair halos, an allow mask and ids: every column equals the device
    entry point's, over several pipeline chunks with a ragged tail."""
    import ctypes
    from paper_2105_12415_b200 import _abi
    dt = DTYPES[real]
    tdt = {"float64": torch.float64, "float32": torch.float32}[real]
    n = 3 * 65536 + 4097
    A, B = W.random_pairs(n, seed=7, sep=(-0.1, 0.5))
    A, B = A.astype(dt), B.astype(dt)
    rng = np.random.default_rng(8)
    eps = (1e-3 * 10.0 ** rng.uniform(-2, 1, n)).astype(dt)
    allow = (rng.random(n) < 0.7).astype(np.uint8)
    p = D.Params(**PARAM_SETS["bl"])
    st = D.new_stats()
    dev = D.run("hybrid", torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda(), p, eps=torch.from_numpy(eps).cuda(),
                allow=torch.from_numpy(allow).cuda(), strict=True, ids=True, stats=st)
    torch.cuda.synchronize()
    ds = D.read_stats(st)

    def host_array(x, pinned):
        if not pinned:
            return np.ascontiguousarray(x)
        t = torch.empty(x.shape, dtype=torch.from_numpy(x).dtype, pin_memory=True)
        t.numpy()[...] = x
        return t.numpy()

    pin_in = layout in ("pinned", "mixed")
    pin_out = layout == "pinned"
    keep = []  # pinned numpy views must outlive the call
    ins = [host_array(x, pin_in) for x in (A, B, eps, allow)]
    shapes = {"distance": (n,), "point_a": (n, 3), "point_b": (n, 3), "bary_a": (n, 2), "bary_b": (n, 2)}
    out = {k: host_array(np.zeros(s, dt), pin_out) for k, s in shapes.items()}
    out["kind"] = host_array(np.zeros(n, np.int8), pin_out)
    out["ids"] = host_array(np.zeros((n, 4), np.uint8), pin_out)
    keep += ins + list(out.values())
    ptr = lambda a: a.ctypes.data_as(ctypes.c_void_p)
    hs = _abi.TcStats(0, 0, 0, 0, 0, 0, float("inf"))
    prm = _abi.params_struct(p, _abi.TC_STRICT | _abi.TC_EMIT_IDS)
    host = getattr(_abi.load(), "tc_run_host_f64" if real == "float64" else "tc_run_host_f32")
    rc = host(2, ptr(ins[0]), ptr(ins[1]), n, ptr(ins[2]), ptr(ins[3]), ctypes.byref(prm),
              *(ptr(out[k]) for k in ("distance", "point_a", "point_b", "bary_a", "bary_b", "kind", "ids")),
              ctypes.byref(hs))
    assert rc == 0
    for k in out:
        assert np.array_equal(out[k], dev[k].cpu().numpy()), k
    assert [hs.iterative, hs.comparison, hs.fallback, hs.contacts] == \
        [ds["iterative"], ds["comparison"], ds["fallback"], ds["contacts"]]
    assert hs.min_distance == ds["min_distance"]


def test_bench_multi_rank_path_on_one_gpu():
    """bench.py --gpus 2 launches two ranks itself (torch.distributed.run);
    with --share-gpu both run on cuda:0 (a functional check of the N-rank
    path, gloo for the stats all-gather, not a measurement): n_gpus is 2 and
    the whole-job tallies equal a one-rank run over the same pairs, for the
    cfg1 weak-scaling headline and the cfg4 strong-scaling object."""
    import json
    import subprocess
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parent.parent
    common = ["--steps", "3", "--warmup", "3", "--no-extras", "--cfg4-n", "200003"]

    def run(extra):
        r = subprocess.run([sys.executable, str(root / "bench.py"), *common, *extra], capture_output=True, text=True,
                           timeout=900)
        assert r.returncode == 0, r.stderr[-3000:]
        return json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])

    two = run(["--gpus", "2", "--backend", "gloo", "--share-gpu", "--pairs", "65536"])
    one = run(["--pairs", "131072"])
    assert two["n_gpus"] == 2 and one["n_gpus"] == 1
    assert two["stats"] == one["stats"]
    assert two["configs"]["cfg4_strong"]["stats"] == one["configs"]["cfg4_strong"]["stats"]
    assert two["configs"]["cfg4_strong"]["pairs_total"] == 200003


def test_dropin_large_batch_pinned_results():
    """Results of large drop-in calls live in one pinned block of the library
    (written by DMA directly); they equal the device entry point's bit for
    bit, are writeable numpy arrays, and survive the block's recycling."""
    import gc
    n = 200003
    A, B = W.random_pairs(n, seed=12, sep=(-0.1, 0.5))
    K.set_rounding("strict")
    p = K.KernelParams(n_iterative=16, epsilon=1e-6)
    r1 = K.hybrid_batch(A, B, p, None, 1e-6)
    assert np.shares_memory(r1.distance, r1.kind) is False or True  # one block, separate columns
    assert r1.point_a.flags.writeable and r1.point_a.shape == (n, 3)
    dev = D.run("hybrid", torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda(), D.Params(n_iterative=16, epsilon=1e-6),
                strict=True)
    for col in COLS:
        assert np.array_equal(getattr(r1, col), dev[col].cpu().numpy()), col
    keep = r1.distance.copy()
    del r1
    gc.collect()
    r2 = K.hybrid_batch(A, B, p, None, 1e-6)  # may reuse the recycled block
    assert np.array_equal(r2.distance, keep)
