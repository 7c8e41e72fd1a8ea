"""Stand-in for compute-sanitizer (closed on this GPU pool): the TC_DEBUG
library traps on any fallback-queue overflow, out-of-range queued index or
leftover queue entry, and every batched kernel runs at several CTA caps
(tc_debug_set_max_ctas) so the queues see every fill pattern; results must
not depend on the cap (tools/stress_run.py, in a child process so a trap
cannot poison this one's CUDA context).  Plus run-to-run determinism of the
release library."""

import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2105_12415_b200 import _abi, _build, device as D  # noqa: E402
from paper_2105_12415_b200 import workloads as W  # noqa: E402

ROOT = Path(__file__).resolve().parent.parent


def test_debug_library_stress():
    assert _build.LIB_DEBUG.exists(), "build() compiles the TC_DEBUG library"
    env = dict(os.environ, TC_LIB_PATH=str(_build.LIB_DEBUG))
    r = subprocess.run([sys.executable, str(ROOT / "tools" / "stress_run.py")], env=env, capture_output=True,
                       text=True, timeout=1200)
    assert r.returncode == 0 and "stress ok" in r.stdout, (r.stdout[-2000:], r.stderr[-3000:])
    assert "libtricontact_b200_debug.so" in r.stdout


@pytest.mark.parametrize("strict", [True, False])
def test_release_determinism_and_cap_invariance(strict):
    A, B = W.random_pairs(1 << 18, seed=41, sep=(-0.1, 0.5))
    pl = torch.from_numpy(W.to_soa(A, B)).cuda()
    ta, tb = pl[:9], pl[9:]
    P = D.Params(n_iterative=16, epsilon=1e-6)
    lib = _abi.load()
    ref = None
    try:
        for cap in (0, 0, 0, 5, 148, 0):
            lib.tc_debug_set_max_ctas(cap)
            st = D.new_stats()
            out = D.run("hybrid", ta, tb, P, soa=True, strict=strict, ids=True, stats=st)
            torch.cuda.synchronize()
            cur = {k: v.cpu().numpy() for k, v in out.items()}
            cur["stats"] = np.array(list(D.read_stats(st).values()))
            if ref is None:
                ref = cur
            for k in ref:
                assert np.array_equal(ref[k], cur[k]), (cap, k)
    finally:
        lib.tc_debug_set_max_ctas(0)


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
def test_self_serving_instance_equals_plain(dtype):
    """The fast hybrid's self-serving instance (iterative warps run the comparison
    phases for their own open pairs when the ring is nearly full) is selected from
    the device's fallback history (polls of producers on a full ring switch it on,
    no self-served tiles switch it off): a batch with ~84 % fallbacks (cfg3
    near-parallel faces) switches it on, well-separated pairs off again, and every
    column, the ids and the counters equal the plain instance's bit for bit -- with
    and without feature ids, per-pair halos and an allow mask."""
    lib = _abi.load()
    n = 1 << 17
    A3, B3 = W.adversarial_pairs(n)
    # class 0 (near-parallel faces, ~84 % fallbacks, few intersections) mixed with cfg1 pairs
    # (41 % fallbacks, most of them intersecting): both fallback outcomes get self-served
    Ac, Bc = W.random_pairs(n // 8, seed=47, sep=(-0.1, 0.5))
    perm = np.random.default_rng(7).permutation(n + n // 8)[:n]
    Ah, Bh = np.concatenate([A3[:n], Ac])[perm], np.concatenate([B3[:n], Bc])[perm]
    hot = torch.from_numpy(W.to_soa(Ah, Bh)).cuda().to(dtype)
    A1, B1 = W.random_pairs(n, seed=43, sep=(0.3, 0.5))  # well separated: few fallbacks
    cold = torch.from_numpy(W.to_soa(A1, B1)).cuda().to(dtype)
    P = D.Params(n_iterative=16, epsilon=1e-6)
    rng = np.random.default_rng(5)
    eps = torch.from_numpy(rng.uniform(5e-7, 2e-6, n)).cuda().to(dtype)
    allow = torch.from_numpy((rng.random(n) < 0.9).astype(np.uint8)).cuda()

    def run(pl, **kw):
        st = D.new_stats()
        out = D.run("hybrid", pl[:9], pl[9:], P, soa=True, stats=st, **kw)
        torch.cuda.synchronize()
        res = {k: v.cpu().numpy() for k, v in out.items()}
        res["stats"] = np.array(list(D.read_stats(st).values()))
        return res

    def settle(pl, want):
        # the history needs 2^16 freshly counted pairs: a few synchronised launches
        for _ in range(6):
            run(pl)
            if lib.tc_debug_fallback_rate_high() == want:
                return
        raise AssertionError(f"fallback history did not reach {want}")

    settle(cold, 0)
    plain = [run(hot), ]                       # launched with the plain instance
    settle(hot, 1)
    served = [run(hot), run(hot, ids=True), run(hot, ids=True, eps=eps, allow=allow)]
    assert lib.tc_debug_fallback_rate_high() == 1
    settle(cold, 0)
    plain += [run(hot, ids=True), ]            # plain again (the launch reads the history first)
    settle(cold, 0)
    plain += [run(hot, ids=True, eps=eps, allow=allow)]
    assert served[0]["stats"][2] > 0.6 * n     # the batch does fall back
    assert served[0]["stats"][5] > 0.02 * n    # ... and has intersecting pairs
    for a, b in zip(plain, served):
        assert a.keys() == b.keys()
        for k in a:
            assert np.array_equal(a[k], b[k]), k


def test_fused_kernel_for_rare_fallbacks_equals_warp_specialised():
    """Far-apart pairs (under 8 % fallbacks) switch the fast hybrid to the fused kernel,
    ordinary pairs back; both kernels give the same bits."""
    lib = _abi.load()
    n = 1 << 17
    Af, Bf = W.random_pairs(n, seed=51, sep=(2.0, 3.0))
    far = torch.from_numpy(W.to_soa(Af, Bf)).cuda()
    Ac, Bc = W.random_pairs(n, seed=53, sep=(-0.1, 0.5))
    near = torch.from_numpy(W.to_soa(Ac, Bc)).cuda()
    P = D.Params(n_iterative=16, epsilon=1e-6)

    def run(pl, **kw):
        st = D.new_stats()
        out = D.run("hybrid", pl[:9], pl[9:], P, soa=True, stats=st, **kw)
        torch.cuda.synchronize()
        res = {k: v.cpu().numpy() for k, v in out.items()}
        res["stats"] = np.array(list(D.read_stats(st).values()))
        return res

    def settle(pl, want):
        for _ in range(8):
            run(pl)
            if lib.tc_debug_hybrid_mode() == want:
                return
        raise AssertionError(f"hybrid mode did not reach {want}")

    settle(near, 0)
    ws = [run(far, ids=True), ]
    settle(far, 2)
    fused = [run(far, ids=True), run(near, ids=True)]
    settle(near, 0)
    ws += [run(near, ids=True)]
    assert ws[0]["stats"][2] < 0.05 * n
    for a, b in zip(ws, fused):
        for k in a:
            assert np.array_equal(a[k], b[k]), k


def test_fast_hybrid_under_graph_capture():
    """A caller may capture the launch in a CUDA graph: the library then leaves its
    per-device history alone (no allocation, no choice frozen from it) and the
    replayed kernel gives the eager results."""
    n = 1 << 15
    A, B = W.random_pairs(n, seed=61, sep=(-0.1, 0.5))
    pl = torch.from_numpy(W.to_soa(A, B)).cuda()
    P = D.Params(n_iterative=16, epsilon=1e-6)
    eager = D.run("hybrid", pl[:9], pl[9:], P, soa=True)
    torch.cuda.synchronize()
    out = D.alloc_outputs(n, pl.dtype, "cuda", soa=True)
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        D.run("hybrid", pl[:9], pl[9:], P, soa=True, out=out)  # warm-up outside the capture
    torch.cuda.current_stream().wait_stream(side)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        D.run("hybrid", pl[:9], pl[9:], P, soa=True, out=out)
    for v in out.values():
        v.zero_()
    g.replay()
    torch.cuda.synchronize()
    for k in eager:
        assert torch.equal(eager[k], out[k]), k
