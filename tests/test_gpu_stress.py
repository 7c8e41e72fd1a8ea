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
