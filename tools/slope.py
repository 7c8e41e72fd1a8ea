"""Marginal cost of one sweep in situ: hybrid without fallback / iterative / full
hybrid at several sweep counts on 2^24 device-generated cfg1-distribution pairs."""
import ctypes, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from paper_2105_12415_b200 import _abi, device as D
n = 1 << 24
planes = torch.empty((18, n), dtype=torch.float64, device="cuda")
lib = _abi.load()
lib.tc_random_pairs_soa_f64(0, 0, n, -0.1, 0.5, ctypes.c_void_p(planes.data_ptr()), None)
ta, tb = planes[:9], planes[9:]
out = D.alloc_outputs(n, torch.float64, "cuda", soa=True)
no = torch.zeros(n, dtype=torch.uint8, device="cuda")
st = D.new_stats()
def t(fn, reps=5):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps
for N in (4, 8, 12, 16, 20):
    P = D.Params(n_iterative=N, epsilon=1e-6)
    it = t(lambda: D.run("iterative", ta, tb, P, soa=True, out=out, n=n))
    nofb = t(lambda: D.run("hybrid", ta, tb, P, soa=True, out=out, n=n, allow=no))
    D.reset_stats(st)
    hy = t(lambda: D.run("hybrid", ta, tb, P, soa=True, out=out, n=n, stats=st), reps=1)
    s = D.read_stats(st)
    print(f"N={N:2d} iterative {it:.3f} ms  hybrid-nofb {nofb:.3f} ms  hybrid {hy:.3f} ms  fallback {s['fallback']/n:.3f}", flush=True)
