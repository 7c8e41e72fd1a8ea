"""Co-residency probe (tools only): the iterative kernel over all cfg1 pairs and
the comparison kernel over the compacted open pairs, alone and concurrently on
two streams with capped grids -- does overlapping the two roles beat their sum?

    python tools/corun.py
"""
import ctypes, sys
from pathlib import Path
ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import torch
from paper_2105_12415_b200 import _abi, device as D

n = 1 << 24
lib = _abi.load()
planes = torch.empty((18, n), dtype=torch.float64, device="cuda")
_abi.check(lib.tc_random_pairs_soa_f64(0, 0, n, -0.1, 0.5, ctypes.c_void_p(planes.data_ptr()), None), "gen")
P = D.Params(n_iterative=16, epsilon=1e-6)
ta, tb = planes[:9], planes[9:]
out = D.alloc_outputs(n, torch.float64, "cuda", soa=True, ids=True)
D.run("hybrid", ta, tb, P, soa=True, out=out, ids=True)
torch.cuda.synchronize()
idx = torch.nonzero((out["ids"][:, 3] & 4) > 0).squeeze(1)
m = idx.numel()
ca, cb = ta[:, idx].contiguous(), tb[:, idx].contiguous()
o_all = D.alloc_outputs(n, torch.float64, "cuda", soa=True)
o_m = D.alloc_outputs(m, torch.float64, "cuda", soa=True)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
SM = torch.cuda.get_device_properties(0).multi_processor_count


def it(cap, st):
    lib.tc_debug_set_max_ctas(cap)
    D.run("iterative", ta, tb, P, soa=True, out=o_all, stream=st)


def cm(cap, st):
    lib.tc_debug_set_max_ctas(cap)
    D.run("comparison", ca, cb, P, soa=True, out=o_m, stream=st)


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def both(ci, cc):
    def f():
        ev = torch.cuda.Event()
        ev.record()
        s1.wait_event(ev)
        s2.wait_event(ev)
        it(ci, s1)
        cm(cc, s2)
        a, b = torch.cuda.Event(), torch.cuda.Event()
        a.record(s1)
        b.record(s2)
        torch.cuda.current_stream().wait_event(a)
        torch.cuda.current_stream().wait_event(b)
    return f


cur = torch.cuda.current_stream()
print(f"open pairs {m}")
print(f"iterative full grid      {timed(lambda: it(0, cur)):.3f} ms")
print(f"comparison(open) full    {timed(lambda: cm(0, cur)):.3f} ms")
for ci, cc in ((SM, 4 * SM), (SM, 2 * SM), (2 * SM, 2 * SM)):
    print(f"caps it={ci // SM}/SM cmp={cc // SM}/SM: it alone {timed(lambda: it(ci, cur)):.3f}  "
          f"cmp alone {timed(lambda: cm(cc, cur)):.3f}  concurrent {timed(both(ci, cc)):.3f} ms")
lib.tc_debug_set_max_ctas(0)
