"""Time the hybrid kernel of several library builds on the same device-resident
inputs (one process; each variants/*.so loaded through its own ctypes handle).

    python tools/varbench.py [--n N] [--dtype f64|f32] [--rounds R] variants/a.so variants/b.so ...
"""
import argparse
import ctypes
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import torch
from paper_2105_12415_b200 import _abi, device as D, workloads as W

ap = argparse.ArgumentParser()
ap.add_argument("libs", nargs="+")
ap.add_argument("--n", type=int, default=1 << 24)
ap.add_argument("--dtype", default="f64")
ap.add_argument("--rounds", type=int, default=3)
ap.add_argument("--reps", type=int, default=10)
ap.add_argument("--strict", action="store_true")
ap.add_argument("--variant", default="hybrid")
ap.add_argument("--no-fallback", action="store_true", help="hybrid with an all-zero allow mask")
ap.add_argument("--sep", type=float, nargs=2, default=(-0.1, 0.5), help="separation range of the cfg1 generator")
ap.add_argument("--cfg3", type=int, default=-1, help="time class k (0-3) of the adversarial set, 2^20 pairs, instead of cfg1")
args = ap.parse_args()
dt = torch.float64 if args.dtype == "f64" else torch.float32
n = args.n
planes = torch.empty((18, n), dtype=torch.float64, device="cuda")
lib0 = _abi.load()
_abi.check(lib0.tc_random_pairs_soa_f64(0, 0, n, args.sep[0], args.sep[1], ctypes.c_void_p(planes.data_ptr()), None), "gen")
if args.cfg3 >= 0:
    n = 1 << 20
    A3, B3 = W.adversarial_pairs(n)
    sl = slice(args.cfg3 * n, (args.cfg3 + 1) * n)
    planes = torch.from_numpy(W.to_soa(A3[sl], B3[sl])).to("cuda")
planes = planes.to(dt)
ta, tb = planes[:9], planes[9:]
out = D.alloc_outputs(n, dt, "cuda", soa=True)
stats = D.new_stats()
no_fb = torch.zeros(n, dtype=torch.uint8, device="cuda")
P = D.Params(n_iterative=16, epsilon=1e-6)
flags = _abi.TC_SOA | (_abi.TC_STRICT if args.strict else 0)
p = _abi.params_struct(P, flags)
sfx = "f64" if dt == torch.float64 else "f32"
libs = [(Path(x).name, _abi.load(x)) for x in args.libs]
ptr = lambda t: ctypes.c_void_p(t.data_ptr())
cols = [ptr(out[k]) for k in ("distance", "point_a", "point_b", "bary_a", "bary_b", "kind")]
res = {name: [] for name, _ in libs}
hist_of, hist_txt = {}, {}
stats_of = {}
for r in range(args.rounds):
    for name, lib in libs:
        fn = getattr(lib, f"tc_{args.variant}_{sfx}")
        allow = ptr(no_fb) if args.no_fallback else None
        call = (lambda: fn(ptr(ta), ptr(tb), n, None, allow, ctypes.byref(p), *cols, None, ptr(stats), None)) \
            if args.variant == "hybrid" else \
            (lambda: fn(ptr(ta), ptr(tb), n, None, ctypes.byref(p), *cols, None, ptr(stats), None))
        rc = [call() for _ in range(2)]
        if any(rc):
            print(f"{name}: launch failed rc={rc} ({lib.tc_last_error().decode() if hasattr(lib, 'tc_last_error') else ''})",
                  flush=True)
            res[name].append(float('nan'))
            continue
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        lib.tc_stats_reset(ptr(stats), None)
        e0.record()
        for _ in range(args.reps):
            call()
        e1.record()
        torch.cuda.synchronize()
        res[name].append(e0.elapsed_time(e1) / args.reps)
        if hasattr(lib, "tc_debug_fallback_history"):
            h = (ctypes.c_uint64 * 4)()
            lib.tc_debug_fallback_history(h)
            prev = hist_of.get(name, [0, 0, 0, 0])
            d = [int(h[k]) - prev[k] for k in range(4)]
            hist_of[name] = [int(h[k]) for k in range(4)]
            if d[0]:
                hist_txt[name] = (f"history: fb/pair {d[1] / d[0]:.3f} ring waits/tile {32 * d[2] / d[0]:.2f} "
                                  f"self tiles/tile {32 * d[3] / d[0]:.3f}")
        stats_of[name] = D.read_stats(stats)
for name, ts in res.items():
    st = stats_of.get(name, {"fallback": 0, "contacts": 0})
    print(f"{name:40s} {min(ts):7.3f} ms  {n / min(ts) / 1e6:8.1f} M pairs/s  (rounds {' '.join(f'{t:.3f}' for t in ts)})"
          f"  fb {st['fallback'] // (args.reps + 0)} contacts {st['contacts'] // args.reps}  {hist_txt.get(name, '')}", flush=True)
