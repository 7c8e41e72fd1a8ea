"""Bitwise comparison of two library builds' outputs (tools only): every
column of the hybrid (and the stats) on the same device-resident cfg1 pairs.

    python tools/libcmp.py variants/a.so variants/b.so [--n N] [--strict] [--dtype f32] [--aos]
"""
import argparse, ctypes, sys
from pathlib import Path
ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import torch
from paper_2105_12415_b200 import _abi, device as D

ap = argparse.ArgumentParser()
ap.add_argument("libs", nargs=2)
ap.add_argument("--n", type=int, default=1 << 20)
ap.add_argument("--strict", action="store_true")
ap.add_argument("--dtype", default="f64")
ap.add_argument("--eps-mask", action="store_true", help="per-pair eps and a random allow mask")
args = ap.parse_args()
dt = torch.float64 if args.dtype == "f64" else torch.float32
n = args.n
lib0 = _abi.load()
planes = torch.empty((18, n), dtype=torch.float64, device="cuda")
_abi.check(lib0.tc_random_pairs_soa_f64(0, 0, n, -0.1, 0.5, ctypes.c_void_p(planes.data_ptr()), None), "gen")
planes = planes.to(dt)
ta, tb = planes[:9], planes[9:]
P = D.Params(n_iterative=16, epsilon=1e-6)
flags = _abi.TC_SOA | _abi.TC_EMIT_IDS | (_abi.TC_STRICT if args.strict else 0)
p = _abi.params_struct(P, flags)
g = torch.Generator(device="cuda").manual_seed(1)
eps = (torch.rand(n, device="cuda", generator=g, dtype=torch.float64) * 2e-6).to(dt) if args.eps_mask else None
allow = (torch.rand(n, device="cuda", generator=g) < 0.8).to(torch.uint8) if args.eps_mask else None
ptr = lambda t: ctypes.c_void_p(t.data_ptr()) if t is not None else None
res = []
for path in args.libs:
    lib = _abi.load(path)
    out = D.alloc_outputs(n, dt, "cuda", soa=True, ids=True)
    st = D.new_stats()
    fn = getattr(lib, f"tc_hybrid_{'f64' if dt == torch.float64 else 'f32'}")
    cols = [ptr(out[k]) for k in ("distance", "point_a", "point_b", "bary_a", "bary_b", "kind", "ids")]
    rc = fn(ptr(ta), ptr(tb), n, ptr(eps), ptr(allow), ctypes.byref(p), *cols, ptr(st), None)
    torch.cuda.synchronize()
    assert rc == 0, rc
    res.append((out, D.read_stats(st)))
(o0, s0), (o1, s1) = res
bad = {k: int((o0[k].view(torch.uint8) != o1[k].view(torch.uint8)).sum()) for k in o0}
print(f"n={n} strict={args.strict} {args.dtype} eps_mask={args.eps_mask}: differing bytes {bad}")
print(" stats", s0 == s1, s0, s1 if s0 != s1 else "")
sys.exit(0 if (not any(bad.values()) and s0 == s1) else 1)
