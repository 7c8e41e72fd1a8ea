"""hybrid with the fallback disabled (allow = 0) vs the iterative kernel, for each TC_LIB_PATH."""
import sys
from pathlib import Path
ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import torch
from paper_2105_12415_b200 import device as D, workloads as W
n = 1 << 24
A, B = W.random_pairs(n)
planes = torch.from_numpy(W.to_soa(A, B)).to("cuda", torch.float64)
ta, tb = planes[:9], planes[9:]
P = D.Params(n_iterative=16, epsilon=1e-6)
out = D.alloc_outputs(n, torch.float64, "cuda", soa=True)
no = torch.zeros(n, dtype=torch.uint8, device="cuda")
def t(fn, reps=5):
    fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return round(e0.elapsed_time(e1) / reps, 4)
print({"iterative": t(lambda: D.run("iterative", ta, tb, P, soa=True, out=out, n=n)),
       "hybrid_nofb": t(lambda: D.run("hybrid", ta, tb, P, soa=True, out=out, n=n, allow=no)),
       "hybrid": t(lambda: D.run("hybrid", ta, tb, P, soa=True, out=out, n=n))})
