"""Time the drop-in numpy path (kernels.hybrid_batch on pageable arrays,
staged through the library's pinned buffers) against the PCIe floor.

    python tools/e2e_dropin.py [n] [strict|fast]
"""
import sys
import time
from pathlib import Path
ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import numpy as np
from paper_2105_12415_b200 import kernels as K, workloads as W

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 24
mode = sys.argv[2] if len(sys.argv) > 2 else "strict"
K.set_rounding(mode)
A, B = W.random_pairs_mp(n, seed=0, sep=(-0.1, 0.5))
p = K.KernelParams(n_iterative=16, epsilon=1e-6)
r = K.hybrid_batch(A, B, p, None, 1e-6)
del r
for rep in range(3):
    t0 = time.perf_counter()
    r = K.hybrid_batch(A, B, p, None, 1e-6)
    dt = time.perf_counter() - t0
    del r
    print(f"{mode} n={n}: {dt * 1e3:.1f} ms  {n / dt / 1e6:.1f} M pairs/s  "
          f"{(n * 144 + n * 89) / dt / 1e9:.1f} GB/s host<->device payload", flush=True)
