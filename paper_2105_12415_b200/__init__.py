"""B200-native (sm_100a) triangle-pair contact kernels of arXiv 2105.12415.

Hot path: the batched per-pair triangle-triangle distance / contact kernel
of the reference (/root/reference/pkg/src/tricontact/kernels.py) in its
three variants -- comparison (brute force), iterative and hybrid -- as
hand-written CUDA behind the C ABI in include/tricontact_b200.h.

  kernels   drop-in mirror of ``tricontact.kernels`` (numpy in/out, host C-ABI)
  device    device-resident entry points on torch CUDA tensors
  shard     contiguous-range sharding over ranks + stats all-reduce
  workloads seeded synthetic inputs of BASELINE.json's configs
"""

__version__ = "0.1.0"
