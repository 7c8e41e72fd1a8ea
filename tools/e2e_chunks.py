"""e2e (tc_run_host_f64) time per step for a few pipeline chunk sizes: TC_HOST_CHUNK=... python tools/e2e_chunks.py"""
import ctypes, json, os, sys, time
from pathlib import Path
ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import torch
import bench
from paper_2105_12415_b200 import _abi, workloads as W
n = 1 << 24
A, B = W.random_pairs(n, seed=0, sep=bench.SEP)
r = bench.e2e_measure(_abi.load(), _abi, torch, A, B, n, 1, None, torch.device("cuda:0"))
print(os.environ.get("TC_HOST_CHUNK", "default"), json.dumps({k: r[k] for k in ("value", "ms_per_step", "link")}))
