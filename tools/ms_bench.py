"""Run bench.py's multiscale table alone: python tools/ms_bench.py [n_pairs ...]."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2105_12415_b200 import device as D  # noqa: E402

for n in [int(a) for a in sys.argv[1:]] or [1024]:
    print(json.dumps(bench.multiscale_table(D, torch, torch.device("cuda:0"), n_pairs=n)), flush=True)
