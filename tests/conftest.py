import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))

GOLDEN = ROOT / "tests" / "golden"

# the two parameter sets every parity case runs at: the reference defaults
# (RK/kernels.py:56-62) and BASELINE.json config 0's (16 sweeps, eps 1e-6)
PARAM_SETS = {"def": dict(), "bl": dict(n_iterative=16, epsilon=1e-6)}
DTYPES = {"float64": np.float64, "float32": np.float32}


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def golden_inputs():
    return dict(np.load(GOLDEN / "inputs.npz"))


@pytest.fixture(scope="session")
def golden_ref():
    return {real: dict(np.load(GOLDEN / f"ref_{real}.npz")) for real in DTYPES}


@pytest.fixture(scope="session")
def oracle_lib():
    import oracle
    oracle.build()
    return oracle


@pytest.fixture(scope="session")
def golden_r2():
    """Round-2 fixtures from the reference (tests/golden/make_golden_r2.py)."""
    return {real: dict(np.load(GOLDEN / f"r2_{real}.npz")) for real in DTYPES}
