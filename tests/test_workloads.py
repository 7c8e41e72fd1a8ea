"""Workload generators: the counter-based Philox generator of the cfg0
distribution (device: tc_random_pairs_soa_f64; numpy mirror in workloads.py)."""

import ctypes

import numpy as np
import pytest

from paper_2105_12415_b200 import workloads as W


def test_philox_known_answers():
    """Random123's philox4x32_10 known-answer vectors."""
    kat = [((0, 0, 0, 0, 0, 0), (0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8)),
           ((0xFFFFFFFF,) * 6, (0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD)),
           ((0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344, 0xA4093822, 0x299F31D0),
            (0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1))]
    for args, want in kat:
        assert tuple(int(x) for x in W.philox4x32_10(*args)) == want


def test_philox_pairs_distribution_and_shards():
    A, B = W.philox_pairs(1 << 16, seed=4, sep=(-0.05, 0.2))
    assert A.min() >= 0.0 and A.max() < 1.0
    # B is A rigidly moved: same edge lengths; centroid shift |s| with s ~ U[-0.05, 0.2]
    la = np.linalg.norm(np.roll(A, -1, 1) - A, axis=2)
    lb = np.linalg.norm(np.roll(B, -1, 1) - B, axis=2)
    assert np.abs(la - lb).max() < 1e-12
    shift = np.linalg.norm(B.mean(1) - A.mean(1), axis=1)
    assert shift.max() <= 0.2 + 1e-12 and abs(shift.mean() - 0.085) < 2e-3
    a2, b2 = W.philox_pairs(1000, seed=4, sep=(-0.05, 0.2), start=5000)
    assert np.array_equal(a2, A[5000:6000]) and np.array_equal(b2, B[5000:6000])


@pytest.mark.gpu
def test_device_generator_matches_numpy_mirror():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2105_12415_b200 import _abi
    n, start = 50000, 123457
    planes = torch.empty((18, n), dtype=torch.float64, device="cuda")
    lib = _abi.load()
    _abi.check(lib.tc_random_pairs_soa_f64(4, start, n, -0.05, 0.2, ctypes.c_void_p(planes.data_ptr()), None),
               "tc_random_pairs_soa_f64")
    torch.cuda.synchronize()
    P = planes.cpu().numpy()
    A, B = W.philox_pairs(n, seed=4, sep=(-0.05, 0.2), start=start)
    soa = W.to_soa(A, B)
    assert np.array_equal(P[:9], soa[:9])          # the uniforms are exact
    assert np.abs(P[9:] - soa[9:]).max() < 1e-12   # log / sincos / rsqrt round differently
