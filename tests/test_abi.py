"""CPU-side checks of the C-ABI boundary: the library builds for sm_100a,
loads, and exports every symbol include/tricontact_b200.h declares."""

import ctypes
import re
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
HEADER = ROOT / "include" / "tricontact_b200.h"


def header_symbols():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    names = re.findall(r"^\s*(?:const\s+)?[\w\s\*]+?\b(tc_\w+)\s*\(", text, flags=re.M)
    return sorted(set(names))


@pytest.fixture(scope="module")
def lib_path():
    from paper_2105_12415_b200 import _build
    return _build.build()


def test_header_symbols_parsed():
    syms = header_symbols()
    assert "tc_hybrid_f64" in syms and "tc_run_host_f32" in syms
    assert len(syms) >= 20


def test_library_exports_every_header_symbol(lib_path):
    out = subprocess.run(["nm", "-D", "--defined-only", str(lib_path)], capture_output=True, text=True,
                         check=True).stdout
    exported = set(re.findall(r"\b(tc_\w+)$", out, flags=re.M))
    missing = [s for s in header_symbols() if s not in exported]
    assert not missing, missing


def test_ctypes_binding_covers_header(lib_path):
    from paper_2105_12415_b200 import _abi
    assert set(header_symbols()) == set(_abi.SIGNATURES)
    lib = _abi.load(lib_path)
    assert lib.tc_abi_version() == _abi.TC_ABI_VERSION == 2
    p = _abi.TcParams()
    lib.tc_params_default(ctypes.byref(p))
    assert (p.epsilon, p.n_iterative, p.alpha_iterative, p.move_factor) == (1e-2, 4, 10.0, 0.25)


def test_struct_layouts():
    from paper_2105_12415_b200 import _abi
    assert ctypes.sizeof(_abi.TcParams) == 56
    assert ctypes.sizeof(_abi.TcStats) == 56


def test_sass_is_sm100a(lib_path):
    out = subprocess.run(["cuobjdump", "--list-elf", str(lib_path)], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_bad_arguments_fail_without_gpu(lib_path):
    """Argument validation happens before any CUDA call."""
    from paper_2105_12415_b200 import _abi
    lib = _abi.load(lib_path)
    p = _abi.TcParams()
    lib.tc_params_default(ctypes.byref(p))
    assert lib.tc_hybrid_f64(None, None, -1, None, None, ctypes.byref(p), *([None] * 9)) == _abi.TC_EINVAL
    p.n_iterative = 0
    assert lib.tc_iterative_f64(None, None, 4, None, ctypes.byref(p), *([None] * 9)) == _abi.TC_EINVAL
    lib.tc_params_default(ctypes.byref(p))
    # n == 0 is a valid no-op
    assert lib.tc_comparison_f32(None, None, 0, None, ctypes.byref(p), *([None] * 9)) == _abi.TC_OK
