"""Build the in-tree C-ABI library libtricontact_b200.so (sm_100a).

    python -m paper_2105_12415_b200._build

nvcc cross-compiles for sm_100a without a GPU; the .so lands next to this
file so it travels with the repo snapshot to the GPU box.  cudart is linked
statically so the library loads with or without torch in the process.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIB = PKG / "libtricontact_b200.so"
# TC_DEBUG build: device-side traps on queue overflow / out-of-range indices
# (tests/test_gpu_stress.py) -- the checks compute-sanitizer would provide
LIB_DEBUG = PKG / "libtricontact_b200_debug.so"
SOURCES = [CSRC / "tc_kernels.cu"]
DEPS = SOURCES + sorted(CSRC.glob("*.cuh")) + [ROOT / "include" / "tricontact_b200.h"]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-shared",
    "-I", str(ROOT / "include"),
]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found")


def stale(lib: Path = LIB) -> bool:
    if not lib.exists():
        return True
    t = lib.stat().st_mtime
    return any(p.stat().st_mtime > t for p in DEPS)


def _cmd(target: Path, defines, verbose=False):
    tmp = target.with_suffix(".so.tmp")
    return tmp, [nvcc(), *NVCC_FLAGS, *(["-Xptxas", "-v"] if verbose else []), *[f"-D{d}" for d in defines],
                 "-o", str(tmp), *map(str, SOURCES)]


def build(force: bool = False, verbose: bool = False, out: Path | None = None, defines=(), debug=True) -> Path:
    """Compile the library (``out``/``defines``: experiment variants, e.g. launch
    bounds); the default build also compiles the TC_DEBUG library, in parallel."""
    if out is not None or defines:
        target = Path(out) if out else LIB
        tmp, cmd = _cmd(target, defines, verbose)
        subprocess.run(cmd, check=True)
        os.replace(tmp, target)
        return target
    jobs = []
    targets = [(LIB, ())] + ([(LIB_DEBUG, ("TC_DEBUG=1",))] if debug else [])
    for target, defs in targets:
        if force or stale(target):
            tmp, cmd = _cmd(target, defs, verbose)
            jobs.append((subprocess.Popen(cmd), tmp, target))
    for proc, tmp, target in jobs:
        if proc.wait() != 0:
            raise subprocess.CalledProcessError(proc.returncode, "nvcc")
        os.replace(tmp, target)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
