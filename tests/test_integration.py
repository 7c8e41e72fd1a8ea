"""INTEGRATION.md section 2 exercised: the drop-in served as
``tricontact.kernels`` before the reference's callers import it (CPU only;
needs /root/reference, so it is skipped on the GPU box)."""

import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
REF = Path("/root/reference/pkg/src")

SCRIPT = r"""
import sys
sys.path.insert(0, {root!r})
sys.path.insert(1, {ref!r})
import paper_2105_12415_b200.kernels as b200
sys.modules["tricontact.kernels"] = b200     # before anything imports tricontact
import tricontact
tricontact.kernels = b200
import tricontact.stepping as stepping
import tricontact.contact as contact
assert tricontact.kernels is b200
for name in ("DegenerateTriangle", "KernelCounters", "KernelParams", "Kind", "batch_closest", "closest_hybrid",
             "gradient_of_J"):
    assert getattr(tricontact, name) is getattr(b200, name), ("package re-export", name)  # RK/__init__.py:9-11
assert stepping.hybrid_batch is b200.hybrid_batch, "stepping binds by name (RK/stepping.py:21)"
assert contact.hybrid_batch is b200.hybrid_batch, "contact binds by name (RK/contact.py:19)"
# the drop-in's public names cover the reference module's
import importlib.util
spec = importlib.util.spec_from_file_location("tricontact._reference_kernels", {ref!r} + "/tricontact/kernels.py")
ref = importlib.util.module_from_spec(spec)
ref.__package__ = "tricontact"
sys.modules["tricontact._reference_kernels"] = ref
spec.loader.exec_module(ref)
public = [n for n in dir(ref) if not n.startswith("_")
          and getattr(getattr(ref, n), "__module__", None) == "tricontact._reference_kernels"]
missing = [n for n in public if not hasattr(b200, n)]
assert not missing, missing
# signatures and keyword defaults of the batch API match
import inspect
for name in ("comparison_batch", "iterative_batch", "hybrid_batch", "closest_point_triangle_batch",
             "closest_comparison", "closest_iterative", "closest_hybrid", "batch_closest",
             "functional_value", "gradient_of_J"):
    a = inspect.signature(getattr(ref, name)).parameters
    b = inspect.signature(getattr(b200, name)).parameters
    assert list(a) == list(b), (name, list(a), list(b))
    assert [p.default for p in a.values()] == [p.default for p in b.values()], name
print("integration ok", len(public))
"""


@pytest.mark.skipif(not REF.exists(), reason="needs the reference sources (/root/reference)")
def test_dropin_served_as_tricontact_kernels():
    r = subprocess.run([sys.executable, "-c", SCRIPT.format(root=str(ROOT), ref=str(REF))], capture_output=True,
                       text=True, timeout=300)
    assert r.returncode == 0 and "integration ok" in r.stdout, r.stderr[-3000:]
