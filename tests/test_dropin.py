"""The drop-in tricontact.kernels mirror: host-side behaviour on CPU, and on
the GPU the reference's known answers (RT/test_kernels.py semantics,
restated) plus bitwise equality with the golden vectors."""

import numpy as np
import pytest

from paper_2105_12415_b200 import kernels as K

U = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0]], float)


def off(t, dx=0.0, dy=0.0, dz=0.0):
    return np.asarray(t, float) + np.array([dx, dy, dz])


# ---- CPU: argument handling mirrors RK (no device needed) -----------------

def test_params_validation():
    with pytest.raises(ValueError):
        K.KernelParams(epsilon=0.0)
    with pytest.raises(ValueError):
        K.KernelParams(n_iterative=0)
    with pytest.raises(ValueError):
        K.KernelParams(c_factor=-1.0)
    with pytest.raises(ValueError):
        K.KernelParams(alpha_regulariser=0.0)


def test_shape_errors_before_device():
    with pytest.raises(ValueError):
        K.comparison_batch(np.zeros((4, 3)), np.zeros((4, 3)), 1e-2)
    with pytest.raises(ValueError):
        K.iterative_batch(np.zeros((2, 3, 3)), np.zeros((2, 3, 3)), K.KernelParams(), np.ones(3))


def test_empty_and_counters():
    assert K.batch_closest([], K.KernelParams()) == []
    c = K.KernelCounters(1, 2, 3)
    c.merge(K.KernelCounters(1, 1, 1))
    assert c.as_dict() == {"iterative_invocations": 2, "comparison_invocations": 3, "fallback_invocations": 4}


def test_gradient_matches_finite_differences():
    rng = np.random.default_rng(3)
    p = K.KernelParams()
    for _ in range(20):
        A = rng.normal(size=(3, 3))
        B = rng.normal(size=(3, 3)) + np.array([1.0, 0, 0])
        x = rng.uniform(0.05, 0.45, 4)
        g = K.gradient_of_J(A, B, *x, p)
        h = 1e-6
        fd = np.array([(K.functional_value(A, B, *(x + h * e), p) - K.functional_value(A, B, *(x - h * e), p))
                       / (2 * h) for e in np.eye(4)])
        assert np.linalg.norm(g - fd) / max(np.linalg.norm(fd), 1e-12) < 1e-5


def test_gradient_and_functional_equal_reference(golden_r2):
    """RK/kernels.py:677-717 at acceptance criterion 2's points (seed 20260802):
    bit-identical to the reference's own values (tests/golden/make_golden_r2.py)."""
    ref = golden_r2["float64"]
    p = K.KernelParams()
    for row, g, v in zip(ref["grad_points"], ref["grad_gradient"], ref["grad_value"]):
        A, B, x = row[:9].reshape(3, 3), row[9:18].reshape(3, 3), row[18:]
        assert np.array_equal(K.gradient_of_J(A, B, *x, p), g)
        assert K.functional_value(A, B, *x, p) == v


def test_allow_mask_shapes_follow_numpy_broadcasting():
    """RK/kernels.py:590-591 ANDs the mask into the open pairs: a mask that
    does not broadcast to (n,) raises ValueError before any device work."""
    A = np.zeros((4, 3, 3))
    with pytest.raises(ValueError):
        K.hybrid_batch(A, A, K.KernelParams(), None, 1e-2, allow_fallback=np.ones(3, bool))
    with pytest.raises(ValueError):
        K.hybrid_batch(A, A, K.KernelParams(), None, 1e-2, allow_fallback=np.ones((2, 4), bool))
    with pytest.raises(ValueError):
        K.hybrid_batch(A, A, K.KernelParams(), None, np.ones(3))


# ---- GPU: the drop-in computes through the C ABI ----------------------------

torch = pytest.importorskip("torch")
gpu = pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA device")


@pytest.mark.gpu
@gpu
class TestKnownAnswers:
    def test_identical(self):
        r = K.closest_comparison(U, U)
        assert r.distance == pytest.approx(0.0, abs=1e-12) and r.kind == K.Kind.CONTACT

    def test_parallel_offset(self):
        r = K.closest_comparison(U, off(U, dz=1.0))
        assert r.distance == pytest.approx(1.0, abs=1e-12) and r.kind == K.Kind.NO_CONTACT
        assert r.point_b[2] - r.point_a[2] == pytest.approx(1.0)

    def test_vertex_vertex(self):
        r = K.closest_comparison(U, np.array([[2, 0, 0], [3, 0, 0], [2, 1, 0]], float))
        assert r.distance == pytest.approx(1.0)
        assert np.allclose(r.point_a, [1, 0, 0]) and np.allclose(r.point_b, [2, 0, 0])

    def test_intersecting_point_on_plane(self):
        r = K.closest_comparison(U, np.array([[0.2, 0.2, -0.5], [0.4, 0.2, 0.5], [0.3, 0.4, 0.5]]))
        assert r.distance == 0.0 and r.kind == K.Kind.CONTACT
        assert np.allclose(r.point_a, r.point_b) and abs(r.point_a[2]) < 1e-12

    def test_degenerate_raises(self):
        with pytest.raises(K.DegenerateTriangle):
            K.closest_comparison(U, np.array([[0, 0, 0], [1, 0, 0], [2, 0, 0]], float))

    def test_iterative_parallel_offset(self):
        r = K.closest_iterative(U, off(U, dz=1.0), K.KernelParams())
        assert r.kind == K.Kind.NO_CONTACT and r.distance == pytest.approx(1.0, abs=1e-9)

    def test_hybrid_pass_through_and_fallback_counters(self):
        p = K.KernelParams()
        c = K.KernelCounters()
        r = K.closest_hybrid(U, off(U, dz=1.0), p, c)
        assert r.kind != K.Kind.NOT_TERMINATED
        assert (c.iterative_invocations, c.fallback_invocations) == (1, 0)
        c = K.KernelCounters()
        crawl = off(U, dx=40.0, dz=0.01)
        ri = K.closest_iterative(U, crawl, p)
        rh = K.closest_hybrid(U, crawl, p, c)
        assert rh.kind != K.Kind.NOT_TERMINATED
        if ri.kind == K.Kind.NOT_TERMINATED:
            assert c.fallback_invocations == 1
            assert rh.distance == pytest.approx(K.closest_comparison(U, crawl, p).distance, abs=1e-12)
        assert c.comparison_invocations == c.fallback_invocations

    def test_never_not_terminated(self):
        rng = np.random.default_rng(5)
        res = K.hybrid_batch(rng.normal(size=(500, 3, 3)), rng.normal(size=(500, 3, 3)), K.KernelParams(), None, 1e-2)
        assert not (res.kind == K.Kind.NOT_TERMINATED).any()

    def test_allow_fallback_false_keeps_open_pairs(self):
        rng = np.random.default_rng(6)
        A, B = rng.normal(size=(300, 3, 3)), rng.normal(size=(300, 3, 3))
        it = K.iterative_batch(A, B, K.KernelParams(), 1e-2)
        hy = K.hybrid_batch(A, B, K.KernelParams(), None, 1e-2, allow_fallback=False)
        assert np.array_equal(it.kind, hy.kind) and np.array_equal(it.distance, hy.distance)

    def test_batch_closest_positional_errors(self):
        p = K.KernelParams()
        bad = np.array([[0, 0, 0], [1, 0, 0], [2, 0, 0]], float)
        good = off(U, dz=1.0)
        # the collinear triangle against this one stays NOT_TERMINATED after the
        # default 4 sweeps (oracle-checked), so it reaches the fallback, whose
        # degenerate screen reports it positionally (RK/kernels.py:654-668)
        open_b = np.array([[0.206, 0.02, 0.383], [-0.516, -0.114, -0.337], [0.419, 0.028, -0.205]])
        assert K.closest_iterative(bad, open_b, p).kind == K.Kind.NOT_TERMINATED
        c = K.KernelCounters()
        out = K.batch_closest([(U, good), (bad, open_b), (U, good), (bad, good)], p, c)
        assert isinstance(out[0], K.DistanceResult) and isinstance(out[2], K.DistanceResult)
        assert isinstance(out[1], K.DegenerateTriangle) and "pair 1" in str(out[1])
        assert isinstance(out[3], K.DistanceResult)  # settled: the degenerate triangle never reaches the fallback
        assert out[0].distance == pytest.approx(1.0, abs=1e-9)
        assert (c.iterative_invocations, c.fallback_invocations) == (4, 0)
        with pytest.raises(K.DegenerateTriangle):
            K.closest_hybrid(bad, open_b, p)

    def test_batch_closest_equals_scalar_map(self):
        rng = np.random.default_rng(8)
        p = K.KernelParams()
        pairs = [(rng.normal(size=(3, 3)), rng.normal(size=(3, 3))) for _ in range(64)]
        for got, (a, b) in zip(K.batch_closest(pairs, p), pairs):
            want = K.closest_hybrid(a, b, p)
            assert got.kind == want.kind and got.distance == want.distance


@pytest.mark.gpu
@gpu
@pytest.mark.parametrize("pname", ["def", "bl"])
def test_dropin_bitwise_against_golden(golden_inputs, golden_ref, pname):
    from conftest import PARAM_SETS
    ref = golden_ref["float64"]
    A, B = golden_inputs["cfg0_A"], golden_inputs["cfg0_B"]
    p = K.KernelParams(**PARAM_SETS[pname])
    pre = f"cfg0_{pname}"
    c = K.KernelCounters()
    got = {"comparison": K.comparison_batch(A, B, p.epsilon), "iterative": K.iterative_batch(A, B, p, p.epsilon),
           "hybrid": K.hybrid_batch(A, B, p, c, p.epsilon)}
    for v, res in got.items():
        for col in ("kind", "distance", "point_a", "point_b", "bary_a", "bary_b"):
            assert np.array_equal(getattr(res, col), ref[f"{pre}_{v}_{col}"]), (v, col)
    assert [c.iterative_invocations, c.comparison_invocations, c.fallback_invocations] == \
        list(ref[f"{pre}_hybrid_counters"])
    cl, ba = K.closest_point_triangle_batch(golden_inputs["cpt_P"], golden_inputs["cpt_T"])
    assert np.array_equal(cl, ref["cpt_closest"]) and np.array_equal(ba, ref["cpt_bary"])
    assert np.array_equal(K.degenerate_mask(golden_inputs["degenerate_T"]), ref["degenerate_mask"])
