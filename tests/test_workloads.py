"""Host-side workload generators and the cfg3 labeller (geometry only, R12)."""
import numpy as np

import workloads as W


def _point_box_d2(p, lo, hi):
    g = np.maximum(np.maximum(lo - p, p - hi), 0.0)
    return np.sum(g * g, axis=-1)


def test_segment_box_distance_matches_dense_sampling():
    rng = np.random.default_rng(0)
    n = 3000
    p0 = rng.uniform(-1, 1, size=(n, 3))
    p1 = rng.uniform(-1, 1, size=(n, 3))
    c = rng.uniform(-0.5, 0.5, size=(n, 3))
    h = rng.uniform(0.05, 0.3, size=(n, 1))
    lo, hi = c - h, c + h
    d2 = W.segment_box_dist2(p0, p1, lo, hi)
    t = np.linspace(0, 1, 20001)
    brute = np.min(_point_box_d2(p0[:, None] + t[None, :, None] * (p1 - p0)[:, None], lo[:, None], hi[:, None]), axis=1)
    assert np.all(d2 <= brute + 1e-12)  # exact minimum never above a sampled value
    np.testing.assert_allclose(d2, brute, atol=2e-7)


def test_segment_box_special_cases():
    lo, hi = np.array([0.0, 0, 0]), np.array([1.0, 1, 1])
    # through the box
    assert W.segment_box_dist2(np.array([-1.0, 0.5, 0.5]), np.array([2.0, 0.5, 0.5]), lo, hi) == 0.0
    # parallel to the top face at height 0.3
    assert np.isclose(W.segment_box_dist2(np.array([-1.0, 0.5, 1.3]), np.array([2.0, 0.5, 1.3]), lo, hi), 0.09)
    # degenerate segment (a point) near a corner
    assert np.isclose(W.segment_box_dist2(np.array([1.1, 1.2, 1.2]), np.array([1.1, 1.2, 1.2]), lo, hi), 0.09)
    # passes a corner diagonally: closest approach of the line x=y, z=2 to corner (1,1,1)
    d2 = W.segment_box_dist2(np.array([2.0, 0.0, 2.0]), np.array([0.0, 2.0, 2.0]), lo, hi)
    assert np.isclose(d2, 1.0)


def test_labels_tangency_counts():
    cubes = np.array([[[0.0, 0, 0], [1.0, 1, 1]]])
    pts = np.array([[[-1.0, 0.5, 1.05], [2.0, 0.5, 1.05]], [[-1.0, 0.5, 1.0500001], [2.0, 0.5, 1.0500001]]])
    lab = W.capsule_aabb_labels(pts, cubes, 0.05)
    assert lab.tolist() == [1, -1]


def test_generators_deterministic_and_prefix():
    a = W.score_workload("headline", n_queries=100)
    b = W.score_workload("headline", n_queries=1000)
    assert np.array_equal(a.queries, b.queries[:100])
    assert np.array_equal(a.supports, b.supports)
    c = W.score_workload("cfg2", n_queries=10, n_supports=50)
    d = W.score_workload("cfg2", n_queries=10)
    assert np.array_equal(c.supports, d.supports[:50]) and np.array_equal(c.alpha, d.alpha[:50])
    assert a.supports.dtype == np.float32 and a.queries.dtype == np.float32
    assert np.all(np.abs(b.queries) <= np.float32(np.pi))


def test_arm_shapes_follow_readings():
    r3 = W.arm3(np.random.default_rng(1))
    assert r3.dof == 3 and r3.n_cp == 4
    assert np.all((r3.dh[:, 2] >= 0.3) & (r3.dh[:, 2] <= 0.5)) and np.all(r3.dh[:, 1] == 0)
    r7 = W.arm7(8)
    assert r7.dof == 7 and r7.n_cp == 8
    assert np.all(r7.dh[1::2, 2] == 0) and np.all(r7.dh[0::2, 2] > 0)
    assert W.arm7(16).n_cp == 16


def test_cubes_keep_out_of_base():
    cubes = W.random_cubes(np.random.default_rng(3), 50, keep_out=0.15)
    gap = np.maximum(np.maximum(cubes[:, 0], -cubes[:, 1]), 0)
    assert np.all(np.sqrt(np.sum(gap * gap, axis=1)) >= 0.15)
    side = cubes[:, 1] - cubes[:, 0]
    assert np.allclose(side, side[:, :1]) and np.all((side >= 0.1) & (side <= 0.3))
