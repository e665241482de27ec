"""Pins of the oracle's discrete edge check (BASELINE.json cfg4; SPEC.md:379-387;
DESIGN.md R11)."""
import numpy as np

import oracle
import workloads as W


def _model(n=40, seed=0):
    robot = W.arm7(8)
    rng = np.random.default_rng(seed)
    sup = rng.uniform(-np.pi, np.pi, size=(n, 7)).astype(np.float32)
    alpha = (rng.standard_normal(n) + 0.2).astype(np.float32)  # both signs of f occur
    return robot, sup, alpha, oracle.fk(robot, sup)


def test_degenerate_edge_free_point():
    """a = b with f(a) <= 0 -> not in collision."""
    robot, sup, alpha, spos = _model()
    q = np.random.default_rng(1).uniform(-np.pi, np.pi, size=(200, 7)).astype(np.float32)
    f, _ = oracle.score(0, 5.0, oracle.fk(robot, q), spos, alpha)
    free = q[f < 0][:10]
    hit, fmax, _ = oracle.edge(robot, free, free, 64, 0, 5.0, spos, alpha)
    assert np.all(hit == 0)
    np.testing.assert_allclose(fmax, f[f < 0][:10], rtol=1e-12)


def test_endpoint_in_collision():
    """An endpoint with f > 0 puts the edge in collision."""
    robot, sup, alpha, spos = _model()
    q = np.random.default_rng(2).uniform(-np.pi, np.pi, size=(400, 7)).astype(np.float32)
    f, _ = oracle.score(0, 5.0, oracle.fk(robot, q), spos, alpha)
    bad, good = q[f > 0][:10], q[f < 0][:10]
    assert len(bad) == 10 and len(good) == 10
    hit, _, _ = oracle.edge(robot, good, bad, 64, 0, 5.0, spos, alpha)
    assert np.all(hit == 1)
    hit, _, _ = oracle.edge(robot, bad, good, 64, 0, 5.0, spos, alpha)
    assert np.all(hit == 1)


def test_edge_is_or_of_interpolated_scores():
    """in_collision = OR_k f(q_k) > 0 with q_k = a + k/63 (b - a). Endpoints are chosen so
    that every q_k is exactly representable (b - a = 63/64 per joint), so the oracle's
    FK + score on the fp32 points must reproduce its edge scores."""
    robot, sup, alpha, spos = _model()
    rng = np.random.default_rng(3)
    qa = (np.round(rng.uniform(-2, 2, size=(30, 7)) * 64) / 64).astype(np.float32)
    qb = (qa + np.float32(63 / 64)).astype(np.float32)
    hit, fmax, fall = oracle.edge(robot, qa, qb, 64, 0, 5.0, spos, alpha, with_all=True)
    for e in range(30):
        pts = (qa[e][None, :] + (np.arange(64)[:, None] / 64.0)).astype(np.float32)
        f, _ = oracle.score(0, 5.0, oracle.fk(robot, pts), spos, alpha)
        np.testing.assert_allclose(fall[e], f, rtol=1e-13, atol=1e-13)
        assert hit[e] == int(np.any(f > 0))
        assert fmax[e] == np.max(f)
