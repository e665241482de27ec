"""Pins of the oracle's kernels, score and Gram matrix (Eq. 3,
:133-177 Eq. 4 + Claim 1, :183 the Fastron model) against worked values, closed-form
maxima, textbook special cases, hand-computed sums and the paper's claims."""
import json
import math
import os

import numpy as np
import pytest

import oracle
import workloads as W

GOLD = os.path.join(os.path.dirname(__file__), "golden")
KINDS = {"gaussian": oracle.GAUSSIAN, "rq": oracle.RQ}


def test_term_worked_values():
    g = json.load(open(os.path.join(GOLD, "kernel_values.json")))
    for t in g["terms"]:
        assert oracle.rbf_term(KINDS[t["kind"]], t["gamma"], t["d2"]) == pytest.approx(t["value"], rel=1e-15)


@pytest.mark.parametrize("kind", [oracle.GAUSSIAN, oracle.RQ])
def test_self_similarity_is_the_closed_form_maximum(kind):
    """k(x, x) = 1 exactly and 0 < k <= 1."""
    robot = W.arm7(8)
    q = np.random.default_rng(0).uniform(-np.pi, np.pi, size=(40, 7)).astype(np.float32)
    pos = oracle.fk(robot, q)
    for i in range(40):
        assert oracle.kernel_value(kind, 5.0, pos[i], pos[i]) == 1.0
        for j in range(40):
            v = oracle.kernel_value(kind, 5.0, pos[i], pos[j])
            assert 0.0 < v <= 1.0 or (kind == oracle.GAUSSIAN and v == 0.0)
            assert v == oracle.kernel_value(kind, 5.0, pos[j], pos[i])  # symmetry


@pytest.mark.parametrize("kind", [oracle.GAUSSIAN, oracle.RQ])
def test_m1_reduces_to_the_bare_rbf(kind):
    """M = 1: Eq. 4 reduces to Eq. 3 (or the Gaussian) on the single control point;
    the bare RQ of R^3 points is (1 + gamma/2 |u-v|^2)^-2 (Rasmussen & Williams, alpha=2)."""
    rng = np.random.default_rng(1)
    for _ in range(100):
        u, v, g = rng.normal(size=3), rng.normal(size=3), rng.uniform(0.1, 10)
        d2 = float(np.sum((u - v) ** 2))
        ref = math.exp(-g * d2) if kind == oracle.GAUSSIAN else 1.0 / (1.0 + 0.5 * g * d2) ** 2
        assert oracle.kernel_value(kind, g, u, v) == pytest.approx(ref, rel=1e-14)


def test_planar_hand_values():
    """Hand-computed Eq. 4 on the planar arm: x=(0,0) vs x'=(pi,0) puts the control points
    at distance 2 and 4: Gaussian(ln2) -> (2^-4 + 2^-16)/2, RQ(gamma=2) -> (1/25 + 1/289)/2."""
    g = json.load(open(os.path.join(GOLD, "kernel_values.json")))["planar"]
    robot = W.planar_2link()
    pos = oracle.fk(robot, np.array([g["x"], g["xp"]], dtype=np.float32))
    assert oracle.kernel_value(oracle.GAUSSIAN, math.log(2), pos[0], pos[1]) == pytest.approx(g["gaussian_ln2"], rel=1e-12)
    assert oracle.kernel_value(oracle.RQ, 2.0, pos[0], pos[1]) == pytest.approx(g["rq_gamma2"], rel=1e-12)


def test_fig2_ordering():
    """PAPER.md:130, :141 (Fig. 2) and SPEC.md:165: b=(0,0); p=(0,delta) moves only the
    elbow joint, g=(delta,0) only the shoulder. Joint-space RQ distances are equal, so RQ on
    joints is equal; the FK kernel rates p strictly more similar than g."""
    robot = W.planar_2link()
    delta = 0.6
    q = np.array([[0, 0], [0, delta], [delta, 0]], dtype=np.float32)
    pos = oracle.fk(robot, q)
    for kind in (oracle.GAUSSIAN, oracle.RQ):
        # joint-space kernel (M=1 "control point" = the joint vector padded to 3-D)
        jb, jp, jg = (np.array([*q[i].astype(np.float64), 0.0]) for i in range(3))
        assert oracle.kernel_value(kind, 2.0, jb, jp) == oracle.kernel_value(kind, 2.0, jb, jg)
        assert oracle.kernel_value(kind, 2.0, pos[0], pos[1]) > oracle.kernel_value(kind, 2.0, pos[0], pos[2])


def test_score_hand_sum():
    """Brute force on a tiny input: supports x'=(pi,0) with alpha=2 and
    x=(0,0) with alpha=-1, query x=(0,0): f = 2 k(x,x') - 1 = 2 (2^-4+2^-16)/2 - 1."""
    robot = W.planar_2link()
    sup = np.array([[np.pi, 0], [0, 0]], dtype=np.float32)
    spos = oracle.fk(robot, sup)
    qpos = oracle.fk(robot, np.array([[0, 0]], dtype=np.float32))
    f, lab = oracle.score(oracle.GAUSSIAN, math.log(2), qpos, spos, np.array([2.0, -1.0], dtype=np.float32))
    assert f[0] == pytest.approx(2 * (2 ** -4 + 2 ** -16) / 2 - 1, rel=1e-12)
    assert lab[0] == -1
    f, lab = oracle.score(oracle.GAUSSIAN, math.log(2), qpos, spos, np.array([2.0, 1.0], dtype=np.float32))
    assert f[0] == pytest.approx(2 * (2 ** -4 + 2 ** -16) / 2 + 1, rel=1e-12) and lab[0] == 1


def test_score_empty_and_zero_weights():
    """Empty support set or all-zero alpha -> f = 0, label -1 (R8)."""
    robot = W.arm3(np.random.default_rng(1))
    qpos = oracle.fk(robot, np.random.default_rng(2).uniform(-3, 3, size=(5, 3)).astype(np.float32))
    f, lab = oracle.score(oracle.GAUSSIAN, 10.0, qpos, np.zeros((0, 4, 3)), np.zeros(0, dtype=np.float32))
    assert np.all(f == 0) and np.all(lab == -1)
    f, lab = oracle.score(oracle.RQ, 10.0, qpos, qpos, np.zeros(5, dtype=np.float32))
    assert np.all(f == 0) and np.all(lab == -1)


def test_score_linearity_and_permutation():
    wl = W.score_workload("cfg1", n_queries=50, n_supports=60)
    qpos = oracle.fk(wl.robot, wl.queries)
    spos = oracle.fk(wl.robot, wl.supports)
    a = wl.alpha
    f1, _ = oracle.score(0, wl.gamma, qpos, spos, a)
    f2, _ = oracle.score(0, wl.gamma, qpos, spos, (2 * a).astype(np.float32))
    np.testing.assert_allclose(f2, 2 * f1, rtol=1e-13, atol=1e-15)
    perm = np.random.default_rng(0).permutation(60)
    f3, _ = oracle.score(0, wl.gamma, qpos, spos[perm], a[perm])
    np.testing.assert_allclose(f3, f1, rtol=1e-12, atol=1e-14)


@pytest.mark.parametrize("kind", [oracle.GAUSSIAN, oracle.RQ])
def test_gram_symmetry_diagonal_pd(kind):
    """Claim 1 and SPEC.md:163: 50 distinct 3-DOF configurations give a
    PD FK Gram matrix: min eigenvalue > 1e-10 * max eigenvalue; symmetric; unit diagonal."""
    robot = W.arm3(np.random.default_rng(1))
    q = np.random.default_rng(7).uniform(-np.pi, np.pi, size=(50, 3)).astype(np.float32)
    K = oracle.gram(kind, 10.0, oracle.fk(robot, q))
    assert np.array_equal(K, K.T)
    assert np.all(np.diag(K) == 1.0)
    ev = np.linalg.eigvalsh(K)
    assert ev[0] > 1e-10 * ev[-1]


def test_gram_summand_decomposition():
    """K = (1/M) sum_m K_m, K_m the Gram of control point m alone."""
    robot = W.arm7(8)
    q = np.random.default_rng(8).uniform(-np.pi, np.pi, size=(30, 7)).astype(np.float32)
    pos = oracle.fk(robot, q)
    K = oracle.gram(oracle.GAUSSIAN, 5.0, pos)
    Ks = [oracle.gram(oracle.GAUSSIAN, 5.0, pos[:, m:m + 1, :]) for m in range(8)]
    np.testing.assert_allclose(K, sum(Ks) / 8, rtol=1e-14, atol=1e-16)
    for Km in Ks:  # each summand is itself PSD
        assert np.linalg.eigvalsh(Km)[0] > -1e-12


def test_coincident_control_points_still_pd():
    """Claim 1 / Fig. 3: configurations that share the elbow position
    but differ at the tip make K_1 singular yet K PD."""
    robot = W.planar_2link()
    q = np.array([[0.3, 0.0], [0.3, 1.0], [0.3, -1.0], [1.2, 0.5]], dtype=np.float32)
    pos = oracle.fk(robot, q)
    K1 = oracle.gram(oracle.RQ, 2.0, pos[:, :1])
    K = oracle.gram(oracle.RQ, 2.0, pos)
    assert np.linalg.matrix_rank(K1, tol=1e-10) < 4
    assert np.linalg.eigvalsh(K)[0] > 1e-6


# ---- joint-space RBF ("Fastron RBF" baseline, Table I) ----

def test_joint_kernel_worked_values():
    """Eq. 3 on raw joint vectors: ||x - x'||^2 = 1 with gamma = 2 -> (1 + 1)^-2 = 0.25
    (SPEC.md:130); Gaussian gamma = ln 2 -> 0.5; identical vectors -> 1."""
    x = np.zeros(7, np.float32)
    xp = np.zeros(7, np.float32)
    xp[3] = 1.0
    assert oracle.joint_kernel(oracle.RQ, 2.0, x, xp) == 0.25
    assert oracle.joint_kernel(oracle.GAUSSIAN, math.log(2), x, xp) == pytest.approx(0.5, rel=1e-15)
    xp2 = np.array([0.5, 0.5, 0.5, 0.5, 0, 0, 0], np.float32)  # squared distance 1
    assert oracle.joint_kernel(oracle.RQ, 2.0, x, xp2) == 0.25
    assert oracle.joint_kernel(oracle.RQ, 5.0, xp2, xp2) == 1.0


def test_joint_score_and_gram_properties():
    """Brute force on a tiny input, symmetry, unit diagonal and PD (the RQ kernel is PD,
    PAPER.md:123)."""
    rng = np.random.default_rng(3)
    X = rng.uniform(-np.pi, np.pi, size=(40, 7)).astype(np.float32)
    a = rng.standard_normal(40).astype(np.float32)
    K = oracle.gram_joint(oracle.RQ, 1.0, X)
    assert np.array_equal(K, K.T) and np.all(np.diag(K) == 1.0)
    assert np.linalg.eigvalsh(K)[0] > 1e-10 * np.linalg.eigvalsh(K)[-1]
    f, lab = oracle.score_joint(oracle.RQ, 1.0, X[:5], X, a)
    np.testing.assert_allclose(f, K[:5] @ a.astype(np.float64), rtol=1e-12, atol=1e-13)
    assert np.array_equal(lab, np.where(f > 0, 1, -1))


def test_near_base_points_floor_the_fk_kernel():
    """Why SURVEY §8(f) f4 (certified early exit / tile culling) cannot pay on these arms
    (DESIGN.md §11): the first control points stay within ~0.45 m of each other for every
    configuration, so Eq. 4's mean over M never drops below ~0.14 at gamma = 5, and the
    remainder of a partial score is bounded only by ~0.14 * sum |alpha_rest|."""
    robot = W.arm7(8)
    rng = np.random.default_rng(0)
    pos = oracle.fk(robot, W.uniform_configs(rng, 400, 7))
    i, j = rng.integers(0, 400, 5000), rng.integers(0, 400, 5000)
    k = np.array([oracle.kernel_value(oracle.GAUSSIAN, 5.0, pos[a], pos[b]) for a, b in zip(i, j)])
    assert k.min() > 0.13
    # the two base-most points alone give the bound: (1/M) * sum_m exp(-gamma * dmax_m^2)
    d = np.linalg.norm(pos[i][:, :2] - pos[j][:, :2], axis=-1)
    assert d.max() < 0.5
