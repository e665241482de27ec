"""Pins of the oracle's Algorithm 1 against hand-derived traces
(tests/golden/train_cases.json), Claim 2 and the constraints of
Eq. 5."""
import json
import os

import numpy as np
import pytest

import oracle
import workloads as W

GOLD = os.path.join(os.path.dirname(__file__), "golden")
CASES = json.load(open(os.path.join(GOLD, "train_cases.json")))["cases"]


@pytest.mark.parametrize("case", CASES, ids=lambda c: c["name"])
def test_hand_derived_traces(case):
    K = np.array(case["K"], dtype=np.float64)
    r = oracle.train(K, np.array(case["y"], dtype=np.int8), case["beta"], case["iter_max"], case["s_max"],
                     alpha0=case.get("alpha0"), F0=case.get("F0"))
    np.testing.assert_allclose(r["alpha"], case["alpha"], atol=1e-12)
    np.testing.assert_allclose(r["F"], case["F"], atol=1e-12)
    assert r["trace"].tolist() == case["trace"]
    assert (r["iterations"], r["n_add"], r["n_remove"]) == (case["iterations"], case["n_add"], case["n_remove"])
    assert r["converged"] == case["converged"]
    assert r["support"].tolist() == case["support"]


def _dataset(n, seed, dof=3):
    """Small PD problem: distinct 3-DOF configurations labelled by a capsule scene."""
    rng = np.random.default_rng(seed)
    robot = W.arm3(np.random.default_rng(1))
    q = rng.uniform(-np.pi, np.pi, size=(n, 3)).astype(np.float32)
    pos = oracle.fk(robot, q)
    cubes = W.random_cubes(rng, n=3, keep_out=0.1)
    y = W.capsule_aabb_labels(W.chain_points(pos[:, :3]), cubes, 0.05)
    if np.all(y == y[0]):
        y[: n // 3] = -y[0]
    K = oracle.gram(oracle.GAUSSIAN, 10.0, pos)
    return K, y


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_claim2_loss_decrease_and_invariants(seed):
    """Every add step with min margin <= 0 lowers L(alpha) = 1/2 a'Ka - y'Ba by at least 1/2
    (PAPER.md:260 with K_ii = 1); after an add the chosen point's margin is b_i; y_i alpha_i >= 0
    (PAPER.md:189); F = K alpha; a removal keeps the removed point's margin positive;
    convergence means every margin is positive (Claim 2)."""
    K, y = _dataset(60, seed)
    beta = 1.5
    b = np.where(y > 0, beta, 1.0)
    r = oracle.train(K, y, beta, iter_max=5000, with_loss=True)
    L = r["loss_trace"]
    assert L[0] == 0.0
    # replay the trace independently in numpy to check the per-step claims
    alpha = np.zeros(len(y))
    for t, code in enumerate(r["trace"]):
        if code >= 0:
            i = code
            F = K @ alpha
            margin_before = y[i] * F[i]
            assert margin_before <= 0
            # Alg. 1 line "i = argmin y F": no margin is smaller (up to the
            # rounding difference between the oracle's incremental F and K @ alpha)
            assert margin_before <= (y * F).min() + 1e-12
            alpha[i] += b[i] * y[i] - F[i]
            assert y[i] * (K @ alpha)[i] == pytest.approx(b[i], abs=1e-9)
            assert L[t + 1] - L[t] <= -0.5 + 1e-9
            assert L[t + 1] - L[t] == pytest.approx(-0.5 * (b[i] - margin_before) ** 2, abs=1e-8)
        else:
            i = -code - 1
            # removal candidate: argmax over alpha != 0 of y (F - alpha), > 0
            F = K @ alpha
            red = np.where(alpha != 0, y * (F - alpha), -np.inf)
            assert alpha[i] != 0 and red[i] >= red.max() - 1e-12 and red[i] > 0
            alpha[i] = 0.0
            assert y[i] * (K @ alpha)[i] > -1e-12
        assert np.all(y * alpha >= 0)
    np.testing.assert_allclose(alpha, r["alpha"], atol=1e-9)
    np.testing.assert_allclose(r["F"], K @ r["alpha"], atol=1e-9)
    assert r["loss_trace"][-1] == pytest.approx(oracle.loss(K, y, beta, r["alpha"]))
    L_direct = 0.5 * r["alpha"] @ K @ r["alpha"] - (y * b) @ r["alpha"]
    assert r["loss_trace"][-1] == pytest.approx(L_direct, rel=1e-12, abs=1e-12)
    if r["converged"]:
        assert np.all(y * r["F"] > 0)
        # Claim 2's loose step bound on a well-conditioned PD problem
        bound = (y * b) @ np.linalg.solve(K, y * b)
        assert r["n_add"] <= bound + 1e-9
    assert np.array_equal(r["support"], np.flatnonzero(r["alpha"] != 0))


def test_xor_dataset_terminates():
    """an XOR-style 2-DOF labelling, not separable in joint space, still
    terminates with every margin positive (Claim 2, PD Gram)."""
    robot = W.planar_2link()
    rng = np.random.default_rng(11)
    q = rng.uniform(-np.pi, np.pi, size=(80, 2)).astype(np.float32)
    y = np.where((q[:, 0] > 0) ^ (q[:, 1] > 0), 1, -1).astype(np.int8)
    K = oracle.gram(oracle.RQ, 2.0, oracle.fk(robot, q))
    r = oracle.train(K, y, 1.0, iter_max=100000)
    assert r["converged"]
    assert np.all(y * r["F"] > 0)


def test_first_step_is_index_zero():
    """At iteration 1 all margins are 0 (cold start), so the lowest index is chosen (R9)
    and alpha_0 = b_0 y_0 (Eq. 6)."""
    K, y = _dataset(40, 5)
    r = oracle.train(K, y, 2.0, iter_max=1)
    assert r["trace"].tolist() == [0]
    assert r["alpha"][0] == (2.0 if y[0] > 0 else -1.0)


def test_beta_biases_toward_collision():
    """beta >= 1 biases the model toward C_obs: on the training set, the
    number of points predicted in collision does not drop as beta grows."""
    K, y = _dataset(80, 9)
    pos_pred = []
    for beta in (1.0, 2.0, 5.0):
        r = oracle.train(K, y, beta, iter_max=20000)
        pos_pred.append(int(np.sum(r["F"] > 0)))
    assert pos_pred[0] <= pos_pred[1] <= pos_pred[2]
