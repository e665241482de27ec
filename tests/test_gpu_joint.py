"""GPU parity of the joint-space RBF kernel of the "Fastron RBF" baseline
(fastron_score_joint / fastron_gram_joint; Table I) against the
oracle, and Algorithm 1 on its Gram (the update rule is kernel-agnostic)."""
import numpy as np
import pytest

import oracle
import workloads as W
from gpu_helpers import assert_score_parity, dev, require_gpu

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("kind,dof", [(1, 7), (0, 7), (1, 3), (1, 2), (0, 16), (1, 1)])
def test_joint_score_parity(kind, dof):
    require_gpu()
    import torch
    import paper_1910_06451_b200 as fb
    rng = np.random.default_rng(dof + 10 * kind)
    s = rng.uniform(-np.pi, np.pi, size=(1537, dof)).astype(np.float32)
    a = rng.standard_normal(1537).astype(np.float32)
    q = rng.uniform(-np.pi, np.pi, size=(20_001, dof)).astype(np.float32)
    gamma = 0.7 / dof
    sc, lb = fb.fastron_score_joint(dev(q), dev(s), dev(a), kind, gamma)
    torch.cuda.synchronize()
    f, _ = oracle.score_joint(kind, gamma, q, s, a)
    assert_score_parity(sc.cpu().numpy(), f, lb.cpu().numpy(), what=f"joint kind={kind} dof={dof}")


@pytest.mark.parametrize("nq", [33, 77, 128, 129])
def test_joint_score_mid_batches(nq):
    """33..128 queries take the one-query-per-thread instance; 20k supports give > 16
    splits, so the grouped finalize sums them."""
    require_gpu()
    import torch
    import paper_1910_06451_b200 as fb
    rng = np.random.default_rng(nq)
    s = rng.uniform(-np.pi, np.pi, size=(20_000, 7)).astype(np.float32)
    a = rng.standard_normal(20_000).astype(np.float32)
    q = rng.uniform(-np.pi, np.pi, size=(nq, 7)).astype(np.float32)
    sc, lb = fb.fastron_score_joint(dev(q), dev(s), dev(a), 1, 0.1)
    torch.cuda.synchronize()
    f, _ = oracle.score_joint(1, 0.1, q, s, a)
    assert_score_parity(sc.cpu().numpy(), f, lb.cpu().numpy(), what=f"joint nq={nq}")


def test_joint_gram_parity_and_train():
    require_gpu()
    import torch
    import paper_1910_06451_b200 as fb
    wl = W.train_workload(700)
    pos = oracle.fk(wl.robot, wl.X)
    y = W.capsule_aabb_labels(W.chain_points(pos), wl.cubes, wl.radius)
    gamma = 0.3
    K = fb.fastron_gram_joint(dev(wl.X), 1, gamma)
    torch.cuda.synchronize()
    Kg = K.cpu().numpy()
    assert np.array_equal(Kg, Kg.T) and np.all(np.diag(Kg) == 1.0)
    Kr = oracle.gram_joint(1, gamma, wl.X)
    assert_score_parity(Kg.ravel(), Kr.ravel(), what="joint gram")
    # the score with alpha = e_i reproduces row i of the Gram bit for bit
    for i in (0, 5, 699):
        a = torch.zeros(700, device="cuda")
        a[i] = 1.0
        sc, _ = fb.fastron_score_joint(dev(wl.X), dev(wl.X), a, 1, gamma)
        torch.cuda.synchronize()
        assert np.array_equal(sc.cpu().numpy(), Kg[i])
    # Algorithm 1 on the joint-space Gram: trace-exact vs the oracle on the same K (R13)
    out = fb.fastron_train(K, dev(y), 1.0, 5000)
    torch.cuda.synchronize()
    res = fb.train_result(out["result"])
    r = oracle.train(Kg.astype(np.float64), y, 1.0, 5000)
    assert res["iterations"] == r["iterations"] and res["n_support"] == r["n_support"]
    assert np.array_equal(out["trace"].cpu().numpy()[:res["iterations"]], r["trace"])
    np.testing.assert_allclose(out["alpha"].cpu().numpy(), r["alpha"], atol=1e-9 * max(1, np.abs(r["alpha"]).max()))


def test_fig2_joint_vs_fk_on_gpu():
    """PAPER.md:141 (Fig. 2): for the planar arm, the joint-space kernel rates b~p and b~g
    equally while the FK kernel prefers p (the elbow-only motion)."""
    require_gpu()
    import torch
    import paper_1910_06451_b200 as fb
    robot = W.planar_2link()
    q = np.array([[0, 0], [0, 0.6], [0.6, 0]], dtype=np.float32)
    Kj = fb.fastron_gram_joint(dev(q), 1, 2.0)
    Kf = fb.fastron_gram(fb.fastron_fk(robot, dev(q)), 1, 2.0)
    torch.cuda.synchronize()
    Kj, Kf = Kj.cpu().numpy(), Kf.cpu().numpy()
    assert Kj[0, 1] == Kj[0, 2]
    assert Kf[0, 1] > Kf[0, 2]
