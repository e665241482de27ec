"""Randomised parity sweep over the ABI's parameter space (seeded): robots with 1..16
joints, arbitrary twists and 1..32 control points on random frames, both term shapes,
gamma over two decades, support and query counts across tile and batch boundaries
(including the small-batch kernel), leading dimensions above the row length; scores,
Gram and edge checks against the oracle. Extreme-size tests found two bugs this way
(DESIGN.md §11)."""
import numpy as np
import pytest

import oracle
import workloads as W
from gpu_helpers import assert_score_parity, dev, require_gpu

pytestmark = pytest.mark.gpu


def _robot(rng):
    D = int(rng.integers(1, 17))
    M = int(rng.integers(1, 33))
    dh = np.stack([rng.uniform(-1, 1, D), rng.uniform(-0.3, 0.3, D), rng.uniform(-0.4, 0.4, D),
                   rng.uniform(-np.pi, np.pi, D)], axis=1)
    base = np.eye(3, 4)
    if rng.random() < 0.5:
        base[:, 3] = rng.uniform(-0.2, 0.2, 3)
    return W.make_robot("fuzz", dh, rng.integers(0, D + 1, size=M), rng.uniform(-0.15, 0.15, size=(M, 3)), base=base)


@pytest.mark.parametrize("seed", range(40))
def test_score_fuzz(seed):
    require_gpu()
    import torch
    import paper_1910_06451_b200 as fb
    rng = np.random.default_rng(1000 + seed)
    robot = _robot(rng)
    kind = int(rng.integers(0, 2))
    gamma = float(np.exp(rng.uniform(np.log(0.5), np.log(20.0))))
    ns = int(rng.choice([0, 1, 17, 64, 65, 300, 1999]))
    nq = int(rng.choice([1, 3, 32, 33, 511, 513, 2500]))
    D = robot.dh.shape[0]
    sup = rng.uniform(-np.pi, np.pi, size=(ns, D)).astype(np.float32)
    alpha = rng.standard_normal(ns).astype(np.float32)
    q = rng.uniform(-np.pi, np.pi, size=(nq, D + 3)).astype(np.float32)  # ldq = D + 3
    qd = dev(q)[:, :D]
    spos = fb.fastron_fk(robot, dev(sup)) if ns else torch.zeros((robot.n_cp, 0, 4), device="cuda")
    qpos_full = torch.full((robot.n_cp, nq + 5, 4), 7.0, device="cuda")  # ldpos = nq + 5
    fb.fastron_fk(robot, qd, pos=qpos_full[:, :nq])
    s, l = fb.fastron_score(qpos_full[:, :nq], spos, dev(alpha), kind, gamma)
    torch.cuda.synchronize()
    ref, _ = oracle.score(kind, gamma, oracle.fk(robot, np.ascontiguousarray(q[:, :D])),
                          oracle.fk(robot, sup) if ns else np.zeros((0, robot.n_cp, 3)), alpha)
    assert_score_parity(s.cpu().numpy(), ref, l.cpu().numpy(),
                        what=f"fuzz seed={seed} D={D} M={robot.n_cp} kind={kind} ns={ns} nq={nq}")


@pytest.mark.parametrize("seed", range(20))
def test_gram_and_edges_fuzz(seed):
    require_gpu()
    import torch
    import paper_1910_06451_b200 as fb
    rng = np.random.default_rng(2000 + seed)
    robot = _robot(rng)
    kind = int(rng.integers(0, 2))
    gamma = float(np.exp(rng.uniform(np.log(0.5), np.log(20.0))))
    D = robot.dh.shape[0]
    n = int(rng.choice([1, 2, 63, 129, 257]))
    X = rng.uniform(-np.pi, np.pi, size=(n, D)).astype(np.float32)
    K = fb.fastron_gram(fb.fastron_fk(robot, dev(X)), kind, gamma)
    torch.cuda.synchronize()
    Kg = K.cpu().numpy()
    assert np.array_equal(Kg, Kg.T) and np.all(np.diag(Kg) == 1.0)
    Kr = oracle.gram(kind, gamma, oracle.fk(robot, X))
    assert_score_parity(Kg.ravel(), Kr.ravel(), what=f"gram fuzz seed={seed} D={D} M={robot.n_cp} n={n}")
    # edges against the same supports
    ne, ni = int(rng.integers(1, 80)), int(rng.choice([1, 2, 31, 64, 70]))
    qa = rng.uniform(-np.pi, np.pi, size=(ne, D)).astype(np.float32)
    qb = rng.uniform(-np.pi, np.pi, size=(ne, D)).astype(np.float32)
    alpha = rng.standard_normal(n).astype(np.float32) + 0.1
    spos = fb.fastron_fk(robot, dev(X))
    hit, _ = fb.fastron_edge_check(robot, dev(qa), dev(qb), ni, spos, dev(alpha), kind, gamma)
    torch.cuda.synchronize()
    ref_hit, fmax = oracle.edge(robot, qa, qb, ni, kind, gamma, oracle.fk(robot, X), alpha)[:2]
    sure = np.abs(fmax) > 1e-4
    assert np.array_equal(hit.cpu().numpy()[sure], ref_hit[sure])


@pytest.mark.parametrize("seed", range(16))
def test_train_fuzz(seed):
    """Algorithm 1 on random small problems: the GPU trace equals the oracle's on the same
    fp32 Gram (P-exact), with random beta, S_max, iter_max and labels; the lazy mode
    equals the full-Gram run."""
    require_gpu()
    import torch
    import paper_1910_06451_b200 as fb
    rng = np.random.default_rng(3000 + seed)
    robot = _robot(rng)
    if robot.n_cp > 16:  # the lazy mode takes n_cp <= 16
        robot = W.make_robot("fuzz16", robot.dh, robot.cp_frame[:16], robot.cp_offset[:16], base=robot.base)
    kind = int(rng.integers(0, 2))
    gamma = float(np.exp(rng.uniform(np.log(0.5), np.log(20.0))))
    D = robot.dh.shape[0]
    n = int(rng.integers(1, 400))
    X = rng.uniform(-np.pi, np.pi, size=(n, D)).astype(np.float32)
    y = np.where(rng.random(n) < rng.uniform(0.2, 0.8), 1, -1).astype(np.int8)
    beta = float(rng.uniform(1.0, 3.0))
    iter_max = int(rng.integers(0, 3000))
    s_max = int(rng.integers(1, n + 1)) if rng.random() < 0.3 else None
    pos = fb.fastron_fk(robot, dev(X))
    K = fb.fastron_gram(pos, kind, gamma)
    out = fb.fastron_train(K, dev(y), beta, iter_max, s_max)
    lazy = fb.fastron_train_lazy(pos, dev(y), kind, gamma, beta, iter_max, s_max, cache_cols=int(rng.integers(0, n + 1)))
    torch.cuda.synchronize()
    res = fb.train_result(out["result"])
    r = oracle.train(K.cpu().numpy().astype(np.float64), y, beta, iter_max, s_max)
    it = res["iterations"]
    assert it == r["iterations"] and res["n_support"] == len(r["support"])
    assert np.array_equal(out["trace"].cpu().numpy()[:it], r["trace"])
    assert np.abs(out["alpha"].cpu().numpy() - r["alpha"]).max() <= 1e-9 * max(1.0, np.abs(r["alpha"]).max())
    assert fb.train_result(lazy["result"]) == res
    assert np.array_equal(lazy["alpha"].cpu().numpy(), out["alpha"].cpu().numpy())
