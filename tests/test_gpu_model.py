"""FastronModel (the host sequencing of the ABI calls, README usage): fit = Gram +
Algorithm 1, query = FK + score, checked against the oracle on the same data."""
import numpy as np
import pytest

import oracle
import workloads as W
from c4 import assert_stats, score_stats
from gpu_helpers import dev, require_gpu

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("kind", [0, 1])
def test_fit_then_query_matches_oracle(kind):
    require_gpu()
    import torch
    from paper_1910_06451_b200.model import FastronModel
    tw = W.train_workload(1200)
    y = W.capsule_aabb_labels(W.chain_points(oracle.fk(tw.robot, tw.X)), tw.cubes, tw.radius)
    m = FastronModel(tw.robot, kind=kind, gamma=tw.gamma, iter_max=4000)
    res = m.fit(dev(tw.X), dev(y))
    assert res["n_support"] == len(m.supports) > 0
    # the oracle's Algorithm 1 on the GPU Gram picks the same support set
    pos = __import__("paper_1910_06451_b200").fastron_fk(tw.robot, dev(tw.X))
    K = __import__("paper_1910_06451_b200").fastron_gram(pos, kind, tw.gamma).cpu().numpy().astype(np.float64)
    r = oracle.train(K, y, 1.0, 4000)
    assert np.array_equal(r["support"], np.flatnonzero(r["alpha"] != 0))
    sup_X = m.supports.cpu().numpy()
    assert np.array_equal(sup_X, tw.X[r["support"]])
    # queries: scores against the model's support set and (fp32) weights
    q = W.uniform_configs(np.random.default_rng(77), 20_000, 7)
    s, l = m.query(dev(q))
    torch.cuda.synchronize()
    a32 = m.alpha.float().cpu().numpy()
    qp, sp = oracle.fk(tw.robot, q), oracle.fk(tw.robot, sup_X)
    f, _ = oracle.score(kind, tw.gamma, qp, sp, a32)
    # A trained alpha has large entries of both signs (Algorithm 1 never shrinks them), so f
    # is a cancelling sum: fp32 positions and fp32 terms perturb it in proportion to its
    # condition sum_i |alpha_i| k_i, not to |f| ("trained models"). R16 is the
    # pass criterion on the non-cancelling queries (kappa = condition / |f| <= 1e4: the sum
    # loses at most 4 of fp32's 7 digits); the rest are counted and reported. Labels must
    # agree wherever |f_ref| > 1e-4, on every query (the north-star label rule).
    cond, _ = oracle.score(kind, tw.gamma, qp, sp, np.abs(a32))
    sg = s.cpu().numpy().astype(np.float64)
    kappa = cond / np.maximum(np.abs(f), 1e-300)
    ok = kappa <= 1e4
    st = score_stats(sg[ok], f[ok])
    assert ok.sum() > 1000, f"only {ok.sum()} non-cancelling queries"
    assert_stats(st, f"trained model kind={kind}, non-cancelling queries")
    lab = l.cpu().numpy()
    sure = np.abs(f) > 1e-4
    assert np.array_equal(lab[sure], np.where(f[sure] > 0, 1, -1))
    print(f"kind={kind}: {ok.sum()} non-cancelling queries {st}; {np.sum(~ok)} with kappa > 1e4 "
          f"(max err there {np.max(np.abs(sg - f)[~ok]) if (~ok).any() else 0:.2e}); max |alpha| {np.abs(a32).max():.3g}")
    # the training set is classified by its own margins' signs where they are certain
    s_tr, _ = m.query(dev(tw.X))
    F = r["F"]
    sure = np.abs(F) > 1e-3
    assert np.array_equal(np.sign(s_tr.cpu().numpy()[sure]), np.sign(F[sure]))


def test_save_load_round_trip(tmp_path):
    """Checkpoint / resume (loadPreviousModel): a saved and re-loaded model
    scores identically, and continues with update() from the loaded weights."""
    require_gpu()
    import torch
    from paper_1910_06451_b200.model import FastronModel
    tw = W.train_workload(600)
    y = W.capsule_aabb_labels(W.chain_points(oracle.fk(tw.robot, tw.X)), tw.cubes, tw.radius)
    m = FastronModel(tw.robot, kind=0, gamma=tw.gamma, iter_max=2000)
    m.fit(dev(tw.X), dev(y))
    path = str(tmp_path / "fastron.pt")
    m.save(path)
    m2 = FastronModel(tw.robot)
    m2.load(path)
    q = dev(W.uniform_configs(np.random.default_rng(3), 5000, 7))
    s1, l1 = m.query(q)
    s2, l2 = m2.query(q)
    torch.cuda.synchronize()
    assert torch.equal(s1, s2) and torch.equal(l1, l2)
    assert torch.equal(m.alpha, m2.alpha) and m2.kind == 0 and m2.gamma == tw.gamma
    with pytest.raises(ValueError):
        FastronModel(W.arm7(16)).load(path)


def test_query_graph_matches_query():
    """A captured fixed-size query (CUDA graph replay) returns the same scores and labels as
    the launch-by-launch query, for successive different inputs."""
    require_gpu()
    import torch
    from paper_1910_06451_b200.model import FastronModel
    tw = W.train_workload(500)
    y = W.capsule_aabb_labels(W.chain_points(oracle.fk(tw.robot, tw.X)), tw.cubes, tw.radius)
    m = FastronModel(tw.robot, kind=0, gamma=tw.gamma, iter_max=1000)
    m.fit(dev(tw.X), dev(y))
    for nq in (1, 32, 1000):
        run = m.query_graph(nq)
        for seed in (1, 2):
            q = dev(W.uniform_configs(np.random.default_rng(seed), nq, 7))
            s_ref, l_ref = m.query(q)
            s, l = run(q)
            torch.cuda.synchronize()
            assert torch.equal(s, s_ref) and torch.equal(l, l_ref)
