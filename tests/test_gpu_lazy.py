"""fastron_train_lazy (Algorithm 1 with lazily computed K columns)
must reproduce fastron_train on the full Gram exactly: the columns are computed with the
same term function, so the traces, alpha and F are bit-identical; and both match the
oracle's Algorithm 1 on that Gram (R13)."""
import numpy as np
import pytest

import oracle
import workloads as W
from gpu_helpers import dev, require_gpu

pytestmark = pytest.mark.gpu


def _labels(robot, X, cubes, radius):
    pos = oracle.fk(robot, X)
    return W.capsule_aabb_labels(W.chain_points(pos[:, :8] if pos.shape[1] >= 8 else pos), cubes, radius)


@pytest.mark.parametrize("n,m16,kind,cache,beta,s_max", [
    (1000, False, 0, 4096, 1.0, None),
    (5000, False, 0, 4096, 1.0, None),   # cfg3 itself (a 4-CTA cluster)
    (1500, False, 1, 37, 2.0, None),     # tiny cache: most columns recomputed
    (1200, True, 0, 0, 1.0, 100),        # M = 16, no cache at all, S_max gate
])
def test_lazy_equals_full_gram(n, m16, kind, cache, beta, s_max):
    require_gpu()
    import torch
    import paper_1910_06451_b200 as fb
    wl = W.train_workload(n)
    robot = W.arm7(16) if m16 else wl.robot
    y = W.capsule_aabb_labels(W.chain_points(oracle.fk(wl.robot, wl.X)), wl.cubes, wl.radius)
    pos = fb.fastron_fk(robot, dev(wl.X))
    K = fb.fastron_gram(pos, kind, wl.gamma)
    yd = dev(y)
    full = fb.fastron_train(K, yd, beta, 6000, s_max)
    lazy = fb.fastron_train_lazy(pos, yd, kind, wl.gamma, beta, 6000, s_max, cache_cols=cache)
    torch.cuda.synchronize()
    rf, rl = fb.train_result(full["result"]), fb.train_result(lazy["result"])
    assert rf == rl
    it = rf["iterations"]
    assert np.array_equal(full["trace"].cpu().numpy()[:it], lazy["trace"].cpu().numpy()[:it])
    assert np.array_equal(full["alpha"].cpu().numpy(), lazy["alpha"].cpu().numpy())
    assert np.array_equal(full["F"].cpu().numpy(), lazy["F"].cpu().numpy())
    ns = rf["n_support"]
    assert np.array_equal(full["support_idx"].cpu().numpy()[:ns], lazy["support_idx"].cpu().numpy()[:ns])
    if n <= 1500:
        r = oracle.train(K.cpu().numpy().astype(np.float64), y, beta, 6000, s_max)
        assert r["iterations"] == it and np.array_equal(r["trace"], lazy["trace"].cpu().numpy()[:it])


def test_lazy_warm_start():
    require_gpu()
    import torch
    import paper_1910_06451_b200 as fb
    wl = W.train_workload(900)
    y = W.capsule_aabb_labels(W.chain_points(oracle.fk(wl.robot, wl.X)), wl.cubes, wl.radius)
    pos = fb.fastron_fk(wl.robot, dev(wl.X))
    K = fb.fastron_gram(pos, 0, wl.gamma)
    first = oracle.train(K.cpu().numpy().astype(np.float64), y, 1.0, 200)
    y2 = y.copy()
    y2[::5] *= -1
    a0, F0 = dev(first["alpha"], torch.float64), dev(first["F"], torch.float64)
    lazy = fb.fastron_train_lazy(pos, dev(y2), 0, wl.gamma, 1.0, 3000, alpha=a0.clone(), F=F0.clone())
    full = fb.fastron_train(K, dev(y2), 1.0, 3000, alpha=a0.clone(), F=F0.clone())
    torch.cuda.synchronize()
    assert fb.train_result(lazy["result"]) == fb.train_result(full["result"])
    assert np.array_equal(lazy["alpha"].cpu().numpy(), full["alpha"].cpu().numpy())


@pytest.mark.parametrize("M", [3, 5])
def test_lazy_odd_m_equals_full_gram(M):
    """Odd M: the padded control point contributes exactly 0 to a computed column, as it
    does in fastron_gram (same values, same trace)."""
    require_gpu()
    import torch
    import paper_1910_06451_b200 as fb
    wl = W.train_workload(700)
    rng = np.random.default_rng(M)
    robot = W.make_robot("m%d" % M, wl.robot.dh, rng.integers(1, 8, size=M), rng.uniform(-0.1, 0.1, size=(M, 3)))
    y = W.capsule_aabb_labels(W.chain_points(oracle.fk(wl.robot, wl.X)), wl.cubes, wl.radius)
    pos = fb.fastron_fk(robot, dev(wl.X))
    K = fb.fastron_gram(pos, 0, wl.gamma)
    assert np.all(np.diag(K.cpu().numpy()) == 1.0)
    full = fb.fastron_train(K, dev(y), 1.0, 3000)
    lazy = fb.fastron_train_lazy(pos, dev(y), 0, wl.gamma, 1.0, 3000, cache_cols=64)
    torch.cuda.synchronize()
    assert fb.train_result(full["result"]) == fb.train_result(lazy["result"])
    assert np.array_equal(full["alpha"].cpu().numpy(), lazy["alpha"].cpu().numpy())
    assert np.array_equal(full["F"].cpu().numpy(), lazy["F"].cpu().numpy())


def _same(full, lazy):
    import paper_1910_06451_b200 as fb
    rf, rl = fb.train_result(full["result"]), fb.train_result(lazy["result"])
    assert rf == rl
    it = rf["iterations"]
    assert np.array_equal(full["trace"].cpu().numpy()[:it], lazy["trace"].cpu().numpy()[:it])
    assert np.array_equal(full["alpha"].cpu().numpy(), lazy["alpha"].cpu().numpy())
    assert np.array_equal(full["F"].cpu().numpy(), lazy["F"].cpu().numpy())
    ns = rf["n_support"]
    assert np.array_equal(full["support_idx"].cpu().numpy()[:ns], lazy["support_idx"].cpu().numpy()[:ns])
    return rf


def test_lazy_cfg5_scale_equals_full_gram():
    """f1 at cfg5 scale (N = 20,000, M = 16): the 16-CTA slices of
    1,250 points exceed the shared-memory budget, so the point planes live in an
    L2-resident part of the workspace; the run must equal fastron_train(fastron_gram(pos))
    bit for bit — without the 1.6 GB Gram."""
    require_gpu()
    import torch
    import paper_1910_06451_b200 as fb
    robot, X, _, moved = W.cfg5_gram_workload()
    assert X.shape[0] == 20_000 and robot.n_cp == 16
    assert fb.load_library().fastron_train_lazy_max_n(16) >= 20_000
    y = W.capsule_aabb_labels(W.chain_points(oracle.fk(W.arm7(8), X)), moved, 0.05)
    pos = fb.fastron_fk(robot, dev(X))
    yd = dev(y)
    lazy = fb.fastron_train_lazy(pos, yd, 0, 5.0, 1.0, 20_000, cache_cols=4096)
    K = fb.fastron_gram(pos, 0, 5.0)
    full = fb.fastron_train(K, yd, 1.0, 20_000)
    torch.cuda.synchronize()
    del K
    rf = _same(full, lazy)
    assert rf["iterations"] > 1000


def test_lazy_global_planes_forced(tmp_path):
    """The global-plane instance (FASTRON_LAZY_GPTS=1, read per call) on small problems:
    odd M, RQ, a tiny cache, a warm start — equal to the shared-memory lazy run and so to
    the full-Gram run."""
    require_gpu()
    import os
    import torch
    import paper_1910_06451_b200 as fb
    wl = W.train_workload(1700)
    rng = np.random.default_rng(5)
    robot = W.make_robot("m5", wl.robot.dh, rng.integers(1, 8, size=5), rng.uniform(-0.1, 0.1, size=(5, 3)))
    y = W.capsule_aabb_labels(W.chain_points(oracle.fk(wl.robot, wl.X)), wl.cubes, wl.radius)
    pos = fb.fastron_fk(robot, dev(wl.X))
    yd = dev(y)
    for kind, cache in ((0, 4096), (1, 13)):
        ref = fb.fastron_train_lazy(pos, yd, kind, wl.gamma, 1.0, 3000, cache_cols=cache)
        # the all-L2 instance and the split one (5/6 of the slice's planes in shared memory)
        for planes in ("0", None):
            os.environ["FASTRON_LAZY_GPTS"] = "1"
            if planes is not None:
                os.environ["FASTRON_LAZY_SMEM_PLANES"] = planes
            try:
                got = fb.fastron_train_lazy(pos, yd, kind, wl.gamma, 1.0, 3000, cache_cols=cache)
            finally:
                os.environ.pop("FASTRON_LAZY_GPTS", None)
                os.environ.pop("FASTRON_LAZY_SMEM_PLANES", None)
            torch.cuda.synchronize()
            _same(ref, got)
