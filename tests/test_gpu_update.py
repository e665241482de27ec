"""The model-update cycle (PAPER.md:272 two-stage active learning + warm-started
Algorithm 1, :219): GPU sampler, GPU geometric labeller and the composed cycle against
independent references (numpy formulas, the workload labeller, the oracle's Alg. 1)."""
import numpy as np
import pytest

import oracle
import workloads as W
from gpu_helpers import dev, positions_np, require_gpu

pytestmark = pytest.mark.gpu
CHAIN8 = [-1, 0, 1, 2, 3, 4, 5, 6, 7]  # base -> O_1 .. O_7 -> EE (R4, R12)


def test_label_capsules_matches_workload_labeller():
    require_gpu()
    import torch
    import paper_1910_06451_b200 as fb
    wl = W.train_workload()
    pos = fb.fastron_fk(wl.robot, dev(wl.X))
    for seed in range(4):
        cubes = W.random_cubes(np.random.default_rng(100 + seed), n=6 + 10 * seed)
        lab = fb.fastron_label_capsules(pos, CHAIN8, cubes, wl.radius)
        torch.cuda.synchronize()
        P = W.chain_points(positions_np(pos))
        ref = W.capsule_aabb_labels(P, cubes, wl.radius)
        d2 = W.segment_box_dist2(P[:, :-1, None, :], P[:, 1:, None, :], cubes[None, None, :, 0], cubes[None, None, :, 1])
        near = np.any(np.abs(np.sqrt(d2) - wl.radius) < 1e-9, axis=(1, 2))
        bad = np.flatnonzero((lab.cpu().numpy() != ref) & ~near)
        assert bad.size == 0, bad[:10]
        assert 0 < (ref > 0).mean() < 1


def test_active_samples_formula():
    require_gpu()
    import torch
    import paper_1910_06451_b200 as fb
    rng = np.random.default_rng(0)
    S = rng.uniform(-3, 3, size=(50, 7)).astype(np.float32)
    z = rng.standard_normal((150, 7)).astype(np.float32)
    u = rng.uniform(0, 1, size=(40, 7)).astype(np.float32)
    sigma = np.full(7, 0.3, np.float32)
    lo, hi = np.full(7, -np.pi, np.float32), np.full(7, np.pi, np.float32)
    out = fb.fastron_active_samples(dev(S), 3, dev(z), dev(sigma), dev(u), dev(lo), dev(hi))
    torch.cuda.synchronize()
    near = np.clip((np.repeat(S, 3, axis=0) + (sigma * z).astype(np.float32)).astype(np.float32), lo, hi)
    uni = (lo + (u * (hi - lo).astype(np.float32)).astype(np.float32)).astype(np.float32)
    assert np.array_equal(out.cpu().numpy(), np.concatenate([near, uni]))


def test_update_cycle_is_alg1_on_the_relabelled_set():
    """fit -> move 3 cubes (R21) -> update(); the warm-started run must equal the oracle's
    Algorithm 1 from the same alpha_0 and F_0 = K alpha_0 on the GPU Gram (R13)."""
    require_gpu()
    import torch
    import paper_1910_06451_b200 as fb
    from paper_1910_06451_b200.model import CapsuleScene, FastronModel
    wl = W.train_workload(1500)
    X = dev(wl.X)
    y = fb.fastron_label_capsules(fb.fastron_fk(wl.robot, X), CHAIN8, wl.cubes, wl.radius)
    model = FastronModel(wl.robot, 0, wl.gamma, 1.0, 4000)
    model.fit(X, y)
    ns = model.supports.shape[0]
    moved = wl.cubes.copy()
    rng = np.random.default_rng(7)
    for j in rng.choice(len(moved), 3, replace=False):
        v = rng.standard_normal(3)
        moved[j] += 0.1 * v / np.linalg.norm(v)
    z = dev(rng.standard_normal((2 * ns, 7)).astype(np.float32))
    u = dev(rng.uniform(0, 1, (800, 7)).astype(np.float32))
    sigma = dev(np.full(7, 0.05 * 2 * np.pi, np.float32))
    lo, hi = dev(np.full(7, -np.pi, np.float32)), dev(np.full(7, np.pi, np.float32))
    res, Xn, yn, a0 = model.update(CapsuleScene(np.array(CHAIN8), moved, wl.radius), z, u, sigma, lo, hi, 2)
    torch.cuda.synchronize()
    assert Xn.shape[0] == 3 * ns + 800
    K = fb.fastron_gram(fb.fastron_fk(wl.robot, Xn), 0, wl.gamma)
    F0 = fb.fastron_kernel_matvec(K, a0)
    torch.cuda.synchronize()
    Kh = K.cpu().numpy().astype(np.float64)
    np.testing.assert_allclose(F0.cpu().numpy(), Kh @ a0.cpu().numpy(), rtol=1e-12, atol=1e-12)
    r = oracle.train(Kh, yn.cpu().numpy(), 1.0, 4000, alpha0=a0.cpu().numpy(), F0=F0.cpu().numpy())
    assert res["iterations"] == r["iterations"] and res["n_support"] == r["n_support"]
    assert res["converged"] == r["converged"]
    assert np.array_equal(model.alpha.cpu().numpy(), r["alpha"][r["support"]])
    # the updated model answers queries with the new weights
    s, l = model.query(dev(wl.X[:1000]))
    torch.cuda.synchronize()
    assert np.all(np.isfinite(s.cpu().numpy()))


@pytest.mark.parametrize("M", [5, 8, 16])
@pytest.mark.parametrize("kind", [W.GAUSSIAN, W.RQ])
def test_lazy_matvec_equals_gram_matvec(M, kind):
    """fastron_kernel_matvec_lazy (no Gram) equals fastron_kernel_matvec(fastron_gram(pos))
    bit for bit: same K entries (K3's term function, order and 1/M), same fp64 order."""
    require_gpu()
    import torch
    import paper_1910_06451_b200 as fb
    base = W.arm7(8)
    rng = np.random.default_rng(M + 10 * kind)
    robot = base if M == 8 else W.make_robot("m%d" % M, base.dh, rng.integers(0, 8, size=M),
                                              rng.uniform(-0.1, 0.1, size=(M, 3)))
    X = W.uniform_configs(rng, 1234, 7)
    pos = fb.fastron_fk(robot, dev(X))
    a = rng.standard_normal(1234) * (rng.uniform(size=1234) < 0.3) * 50.0  # sparse, large, both signs
    alpha = dev(a)
    F_full = fb.fastron_kernel_matvec(fb.fastron_gram(pos, kind, 5.0), alpha)
    F_lazy = fb.fastron_kernel_matvec_lazy(pos, alpha, kind, 5.0)
    torch.cuda.synchronize()
    assert torch.equal(F_full, F_lazy)


def test_lazy_update_equals_full_update():
    """update() in the lazy mode (no Gram; F_0 from fastron_kernel_matvec_lazy) retraces the
    full mode's warm-started Algorithm 1 exactly (F_0 must be K alpha_0, not
    the fp32-alpha score)."""
    require_gpu()
    import torch
    import paper_1910_06451_b200 as fb
    from paper_1910_06451_b200.model import CapsuleScene, FastronModel
    wl = W.train_workload(1500)
    X = dev(wl.X)
    y = fb.fastron_label_capsules(fb.fastron_fk(wl.robot, X), CHAIN8, wl.cubes, wl.radius)
    full = FastronModel(wl.robot, 0, wl.gamma, 1.0, 4000)
    lazy = FastronModel(wl.robot, 0, wl.gamma, 1.0, 4000, lazy=True)
    full.fit(X, y)
    lazy.fit(X, y)
    assert torch.equal(full.alpha, lazy.alpha)
    ns = full.supports.shape[0]
    moved = wl.cubes.copy()
    rng = np.random.default_rng(8)
    for j in rng.choice(len(moved), 3, replace=False):
        v = rng.standard_normal(3)
        moved[j] += 0.1 * v / np.linalg.norm(v)
    z = dev(rng.standard_normal((2 * ns, 7)).astype(np.float32))
    u = dev(rng.uniform(0, 1, (800, 7)).astype(np.float32))
    sigma = dev(np.full(7, 0.05 * 2 * np.pi, np.float32))
    lo, hi = dev(np.full(7, -np.pi, np.float32)), dev(np.full(7, np.pi, np.float32))
    scene = CapsuleScene(np.array(CHAIN8), moved, wl.radius)
    rf = full.update(scene, z, u, sigma, lo, hi, 2)[0]
    rl = lazy.update(scene, z, u, sigma, lo, hi, 2)[0]
    torch.cuda.synchronize()
    for k in ("iterations", "n_add", "n_remove", "n_support", "converged"):
        assert rf[k] == rl[k], (k, rf, rl)
    assert torch.equal(full.alpha, lazy.alpha) and torch.equal(full.supports, lazy.supports)


@pytest.mark.parametrize("n,nnz", [(1, 1), (130, 0), (777, 777), (3001, 2500), (4500, 4100)])
def test_matvec_index_order_bit_exact(n, nnz):
    """fastron_kernel_matvec: F_j = sum over the nonzero alpha_i, in index order, of
    fl(alpha_i K_ij) with separately rounded fp64 multiply and add (the margins
    of a loaded model) — bit-exact against that sum written out, on sizes that leave a ragged
    last CTA, fill several shared-memory segments of nonzero indices (2,048 each) and on an
    all-zero alpha; K with padded rows (ldk > n)."""
    require_gpu()
    import torch
    import paper_1910_06451_b200 as fb
    rng = np.random.default_rng(n + nnz)
    ldk = (n + 7) // 8 * 8 + 8
    Kh = rng.uniform(0.0, 1.0, (n, ldk)).astype(np.float32)
    alpha = np.zeros(n)
    nz = np.sort(rng.choice(n, nnz, replace=False))
    alpha[nz] = rng.standard_normal(nnz) * 50.0
    K = dev(Kh)[:, :n]
    F = fb.fastron_kernel_matvec(K, dev(alpha))
    torch.cuda.synchronize()
    ref = np.zeros(n)
    for i in nz:  # index order; numpy's elementwise fp64 multiply and add round separately
        ref = ref + alpha[i] * Kh[i, :n].astype(np.float64)
    assert np.array_equal(F.cpu().numpy(), ref)
