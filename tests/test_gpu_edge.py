"""GPU parity of fastron_edge_check (K4: interpolate -> FK -> score -> warp vote) against
the oracle edge check (BASELINE.json cfg4; R11)."""
import numpy as np
import pytest

import oracle
import workloads as W
from gpu_helpers import dev, require_gpu

pytestmark = pytest.mark.gpu


def _gpu_edges(robot, qa, qb, n_interp, sup, alpha, kind, gamma):
    import torch
    import paper_1910_06451_b200 as fb
    spos = fb.fastron_fk(robot, dev(sup))
    hit, idx = fb.fastron_edge_check(robot, dev(qa), dev(qb), n_interp, spos, dev(alpha), kind, gamma)
    torch.cuda.synchronize()
    return hit.cpu().numpy(), idx.cpu().numpy()


def _order(n):
    return [2 * o for o in range((n + 1) // 2)] + [2 * o + 1 for o in range(n // 2)]


def _check(robot, qa, qb, n_interp, sup, alpha, kind, gamma):
    hit, idx = _gpu_edges(robot, qa, qb, n_interp, sup, alpha, kind, gamma)
    ref_hit, fmax, fall = oracle.edge(robot, qa, qb, n_interp, kind, gamma, oracle.fk(robot, sup), alpha,
                                      with_all=True)
    sure = np.abs(fmax) > 1e-4
    bad = np.flatnonzero(sure & (hit != ref_hit))
    assert bad.size == 0, f"{bad.size} edge label mismatches, e.g. {bad[:5]} fmax {fmax[bad[:5]]}"
    order = _order(n_interp)
    for e in range(len(hit)):
        if hit[e]:
            k = idx[e]
            assert 0 <= k < n_interp and fall[e, k] > -1e-4
            r = order.index(k) // 32  # the round that reported the hit; earlier rounds had no hit
            earlier = [order[o] for o in range(0, 32 * r)]
            assert np.all(fall[e, earlier] <= 1e-4)
            same_round = [order[o] for o in range(32 * r, min(32 * r + 32, n_interp))]
            pos_in_round = [kk for kk in same_round if fall[e, kk] > 1e-4]
            if pos_in_round:
                assert k <= min(pos_in_round)
        else:
            assert idx[e] == -1
    return hit, ref_hit, fmax


@pytest.mark.parametrize("kind", [W.GAUSSIAN, W.RQ])
def test_cfg4_subset(kind):
    require_gpu()
    wl = W.edge_workload(n_edges=1500, kind=kind)
    hit, ref, fmax = _check(wl.robot, wl.qa, wl.qb, wl.n_interp, wl.supports, wl.alpha, kind, wl.gamma)
    assert 0 < hit.sum() < len(hit)


@pytest.mark.parametrize("n_interp", [1, 2, 33, 64, 100])
def test_interp_counts_and_rounds(n_interp):
    require_gpu()
    wl = W.edge_workload(n_edges=300, n_supports=700)
    # shorter edges so that both outcomes are frequent
    qb = (wl.qa + 0.25 * (wl.qb - wl.qa)).astype(np.float32)
    _check(wl.robot, wl.qa, qb, n_interp, wl.supports, wl.alpha, 1, wl.gamma)


def test_degenerate_and_endpoint_edges():
    """a = b free -> 0; an endpoint with f > 0 -> 1."""
    require_gpu()
    wl = W.edge_workload(n_edges=10, n_supports=500)
    q = np.random.default_rng(0).uniform(-np.pi, np.pi, size=(3000, 7)).astype(np.float32)
    f, _ = oracle.score(0, wl.gamma, oracle.fk(wl.robot, q), oracle.fk(wl.robot, wl.supports), wl.alpha)
    nb = min(int(np.sum(f < -1e-3)), int(np.sum(f > 1e-3)), 50)
    assert nb >= 8
    free = q[f < -1e-3][:nb]
    bad = q[f > 1e-3][:nb]
    hit, idx = _gpu_edges(wl.robot, free, free, 64, wl.supports, wl.alpha, 0, wl.gamma)
    assert np.all(hit == 0) and np.all(idx == -1)
    hit, idx = _gpu_edges(wl.robot, bad, free, 64, wl.supports, wl.alpha, 0, wl.gamma)
    assert np.all(hit == 1) and np.all(idx == 0)  # k = 0 is the first point of round 1
    hit, idx = _gpu_edges(wl.robot, free, bad, 64, wl.supports, wl.alpha, 0, wl.gamma)
    assert np.all(hit == 1)


def test_edge_equals_or_of_scores():
    """T2: in_collision == OR_k (fastron_score(fastron_fk(q_k)) > 0) with q_k interpolated in
    fp32 exactly as the kernel does (t = k/(n-1), q = a + t (b - a), each op rounded)."""
    require_gpu()
    import torch
    import paper_1910_06451_b200 as fb
    wl = W.edge_workload(n_edges=400, n_supports=900)
    hit, _ = _gpu_edges(wl.robot, wl.qa, wl.qb, 64, wl.supports, wl.alpha, 0, wl.gamma)
    t = (np.arange(64, dtype=np.float32) / np.float32(63)).astype(np.float32)
    d = (wl.qb - wl.qa).astype(np.float32)
    pts = (wl.qa[:, None, :] + (t[None, :, None] * d[:, None, :]).astype(np.float32)).astype(np.float32)
    spos = fb.fastron_fk(wl.robot, dev(wl.supports))
    qpos = fb.fastron_fk(wl.robot, dev(pts.reshape(-1, 7)))
    _, lab = fb.fastron_score(qpos, spos, dev(wl.alpha), 0, wl.gamma)
    torch.cuda.synchronize()
    any_pos = (lab.cpu().numpy().reshape(400, 64) > 0).any(axis=1)
    assert np.array_equal(hit.astype(bool), any_pos)


@pytest.mark.parametrize("kind", [W.GAUSSIAN, W.RQ])
def test_cfg4_full_size_all_edges(kind):
    """cfg4 at its full size (10,000 edges x 64 points against 3,000 supports, the bench
    launch), every edge against the oracle: labels bit-exact wherever
    the edge's max score is outside +-1e-4, and every reported hit point really has
    f_ref > -1e-4; misses report -1."""
    require_gpu()
    wl = W.edge_workload(kind=kind)
    assert len(wl.qa) == 10_000 and wl.n_interp == 64 and len(wl.supports) == 3_000
    hit, idx = _gpu_edges(wl.robot, wl.qa, wl.qb, wl.n_interp, wl.supports, wl.alpha, kind, wl.gamma)
    ref_hit, fmax, fall = oracle.edge(wl.robot, wl.qa, wl.qb, wl.n_interp, kind, wl.gamma,
                                      oracle.fk(wl.robot, wl.supports), wl.alpha, with_all=True)
    sure = np.abs(fmax) > 1e-4
    assert np.array_equal(hit[sure], ref_hit[sure])
    h = np.flatnonzero(hit)
    assert np.all(fall[h, idx[h]] > -1e-4)
    assert np.all(idx[hit == 0] == -1)
    print(f"cfg4 kind={kind}: {int(hit.sum())} of 10,000 in collision, {int((~sure).sum())} ambiguous")


def test_odd_m_robot_edges():
    """Odd M (a padded control point) through the edge path: the FK prologue writes the
    query side, which leaves the padded point at 0 (term exactly 0)."""
    require_gpu()
    wl = W.edge_workload(n_edges=200, n_supports=400)
    rng = np.random.default_rng(5)
    robot = W.make_robot("m5", wl.robot.dh, rng.integers(1, 8, size=5), rng.uniform(-0.1, 0.1, size=(5, 3)))
    _check(robot, wl.qa, wl.qb, wl.n_interp, wl.supports, wl.alpha, 0, wl.gamma)


@pytest.mark.parametrize("kind", [W.GAUSSIAN, W.RQ])
def test_edge_check_packed_equals_edge_check(kind):
    """The packed-model edge check (a model packed once, e.g. broadcast to every GPU) gives
    exactly fastron_edge_check's flags and hit indices."""
    require_gpu()
    import torch
    import paper_1910_06451_b200 as fb
    wl = W.edge_workload(n_edges=2000, kind=kind)
    spos = fb.fastron_fk(wl.robot, dev(wl.supports))
    qa, qb = dev(wl.qa), dev(wl.qb)
    h1, i1 = fb.fastron_edge_check(wl.robot, qa, qb, wl.n_interp, spos, dev(wl.alpha), kind, wl.gamma)
    model = fb.fastron_model_pack(spos, dev(wl.alpha), kind, wl.gamma)
    h2, i2 = fb.fastron_edge_check_packed(wl.robot, qa, qb, wl.n_interp, model)
    torch.cuda.synchronize()
    assert torch.equal(h1, h2) and torch.equal(i1, i2) and 0 < int(h1.sum()) < len(h1)
