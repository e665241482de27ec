"""GPU parity of fastron_score (K2) against the oracle score (PAPER.md:183 with Eq. 4),
end to end from fp32 joint configurations: GPU = fastron_fk + fastron_score, oracle =
fp64 FK + fp64 kernel sums. Tolerance: BASELINE.json north_star (R16)."""
import numpy as np
import pytest

import oracle
import workloads as W
from c4 import assert_stats, c4_sample, score_stats
from gpu_helpers import assert_score_parity, dev, require_gpu, soa_from_oracle

pytestmark = pytest.mark.gpu


def _gpu_scores(robot, supports, alpha, queries, kind, gamma):
    import torch
    import paper_1910_06451_b200 as fb
    spos = fb.fastron_fk(robot, dev(supports))
    qpos = fb.fastron_fk(robot, dev(queries))
    s, l = fb.fastron_score(qpos, spos, dev(alpha), kind, gamma)
    torch.cuda.synchronize()
    return s.cpu().numpy(), l.cpu().numpy()


def _ref_scores(robot, supports, alpha, queries, kind, gamma):
    return oracle.score(kind, gamma, oracle.fk(robot, queries), oracle.fk(robot, supports), alpha)


@pytest.mark.parametrize("kind", [W.GAUSSIAN, W.RQ])
def test_cfg1_full(kind):
    require_gpu()
    wl = W.score_workload("cfg1", kind=kind)
    s, l = _gpu_scores(wl.robot, wl.supports, wl.alpha, wl.queries, kind, wl.gamma)
    f, _ = _ref_scores(wl.robot, wl.supports, wl.alpha, wl.queries, kind, wl.gamma)
    assert_score_parity(s, f, l, what=f"cfg1 kind={kind}")


@pytest.mark.parametrize("kind", [W.GAUSSIAN, W.RQ])
def test_cfg2_full(kind):
    """cfg2 at full size: 2,000 supports against all 1,000,000 queries."""
    require_gpu()
    wl = W.score_workload("cfg2", kind=kind)
    s, l = _gpu_scores(wl.robot, wl.supports, wl.alpha, wl.queries, kind, wl.gamma)
    f, _ = _ref_scores(wl.robot, wl.supports, wl.alpha, wl.queries, kind, wl.gamma)
    st = score_stats(s, f, l)
    print(f"cfg2 kind={kind}: {st}")
    assert_stats(st, f"cfg2 kind={kind}")


def test_cfg5_subset_m16():
    require_gpu()
    wl = W.score_workload("cfg5", n_queries=20_000, n_supports=5_000)
    s, l = _gpu_scores(wl.robot, wl.supports, wl.alpha, wl.queries, 0, wl.gamma)
    f, _ = _ref_scores(wl.robot, wl.supports, wl.alpha, wl.queries, 0, wl.gamma)
    assert_score_parity(s, f, l, what="cfg5 M=16")


@pytest.mark.parametrize("kind", [W.GAUSSIAN, W.RQ])
def test_headline_full_size_sampled(kind):
    """Headline size (1M queries x 20k supports, the bench launch configuration), C4
    protocol: 50,000 seeded uniform queries plus every query with |f_gpu| <= 1e-2 (the
    label boundary, where the 1e-5 floor binds), against the oracle at the R16 tolerance
    for both term shapes (Gaussian: the north star; RQ: Eq. 3)."""
    require_gpu()
    wl = W.score_workload("headline", kind=kind)
    s, l = _gpu_scores(wl.robot, wl.supports, wl.alpha, wl.queries, kind, wl.gamma)
    idx, n_band = c4_sample(s, 50_000, seed=10 + kind)
    assert n_band > 100
    f, _ = _ref_scores(wl.robot, wl.supports, wl.alpha, wl.queries[idx], kind, wl.gamma)
    st = score_stats(s[idx], f, l[idx])
    print(f"headline kind={kind}: {st}")
    assert_stats(st, f"headline sample kind={kind}")


@pytest.mark.parametrize("M", [1, 3, 5, 32])
def test_odd_and_extreme_m(M):
    """Padded control points (odd M) contribute exactly 0; M = 32 is the maximum."""
    require_gpu()
    base = W.arm7(8)
    rng = np.random.default_rng(M)
    frames = rng.integers(0, 8, size=M)
    offs = rng.uniform(-0.1, 0.1, size=(M, 3))
    robot = W.make_robot("m%d" % M, base.dh, frames, offs)
    sup = rng.uniform(-np.pi, np.pi, size=(333, 7)).astype(np.float32)
    alpha = rng.standard_normal(333).astype(np.float32)
    q = rng.uniform(-np.pi, np.pi, size=(1500, 7)).astype(np.float32)
    for kind in (0, 1):
        s, l = _gpu_scores(robot, sup, alpha, q, kind, 5.0)
        f, _ = _ref_scores(robot, sup, alpha, q, kind, 5.0)
        assert_score_parity(s, f, l, what=f"M={M} kind={kind}")


@pytest.mark.parametrize("ns,nq", [(0, 100), (1, 1), (1, 700), (65, 3), (64, 513), (129, 10_000)])
def test_edge_sizes(ns, nq):
    require_gpu()
    robot = W.arm7(8)
    rng = np.random.default_rng(ns * 7 + nq)
    sup = rng.uniform(-np.pi, np.pi, size=(ns, 7)).astype(np.float32)
    alpha = rng.standard_normal(ns).astype(np.float32)
    q = rng.uniform(-np.pi, np.pi, size=(nq, 7)).astype(np.float32)
    if ns == 0:
        import torch
        import paper_1910_06451_b200 as fb
        qpos = fb.fastron_fk(robot, dev(q))
        spos = torch.empty((8, 0, 4), device="cuda")
        s, l = fb.fastron_score(qpos, spos, torch.empty(0, device="cuda"), 0, 5.0)
        assert np.all(s.cpu().numpy() == 0) and np.all(l.cpu().numpy() == -1)
        return
    s, l = _gpu_scores(robot, sup, alpha, q, 0, 5.0)
    f, _ = _ref_scores(robot, sup, alpha, q, 0, 5.0)
    assert_score_parity(s, f, l, what=f"ns={ns} nq={nq}")


def test_self_support_gives_exactly_one():
    """One support at the query with alpha = 1 -> f = k(q, q) = 1 exactly (R18)."""
    require_gpu()
    robot = W.arm7(8)
    q = np.random.default_rng(1).uniform(-np.pi, np.pi, size=(50, 7)).astype(np.float32)
    for kind in (0, 1):
        for i in range(0, 50, 7):
            s, l = _gpu_scores(robot, q[i:i + 1], np.ones(1, np.float32), q[i:i + 1], kind, 5.0)
            assert s[0] == 1.0 and l[0] == 1


def test_deterministic_and_positions_input():
    """Bit-reproducible across runs; and fastron_score on oracle-rounded positions matches the
    oracle score of those same fp32 positions (the score stage alone)."""
    require_gpu()
    import torch
    import paper_1910_06451_b200 as fb
    wl = W.score_workload("cfg2", n_queries=5000, n_supports=700)
    s1, l1 = _gpu_scores(wl.robot, wl.supports, wl.alpha, wl.queries, 0, wl.gamma)
    s2, l2 = _gpu_scores(wl.robot, wl.supports, wl.alpha, wl.queries, 0, wl.gamma)
    assert np.array_equal(s1, s2) and np.array_equal(l1, l2)
    qp = oracle.fk(wl.robot, wl.queries).astype(np.float32).astype(np.float64)
    sp = oracle.fk(wl.robot, wl.supports).astype(np.float32).astype(np.float64)
    s, l = fb.fastron_score(soa_from_oracle(qp), soa_from_oracle(sp), dev(wl.alpha), 0, wl.gamma)
    torch.cuda.synchronize()
    f, _ = oracle.score(0, wl.gamma, qp, sp, wl.alpha)
    assert_score_parity(s.cpu().numpy(), f, l.cpu().numpy(), what="positions input")


def test_linearity_in_alpha():
    require_gpu()
    wl = W.score_workload("cfg1", n_queries=3000, n_supports=300)
    s1, _ = _gpu_scores(wl.robot, wl.supports, wl.alpha, wl.queries, 0, wl.gamma)
    s2, _ = _gpu_scores(wl.robot, wl.supports, (2 * wl.alpha).astype(np.float32), wl.queries, 0, wl.gamma)
    assert np.array_equal(s2, 2 * s1)  # scaling alpha by 2 is exact in binary floating point


def test_query_host_pipeline_matches_device_path():
    """fastron_query with pinned host buffers (chunked H2D/D2H overlap) equals fk + score."""
    require_gpu()
    import torch
    import paper_1910_06451_b200 as fb
    wl = W.score_workload("cfg2", n_queries=600_000, n_supports=500)
    spos = fb.fastron_fk(wl.robot, dev(wl.supports))
    alpha = dev(wl.alpha)
    s_dev, l_dev = _gpu_scores(wl.robot, wl.supports, wl.alpha, wl.queries, 0, wl.gamma)
    qh = torch.from_numpy(wl.queries).pin_memory()
    sh = torch.empty(len(wl.queries), dtype=torch.float32).pin_memory()
    lh = torch.empty(len(wl.queries), dtype=torch.int8).pin_memory()
    fb.fastron_query(wl.robot, qh, spos, alpha, 0, wl.gamma, score=sh, label=lh)
    assert np.array_equal(sh.numpy(), s_dev) and np.array_equal(lh.numpy(), l_dev)
    # pageable host memory and device tensors work too
    qp = torch.from_numpy(wl.queries[:1000].copy())
    sp = torch.empty(1000, dtype=torch.float32)
    fb.fastron_query(wl.robot, qp, spos, alpha, 0, wl.gamma, score=sp)
    assert np.array_equal(sp.numpy(), s_dev[:1000])
    sd = torch.empty(1000, dtype=torch.float32, device="cuda")
    fb.fastron_query(wl.robot, dev(wl.queries[:1000]), spos, alpha, 0, wl.gamma, score=sd)
    torch.cuda.synchronize()
    assert np.array_equal(sd.cpu().numpy(), s_dev[:1000])
    # mixed: host q (3 chunks, the last ragged), device scores, host labels only
    n3 = 2 * 262_144 + 17
    sd3 = torch.empty(n3, dtype=torch.float32, device="cuda")
    lh3 = torch.empty(n3, dtype=torch.int8).pin_memory()
    fb.fastron_query(wl.robot, qh[:n3], spos, alpha, 0, wl.gamma, score=sd3, label=lh3)
    torch.cuda.synchronize()
    assert np.array_equal(sd3.cpu().numpy(), s_dev[:n3]) and np.array_equal(lh3.numpy(), l_dev[:n3])
    lh4 = torch.empty(n3, dtype=torch.int8).pin_memory()
    fb.fastron_query(wl.robot, qh[:n3], spos, alpha, 0, wl.gamma, score=None, label=lh4)
    assert np.array_equal(lh4.numpy(), l_dev[:n3])


@pytest.mark.parametrize("kind", [W.GAUSSIAN, W.RQ])
def test_cfg5_full_size_sampled(kind):
    """cfg5 at its full BASELINE.json size (10M queries x 20k supports, M = 16), C4
    protocol: 10,000 seeded uniform queries plus every query with |f_gpu| <= 1e-2."""
    require_gpu()
    wl = W.score_workload("cfg5", kind=kind)
    assert len(wl.queries) == 10_000_000 and len(wl.supports) == 20_000 and wl.robot.n_cp == 16
    s, l = _gpu_scores(wl.robot, wl.supports, wl.alpha, wl.queries, kind, wl.gamma)
    idx, _ = c4_sample(s, 10_000, seed=20 + kind)
    f, _ = _ref_scores(wl.robot, wl.supports, wl.alpha, wl.queries[idx], kind, wl.gamma)
    st = score_stats(s[idx], f, l[idx])
    print(f"cfg5 kind={kind}: {st}")
    assert_stats(st, f"cfg5 full-size sample kind={kind}")


def test_query_chunks_planned_like_the_batch():
    """fastron_query streams 256k-query chunks; each chunk is planned like the whole batch
    (same support splits, so the same fp64 summation order), so the chunked scores equal
    a single launch over the batch bit for bit — at the headline model size, where the
    split count depends on the batch size."""
    require_gpu()
    import torch
    import paper_1910_06451_b200 as fb
    wl = W.score_workload("headline", n_queries=600_000)
    spos = fb.fastron_fk(wl.robot, dev(wl.supports))
    alpha = dev(wl.alpha)
    s_dev, l_dev = _gpu_scores(wl.robot, wl.supports, wl.alpha, wl.queries, 0, wl.gamma)
    qh = torch.from_numpy(wl.queries).pin_memory()
    sh = torch.empty(len(wl.queries), dtype=torch.float32).pin_memory()
    lh = torch.empty(len(wl.queries), dtype=torch.int8).pin_memory()
    fb.fastron_query(wl.robot, qh, spos, alpha, 0, wl.gamma, score=sh, label=lh)
    assert np.array_equal(sh.numpy(), s_dev) and np.array_equal(lh.numpy(), l_dev)


@pytest.mark.parametrize("M", [4, 5, 8, 16])
@pytest.mark.parametrize("kind", [W.GAUSSIAN, W.RQ])
def test_small_batches(M, kind):
    """nq <= 32 takes the support-parallel kernel (one launch, fixed-order reduction):
    parity for 1..32 queries against 1 to 20,000 supports, and every path agrees with it."""
    require_gpu()
    import torch
    import paper_1910_06451_b200 as fb
    base = W.arm7(8)
    rng = np.random.default_rng(40 + M)
    robot = base if M == 8 else W.make_robot("m%d" % M, base.dh, rng.integers(1, 8, size=M),
                                              rng.uniform(-0.1, 0.1, size=(M, 3)))
    sup = W.uniform_configs(rng, 20_000, 7)
    alpha = rng.standard_normal(20_000).astype(np.float32)
    q = W.uniform_configs(rng, 32, 7)
    spos_ref = oracle.fk(robot, sup)
    qpos_ref = oracle.fk(robot, q)
    for ns in (1, 63, 303, 20_000):
        for nq in (1, 5, 32):
            s, l = _gpu_scores(robot, sup[:ns], alpha[:ns], q[:nq], kind, 5.0)
            f, _ = oracle.score(kind, 5.0, qpos_ref[:nq], spos_ref[:ns], alpha[:ns])
            assert_score_parity(s, f, l, what=f"small M={M} kind={kind} ns={ns} nq={nq}")
    # the packed-model path, the fp64 path and fastron_query give the same small-batch scores
    spos = fb.fastron_fk(robot, dev(sup))
    model = fb.fastron_model_pack(spos, dev(alpha), kind, 5.0)
    qpos = fb.fastron_fk(robot, dev(q[:7]))
    s1, _ = fb.fastron_score_packed(qpos, model)
    s64 = fb.fastron_score_packed_f64(qpos, model)
    sh = torch.empty(7, dtype=torch.float32).pin_memory()
    fb.fastron_query(robot, torch.from_numpy(q[:7].copy()), spos, dev(alpha), kind, 5.0, score=sh)
    torch.cuda.synchronize()
    assert np.array_equal(s1.cpu().numpy(), sh.numpy())
    assert np.array_equal(s1.cpu().numpy(), s64.cpu().numpy().astype(np.float32))
    # fastron_query on device buffers: FK fused into the small-batch kernel, same scores
    sd = torch.empty(7, dtype=torch.float32, device="cuda")
    ld = torch.empty(7, dtype=torch.int8, device="cuda")
    fb.fastron_query(robot, dev(q[:7]), spos, dev(alpha), kind, 5.0, score=sd, label=ld)
    torch.cuda.synchronize()
    assert np.array_equal(s1.cpu().numpy(), sd.cpu().numpy())


@pytest.mark.parametrize("name,nq", [("headline", 33), ("headline", 100), ("headline", 128), ("headline", 129),
                                     ("headline", 4096), ("cfg5", 64), ("cfg5", 1000)])
def test_mid_batches_many_splits(name, nq):
    """Batches between the small-batch kernel and the bulk path against 20k supports:
    one query per thread (33..128 queries) and the grouped finalize (> 16 splits)."""
    require_gpu()
    wl = W.score_workload(name, n_queries=nq)
    s, l = _gpu_scores(wl.robot, wl.supports, wl.alpha, wl.queries, 0, wl.gamma)
    f, _ = _ref_scores(wl.robot, wl.supports, wl.alpha, wl.queries, 0, wl.gamma)
    assert_score_parity(s, f, l, what=f"{name} nq={nq}")


@pytest.mark.parametrize("M,kind,nqs", [
    (8, W.GAUSSIAN, (1, 32, 33, 100, 128, 129, 1000, 2048, 2049, 5000, 100_003)),
    (8, W.RQ, (33, 1000, 5000)),
    (4, W.GAUSSIAN, (40, 10_000)),
    (16, W.GAUSSIAN, (64, 512, 513, 3000)),
    (5, W.RQ, (77, 1500)),
])
def test_query_packed_equals_fk_plus_score(M, kind, nqs):
    """fastron_query_packed (configurations in, scores out, one API call) gives the bits of
    fastron_fk + fastron_score_packed for every batch size: the small-batch kernel with
    the D-H chain inside (nq <= 32), one query per thread, several per thread, few and
    many support splits."""
    require_gpu()
    import torch
    import paper_1910_06451_b200 as fb
    base = W.arm7(8) if M != 4 else W.score_workload("cfg1", n_queries=1, n_supports=1).robot
    rng = np.random.default_rng(300 + M + kind)
    robot = base if M in (4, 8) else W.make_robot("m%d" % M, base.dh, rng.integers(0, 8, size=M),
                                                   rng.uniform(-0.1, 0.1, size=(M, 3)))
    D = robot.dh.shape[0]
    for ns in (300, 3_000, 20_000):
        sup = W.uniform_configs(rng, ns, D)
        alpha = rng.standard_normal(ns).astype(np.float32)
        model = fb.fastron_model_pack(fb.fastron_fk(robot, dev(sup)), dev(alpha), kind, 5.0)
        for nq in nqs:
            qf = rng.uniform(-np.pi, np.pi, size=(nq, D + 2)).astype(np.float32)  # ldq = D + 2
            q = dev(qf)[:, :D]
            s1, l1 = fb.fastron_score_packed(fb.fastron_fk(robot, q), model)
            s2, l2 = fb.fastron_query_packed(robot, q, model)
            torch.cuda.synchronize()
            assert torch.equal(s1, s2) and torch.equal(l1, l2), (ns, nq)
    # and the scores are right (oracle, R16) on one mid-size case
    f, _ = _ref_scores(robot, sup, alpha, np.ascontiguousarray(qf[:, :D]), kind, 5.0)
    assert_score_parity(s2.cpu().numpy(), f, l2.cpu().numpy(), what=f"query_packed M={M} kind={kind}")


def test_query_packed_rejects_host_buffers():
    require_gpu()
    import torch
    import paper_1910_06451_b200 as fb
    robot = W.arm7(8)
    model = fb.fastron_model_pack(fb.fastron_fk(robot, dev(W.uniform_configs(np.random.default_rng(0), 64, 7))),
                                  dev(np.ones(64, np.float32)), 0, 5.0)
    with pytest.raises(ValueError):
        fb.fastron_query_packed(robot, torch.zeros((10, 7)), model)
