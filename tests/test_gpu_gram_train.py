"""GPU parity of fastron_gram (K3) and fastron_train (K5, Algorithm 1) against the
oracle, plus the cross-kernel identity Gram == score(alpha = e_i)."""
import json
import os

import numpy as np
import pytest

import oracle
import workloads as W
from gpu_helpers import assert_score_parity, dev, require_gpu

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _gram(robot, X, kind, gamma):
    import torch
    import paper_1910_06451_b200 as fb
    pos = fb.fastron_fk(robot, dev(X))
    K = fb.fastron_gram(pos, kind, gamma)
    torch.cuda.synchronize()
    return pos, K


@pytest.mark.parametrize("n,kind", [(1, 0), (127, 0), (300, 1), (1000, 0), (1000, 1)])
def test_gram_parity_symmetry_diagonal(n, kind):
    require_gpu()
    wl = W.train_workload(n)
    _, K = _gram(wl.robot, wl.X, kind, wl.gamma)
    Kg = K.cpu().numpy()
    assert np.array_equal(Kg, Kg.T)  # mirrored tiles: exactly symmetric
    assert np.all(np.diag(Kg) == 1.0)  # R18: d^2 = 0 -> every term exactly 1
    Kr = oracle.gram(kind, wl.gamma, oracle.fk(wl.robot, wl.X))
    assert_score_parity(Kg.ravel(), Kr.ravel(), what=f"gram n={n}")
    if n <= 300 and n > 1:
        ev = np.linalg.eigvalsh(Kg.astype(np.float64))
        assert ev[0] >= -1e-6 * ev[-1]  # Claim 1 up to fp32 rounding


def test_gram_m16_and_ldk():
    require_gpu()
    import torch
    import paper_1910_06451_b200 as fb
    robot, X, _, _ = W.cfg5_gram_workload(400)
    pos = fb.fastron_fk(robot, dev(X))
    K = torch.full((400, 416), -3.0, device="cuda")
    fb.fastron_gram(pos, 0, 5.0, K=K[:, :400])  # ldk = 416
    torch.cuda.synchronize()
    Kh = K.cpu().numpy()
    assert np.all(Kh[:, 400:] == -3.0)
    Kr = oracle.gram(0, 5.0, oracle.fk(robot, X))
    assert_score_parity(Kh[:, :400].ravel(), Kr.ravel(), what="gram M=16")


@pytest.mark.parametrize("M", [1, 3, 5, 12, 32])
def test_gram_odd_and_extreme_m(M):
    """Every column-per-lane path (CPL 2 at M <= 16, 1 above), padded control points of odd
    M, and the non-power-of-two 1/M division: parity, exact symmetry, unit diagonal."""
    require_gpu()
    base = W.arm7(8)
    rng = np.random.default_rng(100 + M)
    robot = W.make_robot("m%d" % M, base.dh, rng.integers(0, 8, size=M), rng.uniform(-0.1, 0.1, size=(M, 3)))
    X = rng.uniform(-np.pi, np.pi, size=(301, 7)).astype(np.float32)
    for kind in (0, 1):
        _, K = _gram(robot, X, kind, 5.0)
        Kg = K.cpu().numpy()
        assert np.array_equal(Kg, Kg.T) and np.all(np.diag(Kg) == 1.0)
        Kr = oracle.gram(kind, 5.0, oracle.fk(robot, X))
        assert_score_parity(Kg.ravel(), Kr.ravel(), what=f"gram M={M} kind={kind}")


def test_gram_equals_score_with_unit_alpha():
    """T2 cross-kernel identity: K[i, j] == fastron_score(x_j; supports X, alpha = e_i) bit for bit."""
    require_gpu()
    import torch
    import paper_1910_06451_b200 as fb
    wl = W.train_workload(260)
    pos, K = _gram(wl.robot, wl.X, 0, wl.gamma)
    Kh = K.cpu().numpy()
    for i in (0, 1, 63, 64, 200, 259):
        alpha = torch.zeros(260, device="cuda")
        alpha[i] = 1.0
        s, _ = fb.fastron_score(pos, pos, alpha, 0, wl.gamma)
        torch.cuda.synchronize()
        assert np.array_equal(s.cpu().numpy(), Kh[i]), i


def _labels(wl):
    pos = oracle.fk(wl.robot, wl.X)
    return W.capsule_aabb_labels(W.chain_points(pos), wl.cubes, wl.radius)


def _gpu_train(K, y, beta, iter_max, s_max=None, alpha0=None, F0=None):
    import torch
    import paper_1910_06451_b200 as fb
    out = fb.fastron_train(K, dev(y), beta, iter_max, s_max,
                           alpha=None if alpha0 is None else dev(alpha0, torch.float64),
                           F=None if F0 is None else dev(F0, torch.float64))
    torch.cuda.synchronize()
    res = fb.train_result(out["result"])
    return dict(alpha=out["alpha"].cpu().numpy(), F=out["F"].cpu().numpy(),
                trace=out["trace"].cpu().numpy()[:res["iterations"]],
                support=out["support_idx"].cpu().numpy()[:res["n_support"]], **res)


def _assert_same_run(g, r):
    assert g["iterations"] == r["iterations"] and g["n_add"] == r["n_add"] and g["n_remove"] == r["n_remove"]
    assert np.array_equal(g["trace"], r["trace"]), np.flatnonzero(g["trace"] != r["trace"])[:5]
    assert g["converged"] == r["converged"] and g["n_support"] == r["n_support"]
    assert np.array_equal(g["support"], r["support"])
    scale = max(1.0, float(np.abs(r["alpha"]).max()))
    assert np.abs(g["alpha"] - r["alpha"]).max() <= 1e-9 * scale
    assert np.abs(g["F"] - r["F"]).max() <= 1e-9 * max(1.0, float(np.abs(r["F"]).max()))


@pytest.mark.parametrize("n,beta,s_max", [(1000, 1.0, None), (1000, 2.0, None), (1000, 1.0, 50), (5000, 1.0, None)])
def test_train_trace_exact_on_gpu_gram(n, beta, s_max):
    """P-exact mode: the oracle's Algorithm 1 on the GPU's fp32 Gram
    promoted to fp64 must give the identical trace and alpha. n = 5000 is cfg3 itself."""
    require_gpu()
    wl = W.train_workload(n)
    y = _labels(wl)
    _, K = _gram(wl.robot, wl.X, 0, wl.gamma)
    g = _gpu_train(K, y, beta, wl.iter_max, s_max)
    r = oracle.train(K.cpu().numpy().astype(np.float64), y, beta, wl.iter_max, s_max)
    _assert_same_run(g, r)


def test_train_warm_start_and_iter_max():
    require_gpu()
    wl = W.train_workload(800)
    y = _labels(wl)
    _, K = _gram(wl.robot, wl.X, 1, wl.gamma)
    K64 = K.cpu().numpy().astype(np.float64)
    first = oracle.train(K64, y, 1.0, 300)
    y2 = y.copy()
    y2[::7] *= -1  # labels move: retrain from the previous model
    g = _gpu_train(K, y2, 1.0, 20000, alpha0=first["alpha"], F0=first["F"])
    r = oracle.train(K64, y2, 1.0, 20000, alpha0=first["alpha"], F0=first["F"])
    _assert_same_run(g, r)
    g0 = _gpu_train(K, y2, 1.0, 0)
    assert g0["iterations"] == 0 and not g0["converged"]


@pytest.mark.parametrize("case", json.load(open(os.path.join(GOLD, "train_cases.json")))["cases"],
                         ids=lambda c: c["name"])
def test_train_hand_derived_cases(case):
    require_gpu()
    import torch
    K = torch.tensor(case["K"], dtype=torch.float32, device="cuda")
    K64 = K.cpu().numpy().astype(np.float64)  # 0.9 is not an fp32 value: compare to the fp32-K oracle run
    y = np.array(case["y"], dtype=np.int8)
    g = _gpu_train(K, y, case["beta"], case["iter_max"], case["s_max"], case.get("alpha0"),
                   None if "F0" not in case else (K64 @ np.array(case["alpha0"])))
    r = oracle.train(K64, y, case["beta"], case["iter_max"], case["s_max"], alpha0=case.get("alpha0"),
                     F0=None if "F0" not in case else (K64 @ np.array(case["alpha0"])))
    _assert_same_run(g, r)
    np.testing.assert_allclose(g["alpha"], case["alpha"], atol=1e-6)
    assert g["trace"].tolist() == case["trace"]


def test_cfg5_gram_full_size_sampled_rows():
    """cfg5 Gram at full size (N = 20,000, M = 16, 1.6 GB): 200 seeded rows against the
    oracle's Eq. 4 values (each row = the oracle score of all N points against one support
    with alpha = 1, i.e. K(x_j, x_i) by its definition), plus exact symmetry of those rows
    and columns and the unit diagonal."""
    require_gpu()
    import torch
    import paper_1910_06451_b200 as fb
    robot, X = W.cfg5_gram_workload()[:2]
    assert X.shape == (20_000, 7) and robot.n_cp == 16
    pos = fb.fastron_fk(robot, dev(X))
    K = fb.fastron_gram(pos, 0, 5.0)
    torch.cuda.synchronize()
    rows = np.random.default_rng(11).choice(len(X), 200, replace=False)
    rows[-1] = len(X) - 1  # the ragged last tile
    Kr = K[torch.as_tensor(rows, device=K.device)].cpu().numpy()
    Kc = K[:, torch.as_tensor(rows, device=K.device)].cpu().numpy().T
    del K
    assert np.array_equal(Kr, Kc)
    assert np.all(Kr[np.arange(len(rows)), rows] == 1.0)
    opos = oracle.fk(robot, X)
    for r, i in enumerate(rows):
        ref, _ = oracle.score(0, 5.0, opos, opos[i:i + 1], np.ones(1, np.float32))
        assert_score_parity(Kr[r], ref, what=f"cfg5 Gram row {i}")


def test_train_cluster_path_trace_exact():
    """n = 6,145 > one CTA's 6,144 register slots: Algorithm 1 runs on a 7-CTA cluster
    (slices of 878, DSMEM candidate exchange); the trace, alpha and F must still equal the
    oracle's on the same Gram."""
    require_gpu()
    robot, X = W.arm7(8), W.cfg5_gram_workload(6145)[1]
    cubes = W.train_workload().cubes
    y = W.capsule_aabb_labels(W.chain_points(oracle.fk(robot, X)), cubes, 0.05)
    _, K = _gram(robot, X, 0, 5.0)
    g = _gpu_train(K, y, 1.0, 20_000)
    r = oracle.train(K.cpu().numpy().astype(np.float64), y, 1.0, 20_000)
    _assert_same_run(g, r)


@pytest.mark.parametrize("M,n,kind", [(16, 1000, 0), (5, 777, 1), (8, 1, 0), (8, 129, 0), (8, 385, 0), (4, 1153, 1),
                                       (32, 300, 0)])
def test_gram_forms_bit_identical(M, n, kind):
    """K3 has two forms: the column-slot form (one 64-row tile per CTA, 16-byte mirror
    stores; needs ldk % 4 == 0) and the tile form (any ldk). Both evaluate every entry with
    the same term function and summation order, so an odd ldk (tile form) and a padded one
    (column-slot form) must give the same matrix bit for bit — partial blocks, remainder
    columns, ragged last tiles, odd M — and neither may write outside the n x n matrix."""
    require_gpu()
    import torch
    import paper_1910_06451_b200 as fb
    rng = np.random.default_rng(M + n)
    base = W.arm7(8)
    robot = W.make_robot("t%d" % M, base.dh, rng.integers(0, 8, size=M), rng.uniform(-0.1, 0.1, size=(M, 3)))
    X = rng.uniform(-np.pi, np.pi, size=(n, 7)).astype(np.float32)
    pos = fb.fastron_fk(robot, dev(X))
    out = []
    for pad in (1, 8):  # ldk = n + 1 (odd: tile form), n + 8 (column-slot form when n % 4 == 0)
        ld = n + pad + (0 if pad == 1 else (-(n + pad)) % 4)
        K = torch.full((n + 2, ld), -7.0, device="cuda")  # guard rows and columns
        fb.fastron_gram(pos, kind, 5.0, K=K[:n, :n])
        torch.cuda.synchronize()
        g = K.cpu().numpy()
        assert np.all(g[:, n:] == -7.0) and np.all(g[n:, :] == -7.0)
        g = g[:n, :n]
        assert np.all(np.diag(g) == 1.0) and np.array_equal(g, g.T)
        out.append(g)
    assert np.array_equal(out[0], out[1])


def test_train_every_cluster_size_same_run():
    """The training state can be split over any cluster size; C only changes the slices,
    the slot instances (C = 1 puts 20 slots in each of 256 threads: the largest register
    instances, otherwise used only above 32k points) and the exchange — never the run.
    cfg3 (N = 5,000) at C = 1, 2, 3, 5 (default), 16 against the oracle's trace."""
    require_gpu()
    wl = W.train_workload()
    y = _labels(wl)
    _, K = _gram(wl.robot, wl.X, 0, wl.gamma)
    r = oracle.train(K.cpu().numpy().astype(np.float64), y, 1.0, wl.iter_max)
    old = os.environ.get("FASTRON_TRAIN_CLUSTER")
    try:
        for C in (1, 2, 3, 5, 16):
            os.environ["FASTRON_TRAIN_CLUSTER"] = str(C)
            _assert_same_run(_gpu_train(K, y, 1.0, wl.iter_max), r)
    finally:
        if old is None:
            os.environ.pop("FASTRON_TRAIN_CLUSTER", None)
        else:
            os.environ["FASTRON_TRAIN_CLUSTER"] = old


def test_train_removals_on_cluster():
    """Algorithm 1's removal branch (max over alpha != 0 of y(F - alpha) > 0)
    on the cluster path (N = 2,500 > 2,048: C = 3 by default, and forced C = 2 and 8): a
    cold run and a warm start after label flips at gamma = 20, where the
    runs converge and remove supports, must retrace the oracle exactly, n_remove > 0."""
    require_gpu()
    wl = W.train_workload(2500)
    y = _labels(wl)
    _, K = _gram(wl.robot, wl.X, 0, 20.0)
    K64 = K.cpu().numpy().astype(np.float64)
    first = oracle.train(K64, y, 1.0, 20_000)
    y2 = y.copy()
    y2[::7] *= -1
    warm = oracle.train(K64, y2, 1.0, 20_000, alpha0=first["alpha"], F0=first["F"])
    assert first["n_remove"] > 0 and warm["n_remove"] > 0 and warm["converged"]
    old = os.environ.get("FASTRON_TRAIN_CLUSTER")
    try:
        for C in (None, 2, 8):
            if C is None:
                os.environ.pop("FASTRON_TRAIN_CLUSTER", None)
            else:
                os.environ["FASTRON_TRAIN_CLUSTER"] = str(C)
            _assert_same_run(_gpu_train(K, y, 1.0, 20_000), first)
            _assert_same_run(_gpu_train(K, y2, 1.0, 20_000, alpha0=first["alpha"], F0=first["F"]), warm)
    finally:
        if old is None:
            os.environ.pop("FASTRON_TRAIN_CLUSTER", None)
        else:
            os.environ["FASTRON_TRAIN_CLUSTER"] = old
