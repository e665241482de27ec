"""GPU parity of fastron_fk (K1) against the oracle FK (Eq. 1-2)."""
import numpy as np
import pytest

import oracle
import workloads as W
from gpu_helpers import dev, positions_np, require_gpu

pytestmark = pytest.mark.gpu


def _fk(robot, q, **kw):
    import paper_1910_06451_b200 as fb
    return fb.fastron_fk(robot, dev(q), **kw)


def _check(robot, q, atol=1e-6):
    import torch
    pos = _fk(robot, q)
    torch.cuda.synchronize()
    got = positions_np(pos)
    ref = oracle.fk(robot, q)
    err = np.abs(got - ref)
    assert err.max() <= atol, f"max FK error {err.max():.3g} m"
    # fp64 chain, one rounding: within one fp32 ulp of the rounded oracle value
    ulp = np.spacing(np.abs(ref).astype(np.float32)).astype(np.float64)
    assert np.all(np.abs(got - ref.astype(np.float32).astype(np.float64)) <= ulp + 1e-12)
    assert np.all(pos.cpu().numpy()[:, :, 3] == 0.0)
    return got


@pytest.mark.parametrize("name", ["cfg1", "cfg2", "cfg5"])
def test_fk_parity_configs(name):
    require_gpu()
    nq = {"cfg1": None, "cfg2": None, "cfg5": 1_000_000}[name]
    wl = W.score_workload(name, n_queries=nq)
    _check(wl.robot, wl.queries)
    _check(wl.robot, wl.supports)


@pytest.mark.parametrize("n", [1, 31, 127, 129, 255, 257, 383, 1000, 65537, 65791])
def test_fk_ragged_sizes_and_invariants(n):
    require_gpu()
    robot = W.arm7(16)
    q = np.random.default_rng(n).uniform(-np.pi, np.pi, size=(n, 7)).astype(np.float32)
    got = _check(robot, q)
    # midpoints (R4) and the rigid tool offset hold on the GPU output too
    assert np.allclose(np.linalg.norm(got[:, 15] - got[:, 13], axis=1), np.float32(W.TOOL_OFFSET), atol=1e-6)


def test_fk_strides_base_and_frame0():
    require_gpu()
    import torch
    import paper_1910_06451_b200 as fb
    base = np.array([[0, -1, 0, 0.2], [1, 0, 0, -0.1], [0, 0, 1, 0.3]], dtype=np.float64)
    robot = W.make_robot("b", W.arm7(8).dh, [0, 3, 7, 7, 2], [[0.1, 0.2, 0.3], [0, 0, 0], [0, 0, 0.1], [0.05, 0, 0],
                                                           [0, 0, 0]], base=base)
    q = np.random.default_rng(0).uniform(-np.pi, np.pi, size=(300, 9)).astype(np.float32)  # ldq = 9 > dof
    qd = dev(q)
    pos = torch.full((5, 320, 4), 7.0, device="cuda")  # ldpos = 320 > n
    fb.fastron_fk(robot, qd, pos=pos)
    torch.cuda.synchronize()
    got = np.transpose(pos.cpu().numpy()[:, :300, :3], (1, 0, 2)).astype(np.float64)
    ref = oracle.fk(robot, np.ascontiguousarray(q[:, :7]))
    assert np.abs(got - ref).max() <= 1e-6
    assert np.all(pos.cpu().numpy()[:, 300:, :] == 7.0)  # padding columns untouched


def test_fk_planar_spec_examples():
    require_gpu()
    robot = W.planar_2link()
    q = np.array([[0, 0], [np.pi / 2, 0], [np.pi / 2, np.pi / 2]], dtype=np.float32)
    got = positions_np(_fk(robot, q))
    np.testing.assert_allclose(got[:, 1], [[2, 0, 0], [0, 2, 0], [-1, 1, 0]], atol=3e-7)


def test_fk_maximum_dof_and_control_points():
    """D = 16 joints with random theta offsets, d, a and alpha (any real alpha, not only
    0 / +-pi/2) and M = 32 control points on random frames with random offsets: the
    largest robot the ABI accepts."""
    require_gpu()
    rng = np.random.default_rng(16)
    dh = np.stack([rng.uniform(-1, 1, 16), rng.uniform(-0.2, 0.2, 16), rng.uniform(-0.2, 0.2, 16),
                   rng.uniform(-np.pi, np.pi, 16)], axis=1)
    robot = W.make_robot("d16m32", dh, rng.integers(0, 17, size=32), rng.uniform(-0.1, 0.1, size=(32, 3)))
    q = rng.uniform(-np.pi, np.pi, size=(777, 16)).astype(np.float32)
    _check(robot, q)


def test_fk_large_angles():
    """Joint values far outside [-pi, pi]: the table sincos's Cody-Waite reduction (|k pi/64|
    up to ~5e4 rad here) and, past 1e6 multiples of pi/64, its fall-back to the library
    sincos keep positions within one fp32 ulp of the oracle."""
    require_gpu()
    robot = W.arm7(8)
    rng = np.random.default_rng(7)
    q = np.concatenate([rng.uniform(-1000, 1000, size=(500, 7)), rng.uniform(-5e4, 5e4, size=(200, 7)),
                        rng.uniform(2e4, 2.5e4, size=(100, 7)) * rng.choice([-1, 1], size=(100, 7)),
                        np.full((1, 7), np.float32(np.pi)), np.full((1, 7), np.float32(-np.pi / 2))]).astype(np.float32)
    _check(robot, q, atol=2e-6)
