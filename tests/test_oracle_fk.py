"""Pins of the oracle's forward kinematics (Eq. 1-2) against things
other than itself: the D-H convention's definition as a product of elementary
transforms, SPEC's worked examples, textbook closed forms, and invariants."""
import json
import math
import os

import numpy as np
import pytest

import oracle
import workloads as W

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def rz(t):
    c, s = math.cos(t), math.sin(t)
    return np.array([[c, -s, 0, 0], [s, c, 0, 0], [0, 0, 1, 0], [0, 0, 0, 1.0]])


def rx(t):
    c, s = math.cos(t), math.sin(t)
    return np.array([[1, 0, 0, 0], [0, c, -s, 0], [0, s, c, 0], [0, 0, 0, 1.0]])


def trans(x, y, z):
    T = np.eye(4)
    T[:3, 3] = (x, y, z)
    return T


def test_dh_transform_is_the_standard_dh_product():
    """Standard D-H: A = Rot_z(theta) Trans_z(d) Trans_x(a) Rot_x(alpha); Eq. 1 is its
    expansion. A transposed block or a swapped d/a fails this."""
    rng = np.random.default_rng(0)
    for _ in range(200):
        th, d, a, al = rng.uniform(-4, 4), rng.uniform(-1, 1), rng.uniform(-1, 1), rng.uniform(-4, 4)
        ref = rz(th) @ trans(0, 0, d) @ trans(a, 0, 0) @ rx(al)
        np.testing.assert_allclose(oracle.dh_transform(th, d, a, al), ref, atol=1e-14)


def test_dh_examples_spec():
    g = json.load(open(os.path.join(GOLD, "dh_examples.json")))
    for c in g["cases"]:
        np.testing.assert_allclose(oracle.dh_transform(c["theta"], c["d"], c["a"], c["alpha"]), np.array(c["T"]),
                                   atol=1e-15, err_msg=c["note"])


def test_planar_2link_spec_examples():
    g = json.load(open(os.path.join(GOLD, "planar_2link.json")))
    robot = W.planar_2link(g["robot"]["a1"], g["robot"]["a2"])
    for c in g["cases"]:
        pos = oracle.fk(robot, np.array([c["q"]], dtype=np.float32))[0]
        # fp32 inputs: pi/2 in float32 is off by 4.4e-8 rad -> positions off by <= 1e-7
        np.testing.assert_allclose(pos[1], c["O2"], atol=2e-7)
        if "control_points" in c:
            np.testing.assert_allclose(pos, c["control_points"], atol=1e-15)


def test_planar_2link_closed_form_random():
    """Textbook planar 2R: O1 = a1 (c1, s1, 0), O2 = O1 + a2 (c12, s12, 0)."""
    rng = np.random.default_rng(1)
    a1, a2 = 0.7, 0.45
    robot = W.planar_2link(a1, a2)
    q = rng.uniform(-np.pi, np.pi, size=(500, 2)).astype(np.float32)
    pos = oracle.fk(robot, q)
    t1, t2 = q[:, 0].astype(np.float64), q[:, 1].astype(np.float64)
    a1f, a2f = float(np.float32(a1)), float(np.float32(a2))
    O1 = np.stack([a1f * np.cos(t1), a1f * np.sin(t1), 0 * t1], 1)
    O2 = O1 + np.stack([a2f * np.cos(t1 + t2), a2f * np.sin(t1 + t2), 0 * t1], 1)
    np.testing.assert_allclose(pos[:, 0], O1, atol=1e-14)
    np.testing.assert_allclose(pos[:, 1], O2, atol=1e-14)


def test_elbow_manipulator_closed_form():
    """Textbook 3-DOF articulated (elbow) arm, D-H rows (th1, d1, 0, +pi/2),
    (th2, 0, a2, 0), (th3, 0, a3, 0): the wrist centre is
    (c1 (a2 c2 + a3 c23), s1 (a2 c2 + a3 c23), d1 + a2 s2 + a3 s23).
    Exercises the alpha != 0 entries of Eq. 1 that the planar arm leaves at 0."""
    d1, a2, a3 = 0.3, 0.5, 0.4
    robot = W.make_robot("elbow", [[0, d1, 0, np.pi / 2], [0, 0, a2, 0], [0, 0, a3, 0]], [3], [[0, 0, 0]])
    rng = np.random.default_rng(2)
    q = rng.uniform(-np.pi, np.pi, size=(500, 3)).astype(np.float32)
    p = oracle.fk(robot, q)[:, 0]
    t = q.astype(np.float64)
    d1f, a2f, a3f = (float(np.float32(v)) for v in (d1, a2, a3))
    al = float(np.float32(np.pi / 2))
    # alpha is the fp32-rounded pi/2: cos(alpha) = -4.4e-8, which the closed form ignores
    r = a2f * np.cos(t[:, 1]) + a3f * np.cos(t[:, 1] + t[:, 2])
    ref = np.stack([np.cos(t[:, 0]) * r, np.sin(t[:, 0]) * r,
                    d1f + a2f * np.sin(t[:, 1]) + a3f * np.sin(t[:, 1] + t[:, 2])], 1)
    assert abs(math.cos(al)) < 1e-7
    np.testing.assert_allclose(p, ref, atol=1e-7)


@pytest.mark.parametrize("robot", [W.arm3(np.random.default_rng(1)), W.arm7(8), W.arm7(16)], ids=lambda r: r.name)
def test_link_length_and_orthonormality_invariants(robot):
    """||O_i - O_{i-1}||^2 = a_i^2 + d_i^2 for every configuration (the translation
    column of Eq. 1 has norm sqrt(a^2 + d^2) and the chain rotations are orthonormal);
    rotations stay orthonormal with det +1."""
    rng = np.random.default_rng(3)
    for _ in range(50):
        q = rng.uniform(-np.pi, np.pi, size=robot.dof).astype(np.float32)
        P = oracle.joint_poses(robot, q)
        for i in range(1, robot.dof + 1):
            d, a = float(robot.dh[i - 1, 1]), float(robot.dh[i - 1, 2])
            gap = P[i, :3, 3] - P[i - 1, :3, 3]
            assert abs(gap @ gap - (a * a + d * d)) < 1e-13
            R = P[i, :3, :3]
            np.testing.assert_allclose(R.T @ R, np.eye(3), atol=1e-13)
            assert abs(np.linalg.det(R) - 1.0) < 1e-13


def test_control_points_are_joint_origins_and_tool():
    """PAPER.md:139 (T_m = I at joint origins) and R4's tool point: the M=8 arm's
    control points are O_1..O_7 and a point 0.10 m from O_7."""
    robot = W.arm7(8)
    rng = np.random.default_rng(4)
    q = rng.uniform(-np.pi, np.pi, size=(20, 7)).astype(np.float32)
    pos = oracle.fk(robot, q)
    for k in range(20):
        P = oracle.joint_poses(robot, q[k])
        np.testing.assert_allclose(pos[k, :7], P[1:8, :3, 3], atol=1e-15)
        assert abs(np.linalg.norm(pos[k, 7] - pos[k, 6]) - np.float32(W.TOOL_OFFSET)) < 1e-9


def test_m16_midpoints_are_segment_midpoints():
    """R4 reading for cfg5: the static offset 1/2 (-a, -d sin(alpha), -d cos(alpha)) in
    frame i is the midpoint of O_{i-1} O_i, for any configuration."""
    robot = W.arm7(16)
    rng = np.random.default_rng(5)
    q = rng.uniform(-np.pi, np.pi, size=(20, 7)).astype(np.float32)
    pos = oracle.fk(robot, q)
    for k in range(20):
        P = oracle.joint_poses(robot, q[k])
        O = P[:, :3, 3]
        for i in range(1, 8):
            np.testing.assert_allclose(pos[k, 2 * (i - 1)], 0.5 * (O[i - 1] + O[i]), atol=2e-8)
            np.testing.assert_allclose(pos[k, 2 * (i - 1) + 1], O[i], atol=1e-15)
        np.testing.assert_allclose(pos[k, 14], 0.5 * (O[7] + pos[k, 15]), atol=2e-8)


def test_base_transform_composes():
    """wA_i = wA_0 0A_1 ... ; a base rotation+translation moves every
    control point rigidly."""
    robot = W.arm3(np.random.default_rng(1))
    R = rz(0.7) @ rx(-0.3)
    base = R[:3, :4].copy()
    base[:, 3] = (0.1, -0.2, 0.3)
    moved = W.make_robot("moved", robot.dh, robot.cp_frame, robot.cp_offset, base=base)
    q = np.random.default_rng(6).uniform(-np.pi, np.pi, size=(30, 3)).astype(np.float32)
    p0 = oracle.fk(robot, q)
    p1 = oracle.fk(moved, q)
    b32 = moved.base.astype(np.float64)
    np.testing.assert_allclose(p1, p0 @ b32[:, :3].T + b32[:, 3], atol=1e-14)
