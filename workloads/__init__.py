"""Seeded synthetic workload generators shared by tests, bench.py and the oracle harness.

This module holds NONE of the method's arithmetic (no forward kinematics, no kernel,
no Fastron update). It draws robot descriptions, configurations, weights, edges and
obstacle scenes with numpy PCG64, and provides the cfg3 workload labeller, a pure
geometry routine (capsule vs axis-aligned cube) that takes segment end points as input
— whoever calls it supplies the control-point positions (the oracle's FK in tests, the
product's FK in bench.py).

Recipes follow BASELINE.json `configs` and the readings in DESIGN.md §3 (R4, R7, R12,
R14, R15, R21). Every array is generated in float64 and rounded once to float32 (R15);
the oracle promotes those exact float32 values back to float64.

Seeds: cfg k uses numpy.random.default_rng(k); the headline uses 6. The 7-DOF arm
shared by cfg2–5 and the headline is always drawn from default_rng(2) (cfg2's seed).
Draw order inside a workload: robot -> supports -> alpha -> queries/edges/cubes ->
dataset. numpy's uniform/normal draws are sequential, so a smaller size of the same
workload is a prefix of the full one (used for oracle-sized parity subsets).
"""
from __future__ import annotations

import dataclasses
import math
from typing import Optional

import numpy as np

PI = math.pi
TOOL_OFFSET = 0.10  # R4: end effector = frame D translated 0.10 m along its z axis


@dataclasses.dataclass(frozen=True)
class Robot:
    """Standard-DH serial arm (Eq. 1-2) with control points.

    dh:        (D, 4) float32 rows (theta_offset, d, a, alpha)
    base:      (3, 4) float32 row-major affine wA_0
    cp_frame:  (M,) int32, frame index j_m in [0, D] (0 = base frame)
    cp_offset: (M, 3) float32, translation of T_m in frame j_m
    """

    name: str
    dh: np.ndarray
    base: np.ndarray
    cp_frame: np.ndarray
    cp_offset: np.ndarray

    @property
    def dof(self) -> int:
        return int(self.dh.shape[0])

    @property
    def n_cp(self) -> int:
        return int(self.cp_frame.shape[0])


def _f32(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64).astype(np.float32))


def make_robot(name, dh, cp_frame, cp_offset, base=None) -> Robot:
    if base is None:
        base = np.eye(3, 4)
    return Robot(name=name, dh=_f32(dh), base=_f32(base),
                 cp_frame=np.ascontiguousarray(np.asarray(cp_frame, dtype=np.int32)),
                 cp_offset=_f32(np.asarray(cp_offset, dtype=np.float64).reshape(-1, 3)))


def planar_2link(a1: float = 1.0, a2: float = 1.0) -> Robot:
    """SPEC.md:72-74 planar 2-link arm (a1, a2, all other DH constants 0); control
    points at both joint origins (T_m = I at each joint frame)."""
    dh = [[0.0, 0.0, a1, 0.0], [0.0, 0.0, a2, 0.0]]
    return make_robot("planar2", dh, [1, 2], np.zeros((2, 3)))


def arm3(rng: np.random.Generator) -> Robot:
    """cfg1: 3-DOF spatial arm, a_i ~ U[0.3, 0.5], d_i = 0, alpha_i uniform over
    {0, +pi/2, -pi/2} (R7). Control points O_1, O_2, O_3 and the end effector (R4): M = 4."""
    a = rng.uniform(0.3, 0.5, size=3)
    alpha = rng.choice(np.array([0.0, PI / 2, -PI / 2]), size=3)
    dh = np.stack([np.zeros(3), np.zeros(3), a, alpha], axis=1)
    cp_frame = [1, 2, 3, 3]
    cp_offset = [[0, 0, 0], [0, 0, 0], [0, 0, 0], [0, 0, TOOL_OFFSET]]
    return make_robot("arm3", dh, cp_frame, cp_offset)


def _arm7_draw(rng: np.random.Generator):
    d = rng.uniform(0.1, 0.4, size=7)
    a_draw = rng.uniform(0.1, 0.4, size=7)
    return d, a_draw


ARM7_ALPHA = (-PI / 2, PI / 2, -PI / 2, PI / 2, -PI / 2, PI / 2, 0.0)


def arm7(n_cp: int = 8) -> Robot:
    """cfg2-5 and the headline: one shared Baxter-like 7-DOF arm drawn from
    default_rng(2) (R7): alpha = (-,+,-,+,-,+,0)*pi/2, d_i ~ U[0.1, 0.4],
    a_i ~ U[0.1, 0.4] for odd i (1-based), 0 for even i.

    n_cp = 8: O_1..O_7 + end effector (R4).
    n_cp = 16: for each of the 8 rigid segments O_{i-1}->O_i (i = 1..7) and O_7->EE,
    its midpoint and its distal end (R4). The midpoint of link i is static in frame i
    at 1/2 * (-a_i, -d_i sin alpha_i, -d_i cos alpha_i) (the position of O_{i-1} in
    frame i, halved); the tool midpoint is at 1/2 * (0, 0, TOOL_OFFSET) in frame 7.
    """
    d, a_draw = _arm7_draw(np.random.default_rng(2))
    a = np.where(np.arange(1, 8) % 2 == 1, a_draw, 0.0)
    alpha = np.asarray(ARM7_ALPHA)
    dh = np.stack([np.zeros(7), d, a, alpha], axis=1)
    if n_cp == 8:
        cp_frame = [1, 2, 3, 4, 5, 6, 7, 7]
        cp_offset = np.zeros((8, 3))
        cp_offset[7, 2] = TOOL_OFFSET
        name = "arm7_m8"
    elif n_cp == 16:
        # offsets from the float32-rounded DH values the kernels see
        dh32 = dh.astype(np.float32).astype(np.float64)
        cp_frame, cp_offset = [], []
        for i in range(7):
            di, ai, ali = dh32[i, 1], dh32[i, 2], dh32[i, 3]
            cp_frame += [i + 1, i + 1]
            cp_offset += [[-0.5 * ai, -0.5 * di * math.sin(ali), -0.5 * di * math.cos(ali)], [0.0, 0.0, 0.0]]
        cp_frame += [7, 7]
        cp_offset += [[0.0, 0.0, 0.5 * TOOL_OFFSET], [0.0, 0.0, TOOL_OFFSET]]
        name = "arm7_m16"
    else:
        raise ValueError("arm7 supports n_cp in {8, 16}")
    return make_robot(name, dh, cp_frame, cp_offset)


def uniform_configs(rng: np.random.Generator, n: int, dof: int) -> np.ndarray:
    """Joint configurations U[-pi, pi]^D (all joints revolute, limits +-pi; R6)."""
    return _f32(rng.uniform(-PI, PI, size=(n, dof)))


def normal_alpha(rng: np.random.Generator, n: int) -> np.ndarray:
    return _f32(rng.standard_normal(n))


@dataclasses.dataclass
class ScoreWorkload:
    name: str
    robot: Robot
    kind: int  # 0 = Gaussian (north star), 1 = RQ (Eq. 3)
    gamma: float
    supports: np.ndarray  # (S, D) float32
    alpha: np.ndarray  # (S,) float32
    queries: np.ndarray  # (Q, D) float32


@dataclasses.dataclass
class EdgeWorkload:
    name: str
    robot: Robot
    kind: int
    gamma: float
    supports: np.ndarray
    alpha: np.ndarray
    qa: np.ndarray  # (E, D)
    qb: np.ndarray  # (E, D)
    n_interp: int


@dataclasses.dataclass
class TrainWorkload:
    name: str
    robot: Robot
    kind: int
    gamma: float
    X: np.ndarray  # (N, D)
    cubes: np.ndarray  # (6, 2, 3) float64 lo/hi corners
    radius: float
    beta: float
    iter_max: int
    s_max: int


GAUSSIAN, RQ = 0, 1


def score_workload(name: str, n_queries: Optional[int] = None, n_supports: Optional[int] = None,
                   kind: int = GAUSSIAN) -> ScoreWorkload:
    """cfg1, cfg2, cfg5 (scoring part) and the headline (R14: cfg2 arm, S=20k, Q=1M)."""
    table = {
        "cfg1": (1, 1_000, 10_000, 10.0),
        "cfg2": (2, 2_000, 1_000_000, 5.0),
        "cfg5": (5, 20_000, 10_000_000, 5.0),
        "headline": (6, 20_000, 1_000_000, 5.0),
    }
    seed, S, Q, gamma = table[name]
    rng = np.random.default_rng(seed)
    if name == "cfg1":
        robot = arm3(rng)
    else:
        if name == "cfg2":
            _arm7_draw(rng)  # cfg2's own stream draws the shared arm first
        robot = arm7(16 if name == "cfg5" else 8)
    S_full = S
    S = S if n_supports is None else min(n_supports, S_full)
    sup_full = rng.uniform(-PI, PI, size=(S_full, robot.dof))
    alpha_full = rng.standard_normal(S_full)
    Q = Q if n_queries is None else n_queries
    queries = uniform_configs(rng, Q, robot.dof)
    return ScoreWorkload(name, robot, kind, gamma, _f32(sup_full[:S]), _f32(alpha_full[:S]), queries)


def edge_workload(n_edges: Optional[int] = None, n_supports: Optional[int] = None, kind: int = GAUSSIAN) -> EdgeWorkload:
    """cfg4: 3,000 supports (alpha ~ N(0,1), gamma = 5), 10,000 random edges with both
    endpoints uniform, 64 interpolated configurations per edge, t = k/63 (R11)."""
    rng = np.random.default_rng(4)
    robot = arm7(8)
    S_full, E_full = 3_000, 10_000
    sup = rng.uniform(-PI, PI, size=(S_full, 7))
    alpha = rng.standard_normal(S_full)
    E = E_full if n_edges is None else n_edges
    ends = rng.uniform(-PI, PI, size=(E, 2, 7))
    S = S_full if n_supports is None else min(n_supports, S_full)
    return EdgeWorkload("cfg4", robot, kind, 5.0, _f32(sup[:S]), _f32(alpha[:S]),
                        _f32(ends[:, 0]), _f32(ends[:, 1]), 64)


def random_cubes(rng: np.random.Generator, n: int = 6, keep_out: float = 0.15) -> np.ndarray:
    """R12: n axis-aligned cubes, side U[0.1, 0.3] m, centre U([-0.5, 0.5]^3);
    a cube is redrawn while it comes within `keep_out` of the base origin.
    Returns (n, 2, 3) float64 [lo, hi] corners."""
    cubes = []
    while len(cubes) < n:
        side = rng.uniform(0.1, 0.3)
        c = rng.uniform(-0.5, 0.5, size=3)
        lo, hi = c - side / 2, c + side / 2
        gap = np.maximum(np.maximum(lo, -hi), 0.0)  # distance of the origin to the box
        if np.sqrt(np.sum(gap * gap)) < keep_out:
            continue
        cubes.append(np.stack([lo, hi]))
    return np.asarray(cubes)


def train_workload(n: Optional[int] = None) -> TrainWorkload:
    """cfg3: 5,000 uniform 7-DOF configurations, labelled by the capsule-vs-6-cubes
    labeller (R12; capsule radius 0.05 m on the R4 segments), Gram 5,000^2 fp32 + Alg. 1
    with beta = 1, iter_max = 20,000, S_max = N, cold start (R10)."""
    rng = np.random.default_rng(3)
    robot = arm7(8)
    cubes = random_cubes(rng)
    N_full = 5_000
    X = rng.uniform(-PI, PI, size=(N_full, 7))
    N = N_full if n is None else n
    return TrainWorkload("cfg3", robot, GAUSSIAN, 5.0, _f32(X[:N]), cubes, 0.05, 1.0, 20_000, N)


def cfg5_gram_workload(n: Optional[int] = None):
    """cfg5 Gram rebuild (R21): 6 cubes, 3 of them moved by 0.1 m in seeded random
    directions, then a fresh seeded set of 20,000 configurations whose M=16 Gram is
    rebuilt. Returns (robot, X, cubes_before, cubes_after)."""
    rng = np.random.default_rng(55)
    robot = arm7(16)
    cubes = random_cubes(rng)
    moved = cubes.copy()
    for j in rng.choice(6, size=3, replace=False):
        v = rng.standard_normal(3)
        moved[j] += 0.1 * v / np.linalg.norm(v)
    N_full = 20_000
    X = rng.uniform(-PI, PI, size=(N_full, 7))
    N = N_full if n is None else n
    return robot, _f32(X[:N]), cubes, moved


# ---------------------------------------------------------------------------------
# Workload labeller (R12): capsule (segment + radius) vs axis-aligned box, exact.
# Pure geometry on caller-supplied segment end points; not part of the method.
# ---------------------------------------------------------------------------------

def segment_box_dist2(p0: np.ndarray, p1: np.ndarray, lo: np.ndarray, hi: np.ndarray) -> np.ndarray:
    """Exact min over t in [0,1] of dist^2(p0 + t (p1 - p0), box[lo, hi]).

    dist^2(t) is convex and piecewise quadratic, with breakpoints where a coordinate
    crosses a slab face. Split [0,1] at those (<= 6) breakpoints; on each piece the
    active faces are fixed, so the piece is A t^2 + B t + C, minimised in closed form.
    Shapes broadcast: p0, p1 (..., 3); lo, hi (..., 3).
    """
    p0, p1, lo, hi = np.broadcast_arrays(p0, p1, lo, hi)
    dv = p1 - p0
    with np.errstate(divide="ignore", invalid="ignore"):
        tb = np.concatenate([(lo - p0) / dv, (hi - p0) / dv], axis=-1)  # (..., 6)
    tb = np.where(np.isfinite(tb), np.clip(tb, 0.0, 1.0), 1.0)
    zeros = np.zeros(tb.shape[:-1] + (1,))
    ones = np.ones(tb.shape[:-1] + (1,))
    ts = np.sort(np.concatenate([zeros, tb, ones], axis=-1), axis=-1)  # (..., 8)
    best = None
    for k in range(7):
        ta, tc = ts[..., k], ts[..., k + 1]
        tm = 0.5 * (ta + tc)
        pm = p0 + tm[..., None] * dv
        below = pm < lo
        above = pm > hi
        bound = np.where(below, lo, np.where(above, hi, 0.0))
        active = below | above
        e = np.where(active, p0 - bound, 0.0)  # p(t) - bound = e + t dv
        w = np.where(active, dv, 0.0)
        A = np.sum(w * w, axis=-1)
        B = 2.0 * np.sum(w * e, axis=-1)
        C = np.sum(e * e, axis=-1)
        with np.errstate(divide="ignore", invalid="ignore"):
            tstar = np.where(A > 0, -B / (2.0 * np.where(A > 0, A, 1.0)), ta)
        tstar = np.clip(tstar, ta, tc)
        val = np.maximum(A * tstar * tstar + B * tstar + C, 0.0)
        best = val if best is None else np.minimum(best, val)
    return best


def capsule_aabb_labels(points: np.ndarray, cubes: np.ndarray, radius: float) -> np.ndarray:
    """Collision labels (+1 = C_obs) for configurations whose chain of
    points (N, P, 3) — base origin first, then the control points along the arm —
    defines P-1 capsules of `radius`. Tangency counts as collision (<= r^2)."""
    p0 = points[:, :-1, None, :]  # (N, P-1, 1, 3)
    p1 = points[:, 1:, None, :]
    lo = cubes[None, None, :, 0, :]
    hi = cubes[None, None, :, 1, :]
    d2 = segment_box_dist2(p0, p1, lo, hi)  # (N, P-1, n_cubes)
    hit = np.any(d2 <= radius * radius, axis=(1, 2))
    return np.where(hit, 1, -1).astype(np.int8)


def chain_points(cp_pos: np.ndarray, base_origin=(0.0, 0.0, 0.0)) -> np.ndarray:
    """(N, M, 3) control-point positions of an R4 arm (O_1..O_D, EE) -> (N, M+1, 3)
    with the base origin prepended, i.e. the capsule chain O_0 -> O_1 -> ... -> EE."""
    n = cp_pos.shape[0]
    base = np.broadcast_to(np.asarray(base_origin, dtype=np.float64), (n, 1, 3))
    return np.concatenate([base, cp_pos.astype(np.float64)], axis=1)
