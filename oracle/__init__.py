"""ctypes wrapper of oracle/liboracle.so — the fp64 CPU oracle (TEST INFRASTRUCTURE).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / `--impl reference`
legs may import this package. It shares no code with paper_1910_06451_b200/ and never
imports it. See oracle/oracle.c for the per-function citations of PAPER.md.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

GAUSSIAN, RQ = 0, 1

BUILD_CMD = ["gcc", "-O2", "-ffp-contract=off", "-fopenmp", "-Wall", "-shared", "-fPIC", _SRC, "-o", _LIB, "-lm"]


def build(force: bool = False) -> str:
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(BUILD_CMD)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        dp = ctypes.POINTER(ctypes.c_double)
        fp = ctypes.POINTER(ctypes.c_float)
        ip = ctypes.POINTER(ctypes.c_int32)
        i8 = ctypes.POINTER(ctypes.c_int8)
        u8 = ctypes.POINTER(ctypes.c_uint8)
        i64 = ctypes.c_int64
        L.oracle_dh_transform.argtypes = [ctypes.c_double] * 4 + [dp]
        L.oracle_dh_transform.restype = None
        L.oracle_joint_poses.argtypes = [ctypes.c_int, dp, dp, fp, dp]
        L.oracle_joint_poses.restype = None
        L.oracle_fk.argtypes = [ctypes.c_int, dp, dp, ctypes.c_int, ip, dp, fp, i64, i64, dp]
        L.oracle_fk.restype = None
        L.oracle_rbf_term.argtypes = [ctypes.c_int, ctypes.c_double, ctypes.c_double]
        L.oracle_rbf_term.restype = ctypes.c_double
        L.oracle_kernel_value.argtypes = [ctypes.c_int, ctypes.c_double, ctypes.c_int, dp, dp]
        L.oracle_kernel_value.restype = ctypes.c_double
        L.oracle_score.argtypes = [ctypes.c_int, ctypes.c_double, ctypes.c_int, dp, i64, dp, dp, i64, dp, i8]
        L.oracle_score.restype = None
        L.oracle_gram.argtypes = [ctypes.c_int, ctypes.c_double, ctypes.c_int, dp, i64, dp]
        L.oracle_gram.restype = None
        L.oracle_loss.argtypes = [dp, i64, i8, ctypes.c_double, dp]
        L.oracle_loss.restype = ctypes.c_double
        L.oracle_train.argtypes = [dp, i64, i8, ctypes.c_double, i64, i64, dp, dp, ip, dp, ip,
                                   ctypes.POINTER(ctypes.c_int64)]
        L.oracle_train.restype = None
        L.oracle_edge.argtypes = [ctypes.c_int, dp, dp, ctypes.c_int, ip, dp, fp, fp, i64, ctypes.c_int,
                                  ctypes.c_int, ctypes.c_double, dp, dp, i64, u8, dp, dp]
        L.oracle_edge.restype = None
        L.oracle_joint_kernel.argtypes = [ctypes.c_int, ctypes.c_double, ctypes.c_int, fp, fp]
        L.oracle_joint_kernel.restype = ctypes.c_double
        L.oracle_score_joint.argtypes = [ctypes.c_int, ctypes.c_double, ctypes.c_int, fp, i64, i64, fp, i64, i64, dp, dp,
                                         i8]
        L.oracle_score_joint.restype = None
        L.oracle_gram_joint.argtypes = [ctypes.c_int, ctypes.c_double, ctypes.c_int, fp, i64, i64, dp]
        L.oracle_gram_joint.restype = None
        L.oracle_num_threads.argtypes = []
        L.oracle_num_threads.restype = ctypes.c_int
        L.oracle_set_num_threads.argtypes = [ctypes.c_int]
        L.oracle_set_num_threads.restype = None
        _lib = L
    return _lib


def _p(a, ct):
    return a.ctypes.data_as(ctypes.POINTER(ct)) if a is not None else None


def _robot_arrays(robot):
    dh = np.ascontiguousarray(np.asarray(robot.dh, dtype=np.float32).astype(np.float64))
    base = np.ascontiguousarray(np.asarray(robot.base, dtype=np.float32).astype(np.float64))
    cpf = np.ascontiguousarray(np.asarray(robot.cp_frame, dtype=np.int32))
    cpo = np.ascontiguousarray(np.asarray(robot.cp_offset, dtype=np.float32).astype(np.float64))
    return dh, base, cpf, cpo


def num_threads() -> int:
    return int(lib().oracle_num_threads())


def set_num_threads(n: int) -> None:
    """OpenMP thread count of the oracle loops (timing only)."""
    lib().oracle_set_num_threads(int(n))


def dh_transform(theta, d, a, alpha) -> np.ndarray:
    out = np.zeros(16)
    lib().oracle_dh_transform(float(theta), float(d), float(a), float(alpha), _p(out, ctypes.c_double))
    return out.reshape(4, 4)


def joint_poses(robot, q) -> np.ndarray:
    """(D+1, 4, 4) poses wA_0..wA_D of one fp32 configuration."""
    dh, base, _, _ = _robot_arrays(robot)
    q = np.ascontiguousarray(np.asarray(q, dtype=np.float32))
    out = np.zeros((robot.dof + 1) * 16)
    lib().oracle_joint_poses(robot.dof, _p(dh, ctypes.c_double), _p(base, ctypes.c_double), _p(q, ctypes.c_float),
                             _p(out, ctypes.c_double))
    return out.reshape(-1, 4, 4)


def fk(robot, q) -> np.ndarray:
    """Control-point positions (N, M, 3) float64 of fp32 configurations q (N, D)."""
    dh, base, cpf, cpo = _robot_arrays(robot)
    q = np.ascontiguousarray(np.asarray(q, dtype=np.float32).reshape(-1, robot.dof))
    n = q.shape[0]
    pos = np.zeros((n, robot.n_cp, 3))
    lib().oracle_fk(robot.dof, _p(dh, ctypes.c_double), _p(base, ctypes.c_double), robot.n_cp, _p(cpf, ctypes.c_int32),
                    _p(cpo, ctypes.c_double), _p(q, ctypes.c_float), n, robot.dof, _p(pos, ctypes.c_double))
    return pos


def rbf_term(kind, gamma, d2) -> float:
    return float(lib().oracle_rbf_term(int(kind), float(gamma), float(d2)))


def kernel_value(kind, gamma, u, v) -> float:
    u = np.ascontiguousarray(np.asarray(u, dtype=np.float64).reshape(-1, 3))
    v = np.ascontiguousarray(np.asarray(v, dtype=np.float64).reshape(-1, 3))
    return float(lib().oracle_kernel_value(int(kind), float(gamma), u.shape[0], _p(u, ctypes.c_double),
                                           _p(v, ctypes.c_double)))


def score(kind, gamma, qpos, spos, alpha, exact_alpha=False):
    """f (nq,) float64 and labels (nq,) int8 for positions qpos (nq, M, 3), spos (ns, M, 3).
    alpha is taken as fp32 values (the inputs of the fp32 path) unless exact_alpha, when
    fp64 weights are used unrounded (the fp64 path scores Algorithm 1's fp64 alpha)."""
    qpos = np.ascontiguousarray(np.asarray(qpos, dtype=np.float64))
    spos = np.ascontiguousarray(np.asarray(spos, dtype=np.float64))
    alpha = np.ascontiguousarray(np.asarray(alpha, dtype=np.float64) if exact_alpha else
                                 np.asarray(alpha, dtype=np.float32).astype(np.float64))
    nq, M = qpos.shape[0], qpos.shape[1]
    ns = spos.shape[0]
    f = np.zeros(nq)
    lab = np.zeros(nq, dtype=np.int8)
    lib().oracle_score(int(kind), float(gamma), M, _p(qpos, ctypes.c_double), nq, _p(spos, ctypes.c_double),
                       _p(alpha, ctypes.c_double), ns, _p(f, ctypes.c_double), _p(lab, ctypes.c_int8))
    return f, lab


def gram(kind, gamma, pos) -> np.ndarray:
    pos = np.ascontiguousarray(np.asarray(pos, dtype=np.float64))
    n, M = pos.shape[0], pos.shape[1]
    K = np.zeros((n, n))
    lib().oracle_gram(int(kind), float(gamma), M, _p(pos, ctypes.c_double), n, _p(K, ctypes.c_double))
    return K


def loss(K, y, beta, alpha) -> float:
    K = np.ascontiguousarray(K, dtype=np.float64)
    y = np.ascontiguousarray(y, dtype=np.int8)
    alpha = np.ascontiguousarray(alpha, dtype=np.float64)
    return float(lib().oracle_loss(_p(K, ctypes.c_double), K.shape[0], _p(y, ctypes.c_int8), float(beta),
                                   _p(alpha, ctypes.c_double)))


def train(K, y, beta=1.0, iter_max=20000, s_max=None, alpha0=None, F0=None, with_loss=False):
    """Algorithm 1 on a dense fp64 K. Returns a dict with alpha, F,
    trace (int32), loss_trace (or None), support (int32), iterations, n_add, n_remove,
    converged, n_support."""
    K = np.ascontiguousarray(K, dtype=np.float64)
    n = K.shape[0]
    y = np.ascontiguousarray(y, dtype=np.int8)
    s_max = n if s_max is None else int(s_max)
    alpha = np.zeros(n) if alpha0 is None else np.array(alpha0, dtype=np.float64, copy=True)
    F = np.zeros(n) if F0 is None else np.array(F0, dtype=np.float64, copy=True)
    trace = np.zeros(max(iter_max, 1), dtype=np.int32)
    lt = np.zeros(iter_max + 1) if with_loss else None
    sup = np.zeros(max(n, 1), dtype=np.int32)
    out = (ctypes.c_int64 * 5)()
    lib().oracle_train(_p(K, ctypes.c_double), n, _p(y, ctypes.c_int8), float(beta), int(iter_max), s_max,
                       _p(alpha, ctypes.c_double), _p(F, ctypes.c_double), _p(trace, ctypes.c_int32),
                       _p(lt, ctypes.c_double), _p(sup, ctypes.c_int32), out)
    it = int(out[0])
    return dict(alpha=alpha, F=F, trace=trace[:it].copy(), loss_trace=None if lt is None else lt[:it + 1].copy(),
                support=sup[:int(out[4])].copy(), iterations=it, n_add=int(out[1]), n_remove=int(out[2]),
                converged=bool(out[3]), n_support=int(out[4]))


def edge(robot, qa, qb, n_interp, kind, gamma, spos, alpha, with_all=False):
    """Per-edge any-in-collision (E,) uint8, max_k f (E,), and optionally all (E, n_interp) scores."""
    dh, base, cpf, cpo = _robot_arrays(robot)
    qa = np.ascontiguousarray(np.asarray(qa, dtype=np.float32))
    qb = np.ascontiguousarray(np.asarray(qb, dtype=np.float32))
    spos = np.ascontiguousarray(np.asarray(spos, dtype=np.float64))
    alpha = np.ascontiguousarray(np.asarray(alpha, dtype=np.float32).astype(np.float64))
    if qa.shape != qb.shape or qa.ndim != 2 or qa.shape[1] != robot.dof:
        raise ValueError("qa, qb must both be (E, D)")
    E = qa.shape[0]
    hit = np.zeros(E, dtype=np.uint8)
    fmax = np.zeros(E)
    fall = np.zeros((E, n_interp)) if with_all else None
    lib().oracle_edge(robot.dof, _p(dh, ctypes.c_double), _p(base, ctypes.c_double), robot.n_cp,
                      _p(cpf, ctypes.c_int32), _p(cpo, ctypes.c_double), _p(qa, ctypes.c_float), _p(qb, ctypes.c_float),
                      E, int(n_interp), int(kind), float(gamma), _p(spos, ctypes.c_double), _p(alpha, ctypes.c_double),
                      spos.shape[0], _p(hit, ctypes.c_uint8), _p(fmax, ctypes.c_double), _p(fall, ctypes.c_double))
    return hit, fmax, fall


def joint_kernel(kind, gamma, x, xp) -> float:
    x = np.ascontiguousarray(np.asarray(x, dtype=np.float32))
    xp = np.ascontiguousarray(np.asarray(xp, dtype=np.float32))
    return float(lib().oracle_joint_kernel(int(kind), float(gamma), x.shape[0], _p(x, ctypes.c_float),
                                           _p(xp, ctypes.c_float)))


def score_joint(kind, gamma, q, s, alpha):
    """Joint-space RBF ("Fastron RBF") scores of fp32 configurations q (nq, D) vs supports s (ns, D)."""
    q = np.ascontiguousarray(np.asarray(q, dtype=np.float32))
    s = np.ascontiguousarray(np.asarray(s, dtype=np.float32))
    alpha = np.ascontiguousarray(np.asarray(alpha, dtype=np.float32).astype(np.float64))
    nq, D = q.shape
    ns = s.shape[0]
    f = np.zeros(nq)
    lab = np.zeros(nq, dtype=np.int8)
    lib().oracle_score_joint(int(kind), float(gamma), D, _p(q, ctypes.c_float), nq, D, _p(s, ctypes.c_float), ns, D,
                             _p(alpha, ctypes.c_double), _p(f, ctypes.c_double), _p(lab, ctypes.c_int8))
    return f, lab


def gram_joint(kind, gamma, x) -> np.ndarray:
    x = np.ascontiguousarray(np.asarray(x, dtype=np.float32))
    n, D = x.shape
    K = np.zeros((n, n))
    lib().oracle_gram_joint(int(kind), float(gamma), D, _p(x, ctypes.c_float), n, D, _p(K, ctypes.c_double))
    return K
