"""Thin Python binding of libfastron_b200.so (include/fastron.h).

Argument marshalling only: every step of the hot path runs in the library's sm_100a
kernels. PyTorch provides device memory and streams. The functions keep the C names
(fastron_fk, fastron_score, fastron_gram, fastron_train, fastron_edge_check,
fastron_query) and take torch tensors; outputs are allocated when not given.

There is no CPU fallback: importing this package without the built library, or
calling it without a CUDA device, raises.
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FASTRON_LIB", os.path.join(_HERE, "libfastron_b200.so"))

FASTRON_OK, FASTRON_ERR_INVALID_ARG, FASTRON_ERR_CUDA, FASTRON_ERR_WORKSPACE, FASTRON_ERR_UNSUPPORTED = range(5)
GAUSSIAN, RQ = 0, 1
MAX_DOF, MAX_CP = 16, 32

# Symbols declared in include/fastron.h (checked by tests/test_abi_cpu.py).
EXPORTED = [
    "fastron_fk", "fastron_score_workspace_bytes", "fastron_score", "fastron_gram_workspace_bytes", "fastron_gram",
    "fastron_train_max_n", "fastron_train", "fastron_edge_workspace_bytes", "fastron_edge_check",
    "fastron_query_workspace_bytes", "fastron_query", "fastron_last_error", "fastron_version",
    "fastron_launch_count", "fastron_model_bytes", "fastron_model_pack", "fastron_score_packed_workspace_bytes",
    "fastron_score_packed", "fastron_score_joint_workspace_bytes", "fastron_score_joint",
    "fastron_gram_joint_workspace_bytes", "fastron_gram_joint", "fastron_train_lazy_max_n",
    "fastron_train_lazy_workspace_bytes", "fastron_train_lazy", "fastron_active_samples", "fastron_label_capsules",
    "fastron_kernel_matvec", "fastron_score_packed_f64", "fastron_set_validation", "fastron_validation",
    "fastron_kernel_matvec_lazy_workspace_bytes", "fastron_kernel_matvec_lazy",
    "fastron_query_packed_workspace_bytes", "fastron_query_packed",
    "fastron_edge_packed_workspace_bytes", "fastron_edge_check_packed", "fastron_fk64", "fastron_score_precise",
]


class FastronError(RuntimeError):
    def __init__(self, status: int, message: str):
        super().__init__(f"fastron status {status}: {message}")
        self.status = status


class fastron_kernel(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("gamma", ctypes.c_float)]


class fastron_robot(ctypes.Structure):
    _fields_ = [
        ("dof", ctypes.c_int32),
        ("n_cp", ctypes.c_int32),
        ("dh", (ctypes.c_float * 4) * MAX_DOF),
        ("base", (ctypes.c_float * 4) * 3),
        ("cp_frame", ctypes.c_int32 * MAX_CP),
        ("cp_offset", (ctypes.c_float * 3) * MAX_CP),
    ]


class fastron_train_result(ctypes.Structure):
    _fields_ = [("iterations", ctypes.c_int64), ("n_add", ctypes.c_int64), ("n_remove", ctypes.c_int64),
                ("converged", ctypes.c_int32), ("n_support", ctypes.c_int32)]


_lib = None


def load_library(path: str = LIB_PATH):
    """Load the in-tree library (build it first with paper_1910_06451_b200._build)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path) and path == LIB_PATH:
        # a checkout without the built artefact (the .so is git-ignored): build it in-tree
        # with nvcc once; anything short of the real library is an error (no CPU fallback)
        try:
            from . import _build
            _build.build()
        except Exception as e:  # nvcc missing, compile error
            raise ImportError(f"{path} is missing and could not be built ({e}); build it with "
                              "`python -m paper_1910_06451_b200._build` (there is no CPU fallback)") from e
    if not os.path.exists(path):
        raise ImportError(f"{path} is missing: build it with `python -m paper_1910_06451_b200._build` "
                          "(there is no CPU fallback)")
    L = ctypes.CDLL(path)
    vp, i64, i32, sz = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_size_t
    st = ctypes.c_int
    rp = ctypes.POINTER(fastron_robot)
    L.fastron_fk.argtypes = [rp, vp, i64, i64, vp, i64, vp]
    L.fastron_score_workspace_bytes.argtypes = [i64, i64, i32]
    L.fastron_score_workspace_bytes.restype = sz
    L.fastron_score.argtypes = [vp, i64, i64, vp, vp, i64, i64, i32, fastron_kernel, vp, vp, vp, sz, vp]
    L.fastron_model_bytes.argtypes = [i64, i32]
    L.fastron_model_bytes.restype = sz
    L.fastron_model_pack.argtypes = [vp, vp, i64, i64, i32, fastron_kernel, vp, sz, vp]
    L.fastron_score_packed_workspace_bytes.argtypes = [i64, i64, i32]
    L.fastron_score_packed_workspace_bytes.restype = sz
    L.fastron_score_packed.argtypes = [vp, i64, i64, vp, i64, i32, fastron_kernel, vp, vp, vp, sz, vp]
    L.fastron_score_packed_f64.argtypes = [vp, i64, i64, vp, i64, i32, fastron_kernel, vp, vp, sz, vp]
    L.fastron_score_joint_workspace_bytes.argtypes = [i64, i64, i32]
    L.fastron_score_joint_workspace_bytes.restype = sz
    L.fastron_score_joint.argtypes = [vp, i64, i64, vp, vp, i64, i64, i32, fastron_kernel, vp, vp, vp, sz, vp]
    L.fastron_gram_joint_workspace_bytes.argtypes = [i64, i32]
    L.fastron_gram_joint_workspace_bytes.restype = sz
    L.fastron_gram_joint.argtypes = [vp, i64, i64, i32, fastron_kernel, vp, i64, vp, sz, vp]
    L.fastron_train_lazy_max_n.argtypes = [i32]
    L.fastron_train_lazy_max_n.restype = i64
    L.fastron_train_lazy_workspace_bytes.argtypes = [i64, i32, i64]
    L.fastron_train_lazy_workspace_bytes.restype = sz
    L.fastron_train_lazy.argtypes = [vp, i64, i64, i32, fastron_kernel, vp, ctypes.c_double, i64, i64, vp, vp, vp, vp,
                                     vp, i64, vp, sz, vp]
    L.fastron_active_samples.argtypes = [vp, i64, i64, i32, i32, vp, vp, vp, i64, vp, vp, vp, i64, vp]
    L.fastron_label_capsules.argtypes = [vp, i64, i64, vp, i32, vp, i32, ctypes.c_float, vp, vp]
    L.fastron_kernel_matvec.argtypes = [vp, i64, i64, vp, vp, vp]
    L.fastron_kernel_matvec_lazy_workspace_bytes.argtypes = [i64, i32]
    L.fastron_kernel_matvec_lazy_workspace_bytes.restype = sz
    L.fastron_kernel_matvec_lazy.argtypes = [vp, i64, i64, i32, fastron_kernel, vp, vp, vp, sz, vp]
    L.fastron_gram_workspace_bytes.argtypes = [i64, i32]
    L.fastron_gram_workspace_bytes.restype = sz
    L.fastron_gram.argtypes = [vp, i64, i64, i32, fastron_kernel, vp, i64, vp, sz, vp]
    L.fastron_train_max_n.argtypes = []
    L.fastron_train_max_n.restype = i64
    L.fastron_train.argtypes = [vp, i64, i64, vp, ctypes.c_double, i64, i64, vp, vp, vp, vp, vp, vp]
    L.fastron_edge_workspace_bytes.argtypes = [i64, i64, i32]
    L.fastron_edge_workspace_bytes.restype = sz
    L.fastron_edge_check.argtypes = [rp, vp, vp, i64, i64, i32, vp, vp, i64, i64, fastron_kernel, vp, vp, vp, sz, vp]
    L.fastron_fk64.argtypes = [rp, vp, i64, i64, vp, i64, vp]
    L.fastron_score_precise.argtypes = [vp, i64, i64, vp, vp, i64, i64, i32, fastron_kernel, vp, vp, vp]
    L.fastron_edge_packed_workspace_bytes.argtypes = [i64, i64, i32]
    L.fastron_edge_packed_workspace_bytes.restype = sz
    L.fastron_edge_check_packed.argtypes = [rp, vp, vp, i64, i64, i32, vp, i64, i32, fastron_kernel, vp, vp, vp, sz,
                                            vp]
    L.fastron_query_workspace_bytes.argtypes = [i64, i64, i32, i32]
    L.fastron_query_workspace_bytes.restype = sz
    L.fastron_query.argtypes = [rp, vp, i64, i64, vp, vp, i64, i64, fastron_kernel, vp, vp, vp, sz, vp]
    L.fastron_query_packed_workspace_bytes.argtypes = [i64, i64, i32, i32]
    L.fastron_query_packed_workspace_bytes.restype = sz
    L.fastron_query_packed.argtypes = [rp, vp, i64, i64, vp, i64, i32, fastron_kernel, vp, vp, vp, sz, vp]
    for f in ("fastron_fk", "fastron_score", "fastron_gram", "fastron_train", "fastron_edge_check", "fastron_query",
              "fastron_model_pack", "fastron_score_packed", "fastron_score_joint", "fastron_gram_joint", "fastron_train_lazy", "fastron_active_samples",
              "fastron_label_capsules", "fastron_kernel_matvec", "fastron_score_packed_f64",
              "fastron_kernel_matvec_lazy", "fastron_query_packed", "fastron_edge_check_packed", "fastron_fk64",
              "fastron_score_precise"):
        getattr(L, f).restype = st
    L.fastron_last_error.argtypes = []
    L.fastron_last_error.restype = ctypes.c_char_p
    L.fastron_version.argtypes = []
    L.fastron_version.restype = ctypes.c_char_p
    L.fastron_launch_count.argtypes = []
    L.fastron_launch_count.restype = i64
    L.fastron_set_validation.argtypes = [i32]
    L.fastron_set_validation.restype = None
    L.fastron_validation.argtypes = []
    L.fastron_validation.restype = i32
    _lib = L
    return L


def _check(status: int):
    if status != FASTRON_OK:
        raise FastronError(status, _lib.fastron_last_error().decode())


def make_robot_struct(robot) -> fastron_robot:
    """Marshal any object with dof, dh (D,4), base (3,4), cp_frame (M,), cp_offset (M,3)."""
    r = fastron_robot()
    dh = np.asarray(robot.dh, dtype=np.float32)
    D = dh.shape[0]
    cpf = np.asarray(robot.cp_frame, dtype=np.int32)
    cpo = np.asarray(robot.cp_offset, dtype=np.float32).reshape(-1, 3)
    M = cpf.shape[0]
    if not (1 <= D <= MAX_DOF and 1 <= M <= MAX_CP):
        raise ValueError("dof must be in [1,16] and n_cp in [1,32]")
    r.dof, r.n_cp = D, M
    for i in range(D):
        for c in range(4):
            r.dh[i][c] = float(dh[i, c])
    base = np.asarray(robot.base, dtype=np.float32)
    for i in range(3):
        for c in range(4):
            r.base[i][c] = float(base[i, c])
    for m in range(M):
        r.cp_frame[m] = int(cpf[m])
        for c in range(3):
            r.cp_offset[m][c] = float(cpo[m, c])
    return r


def _tstream(stream):
    """The torch stream the call enqueues on (current stream by default; a raw cudaStream_t
    handle is wrapped). Temporaries are allocated under it, so the caching allocator never
    hands their blocks to other work while the kernels still use them."""
    import torch
    if stream is None:
        return torch.cuda.current_stream()
    if isinstance(stream, torch.cuda.Stream):
        return stream
    return torch.cuda.ExternalStream(int(stream))


def _new(shape, dtype, device, ts):
    import torch
    with torch.cuda.stream(ts):
        return torch.empty(shape, dtype=dtype, device=device)


def _zeros(shape, dtype, device, ts):
    import torch
    with torch.cuda.stream(ts):
        return torch.zeros(shape, dtype=dtype, device=device)


def _ptr(t):
    return None if t is None else t.data_ptr()


def _kernel(kind: int, gamma: float) -> fastron_kernel:
    return fastron_kernel(int(kind), float(gamma))


def _require_cuda(*ts):
    for t in ts:
        if t is not None and not t.is_cuda:
            raise ValueError("device tensors required (no CPU fallback); use fastron_query for host buffers")


def _expect(t, dtype, name, dim=None):
    """dtype and inner contiguity (the C ABI takes a pointer plus a leading dimension)."""
    if t is None:
        return
    if t.dtype != dtype:
        raise ValueError(f"{name} must be {dtype}, got {t.dtype}")
    if dim is not None and t.dim() != dim:
        raise ValueError(f"{name} must have {dim} dimensions, got shape {tuple(t.shape)}")
    if t.dim() >= 1 and t.shape[-1] > 1 and t.stride(-1) != 1:
        raise ValueError(f"{name} must be contiguous in its last dimension (stride {t.stride()})")


def _expect_pos(t, name, n_cp=None):
    """Control points (M, n, 4) float32: float4 records, 16-byte aligned rows of a SoA."""
    _expect(t, _torch().float32, name, dim=3)
    if t.shape[2] != 4 or (t.shape[1] > 1 and t.stride(1) != 4) or t.stride(0) % 4 != 0:
        raise ValueError(f"{name} must be (M, n, 4) with float4 records (stride {t.stride()})")
    if t.numel() and t.data_ptr() % 16 != 0:
        raise ValueError(f"{name} must be 16-byte aligned")
    if n_cp is not None and t.shape[0] != n_cp:
        raise ValueError(f"{name} has {t.shape[0]} control points, expected {n_cp}")


def _torch():
    import torch
    return torch


def _workspace(nbytes: int, device, ts):
    return _new(max(int(nbytes), 256), _torch().uint8, device, ts)


def fastron_fk(robot, q, pos=None, stream=None):
    """q (n, >=D) float32 cuda -> pos (M, n, 4) float32 cuda (SoA float4, Eq. 1-2)."""
    torch = _torch()
    L = load_library()
    _require_cuda(q, pos)
    _expect(q, torch.float32, "q", dim=2)
    r = robot if isinstance(robot, fastron_robot) else make_robot_struct(robot)
    if q.shape[1] < r.dof:
        raise ValueError(f"q has {q.shape[1]} columns, the robot has {r.dof} joints")
    n = q.shape[0]
    ts = _tstream(stream)
    if pos is None:
        pos = _new((r.n_cp, n, 4), torch.float32, q.device, ts)
    _expect_pos(pos, "pos", r.n_cp)
    _check(L.fastron_fk(ctypes.byref(r), _ptr(q), n, q.stride(0), _ptr(pos), pos.stride(0) // 4, ts.cuda_stream))
    return pos


def fastron_score(qpos, spos, alpha, kind: int, gamma: float, score=None, label=None, want_score=True,
                  want_label=True, workspace=None, stream=None):
    """qpos (M, nq, 4), spos (M, ns, 4), alpha (ns,) -> (score float32 (nq,), label int8 (nq,))."""
    torch = _torch()
    L = load_library()
    _require_cuda(qpos, spos, alpha, score, label)
    _expect_pos(qpos, "qpos")
    M, nq = qpos.shape[0], qpos.shape[1]
    _expect_pos(spos, "spos", M)
    _expect(alpha, torch.float32, "alpha", dim=1)
    ns = spos.shape[1]
    ts = _tstream(stream)
    if want_score and score is None:
        score = _new(nq, torch.float32, qpos.device, ts)
    if want_label and label is None:
        label = _new(nq, torch.int8, qpos.device, ts)
    _expect(score, torch.float32, "score", dim=1)
    _expect(label, torch.int8, "label", dim=1)
    need = L.fastron_score_workspace_bytes(nq, ns, M)
    if workspace is None or workspace.numel() < need:
        workspace = _workspace(need, qpos.device, ts)
    lds = spos.stride(0) // 4 if ns > 0 else 0
    _check(L.fastron_score(_ptr(qpos), nq, qpos.stride(0) // 4, _ptr(spos) if ns else None,
                           _ptr(alpha) if ns else None, ns, lds, M, _kernel(kind, gamma), _ptr(score), _ptr(label),
                           _ptr(workspace), workspace.numel(), ts.cuda_stream))
    return score, label


class PackedModel:
    """A support set packed once per model update (fastron_model_pack)."""

    def __init__(self, buf, ns: int, n_cp: int, kind: int, gamma: float):
        self.buf, self.ns, self.n_cp, self.kind, self.gamma = buf, ns, n_cp, kind, gamma


def fastron_model_pack(spos, alpha, kind: int, gamma: float, stream=None) -> PackedModel:
    torch = _torch()
    L = load_library()
    _require_cuda(spos, alpha)
    _expect_pos(spos, "spos")
    _expect(alpha, torch.float32, "alpha", dim=1)
    M, ns = spos.shape[0], spos.shape[1]
    ts = _tstream(stream)
    buf = _workspace(L.fastron_model_bytes(ns, M), spos.device, ts)
    lds = spos.stride(0) // 4 if ns > 0 else 0
    _check(L.fastron_model_pack(_ptr(spos) if ns else None, _ptr(alpha) if ns else None, ns, lds, M,
                                _kernel(kind, gamma), _ptr(buf), buf.numel(), ts.cuda_stream))
    return PackedModel(buf, ns, M, kind, gamma)


def fastron_score_packed(qpos, model: PackedModel, score=None, label=None, want_score=True, want_label=True,
                         workspace=None, stream=None):
    torch = _torch()
    L = load_library()
    _require_cuda(qpos, score, label)
    _expect_pos(qpos, "qpos", model.n_cp)
    M, nq = qpos.shape[0], qpos.shape[1]
    ts = _tstream(stream)
    if want_score and score is None:
        score = _new(nq, torch.float32, qpos.device, ts)
    if want_label and label is None:
        label = _new(nq, torch.int8, qpos.device, ts)
    _expect(score, torch.float32, "score", dim=1)
    _expect(label, torch.int8, "label", dim=1)
    need = L.fastron_score_packed_workspace_bytes(nq, model.ns, M)
    if workspace is None or workspace.numel() < need:
        workspace = _workspace(need, qpos.device, ts)
    _check(L.fastron_score_packed(_ptr(qpos), nq, qpos.stride(0) // 4, _ptr(model.buf), model.ns, M,
                                  _kernel(model.kind, model.gamma), _ptr(score), _ptr(label), _ptr(workspace),
                                  workspace.numel(), ts.cuda_stream))
    return score, label


def fastron_score_packed_f64(qpos, model: PackedModel, out=None, workspace=None, stream=None):
    torch = _torch()
    L = load_library()
    _require_cuda(qpos, out)
    _expect_pos(qpos, "qpos", model.n_cp)
    M, nq = qpos.shape[0], qpos.shape[1]
    ts = _tstream(stream)
    if out is None:
        out = _new(nq, torch.float64, qpos.device, ts)
    _expect(out, torch.float64, "out", dim=1)
    need = L.fastron_score_packed_workspace_bytes(nq, model.ns, M)
    if workspace is None or workspace.numel() < need:
        workspace = _workspace(need, qpos.device, ts)
    _check(L.fastron_score_packed_f64(_ptr(qpos), nq, qpos.stride(0) // 4, _ptr(model.buf), model.ns, M,
                                      _kernel(model.kind, model.gamma), _ptr(out), _ptr(workspace), workspace.numel(),
                                      ts.cuda_stream))
    return out


def fastron_gram(pos, kind: int, gamma: float, K=None, workspace=None, stream=None):
    """pos (M, n, 4) -> K (n, n) float32."""
    torch = _torch()
    L = load_library()
    _require_cuda(pos, K)
    _expect_pos(pos, "pos")
    M, n = pos.shape[0], pos.shape[1]
    ts = _tstream(stream)
    if K is None:
        # rows padded to a multiple of 8 floats: 32-byte aligned rows select the library's
        # column-slot Gram kernel with whole-sector mirror stores (ldk % 8 == 0); the result
        # is the (n, n) view (N = 8,446: 0.54 -> 0.13 ms against an unpadded matrix)
        K = _new((n, (n + 7) // 8 * 8), torch.float32, pos.device, ts)[:, :n]
    _expect(K, torch.float32, "K", dim=2)
    need = L.fastron_gram_workspace_bytes(n, M)
    if workspace is None or workspace.numel() < need:
        workspace = _workspace(need, pos.device, ts)
    _check(L.fastron_gram(_ptr(pos), n, pos.stride(0) // 4, M, _kernel(kind, gamma), _ptr(K), K.stride(0),
                          _ptr(workspace), workspace.numel(), ts.cuda_stream))
    return K


def fastron_score_joint(q, s, alpha, kind: int, gamma: float, score=None, label=None, workspace=None, stream=None):
    """Joint-space RBF ("Fastron RBF" baseline): q (nq, >=D), s (ns, >=D) configurations."""
    torch = _torch()
    L = load_library()
    _require_cuda(q, s, alpha, score, label)
    _expect(q, torch.float32, "q", dim=2)
    _expect(s, torch.float32, "s", dim=2)
    _expect(alpha, torch.float32, "alpha", dim=1)
    nq, ns = q.shape[0], s.shape[0]
    dof = q.shape[1]
    ts = _tstream(stream)
    if score is None:
        score = _new(nq, torch.float32, q.device, ts)
    if label is None:
        label = _new(nq, torch.int8, q.device, ts)
    _expect(score, torch.float32, "score", dim=1)
    _expect(label, torch.int8, "label", dim=1)
    need = L.fastron_score_joint_workspace_bytes(nq, ns, dof)
    if workspace is None or workspace.numel() < need:
        workspace = _workspace(need, q.device, ts)
    _check(L.fastron_score_joint(_ptr(q), nq, q.stride(0), _ptr(s) if ns else None, _ptr(alpha) if ns else None, ns,
                                 s.stride(0) if ns else dof, dof, _kernel(kind, gamma), _ptr(score), _ptr(label),
                                 _ptr(workspace), workspace.numel(), ts.cuda_stream))
    return score, label


def fastron_gram_joint(x, kind: int, gamma: float, K=None, workspace=None, stream=None):
    """Joint-space RBF Gram of configurations x (n, D)."""
    torch = _torch()
    L = load_library()
    _require_cuda(x, K)
    _expect(x, torch.float32, "x", dim=2)
    n, dof = x.shape[0], x.shape[1]
    ts = _tstream(stream)
    if K is None:
        K = _new((n, n), torch.float32, x.device, ts)
    _expect(K, torch.float32, "K", dim=2)
    need = L.fastron_gram_joint_workspace_bytes(n, dof)
    if workspace is None or workspace.numel() < need:
        workspace = _workspace(need, x.device, ts)
    _check(L.fastron_gram_joint(_ptr(x), n, x.stride(0), dof, _kernel(kind, gamma), _ptr(K), K.stride(0),
                                _ptr(workspace), workspace.numel(), ts.cuda_stream))
    return K


def _train_outputs(n, iter_max, dev, ts, alpha, F, support_idx, trace, result):
    torch = _torch()
    if alpha is None:
        alpha = _zeros(n, torch.float64, dev, ts)
    if F is None:
        F = _zeros(n, torch.float64, dev, ts)
    _expect(alpha, torch.float64, "alpha", dim=1)
    _expect(F, torch.float64, "F", dim=1)
    sup = _new(max(n, 1), torch.int32, dev, ts) if support_idx is True else support_idx
    tr = _new(max(iter_max, 1), torch.int32, dev, ts) if trace is True else trace
    for t, nm in ((sup, "support_idx"), (tr, "trace")):
        if t is not None and t is not False:
            _expect(t, torch.int32, nm, dim=1)
    res = _zeros(ctypes.sizeof(fastron_train_result), torch.uint8, dev, ts) if result is None else result
    return alpha, F, sup, tr, res


def fastron_train(K, y, beta: float = 1.0, iter_max: int = 20000, s_max: Optional[int] = None, alpha=None, F=None,
                  support_idx=True, trace=True, result=None, stream=None):
    """Algorithm 1 on device. Returns dict of device tensors (alpha, F, support_idx, trace)
    and the result struct as a uint8 device tensor (decode with train_result())."""
    torch = _torch()
    L = load_library()
    _require_cuda(K, y, alpha, F)
    _expect(K, torch.float32, "K", dim=2)
    _expect(y, torch.int8, "y", dim=1)
    n = K.shape[0]
    ts = _tstream(stream)
    s_max = n if s_max is None else int(s_max)
    alpha, F, sup, tr, res = _train_outputs(n, iter_max, K.device, ts, alpha, F, support_idx, trace, result)
    _check(L.fastron_train(_ptr(K), n, K.stride(0) if n else 1, _ptr(y), float(beta), int(iter_max), s_max,
                           _ptr(alpha), _ptr(F), _ptr(sup) if sup is not None and sup is not False else None,
                           _ptr(tr) if tr is not None and tr is not False else None, _ptr(res), ts.cuda_stream))
    return dict(alpha=alpha, F=F, support_idx=sup, trace=tr, result=res)


def fastron_train_lazy(pos, y, kind: int, gamma: float, beta: float = 1.0, iter_max: int = 20000,
                       s_max: Optional[int] = None, alpha=None, F=None, cache_cols: Optional[int] = None,
                       support_idx=True, trace=True, result=None, workspace=None, stream=None):
    """Algorithm 1 with lazily computed, cached K columns (no Gram). pos: (M, n, 4) control points."""
    torch = _torch()
    L = load_library()
    _require_cuda(pos, y, alpha, F)
    _expect_pos(pos, "pos")
    _expect(y, torch.int8, "y", dim=1)
    M, n = pos.shape[0], pos.shape[1]
    ts = _tstream(stream)
    s_max = n if s_max is None else int(s_max)
    cache_cols = min(n, 4096) if cache_cols is None else int(cache_cols)
    alpha, F, sup, tr, res = _train_outputs(n, iter_max, pos.device, ts, alpha, F, support_idx, trace, result)
    need = L.fastron_train_lazy_workspace_bytes(n, M, cache_cols)
    if workspace is None or workspace.numel() < need:
        workspace = _workspace(need, pos.device, ts)
    _check(L.fastron_train_lazy(_ptr(pos), n, pos.stride(0) // 4, M, _kernel(kind, gamma), _ptr(y), float(beta),
                                int(iter_max), s_max, _ptr(alpha), _ptr(F),
                                _ptr(sup) if sup is not None and sup is not False else None,
                                _ptr(tr) if tr is not None and tr is not False else None, _ptr(res), cache_cols,
                                _ptr(workspace), workspace.numel(), ts.cuda_stream))
    return dict(alpha=alpha, F=F, support_idx=sup, trace=tr, result=res)


def fastron_active_samples(S, n_near: int, z, sigma, u, lo, hi, out=None, stream=None):
    """Two-stage active-learning draws; random numbers z ~ N(0,1), u ~ U[0,1) are inputs."""
    torch = _torch()
    L = load_library()
    _require_cuda(S, z, sigma, u, lo, hi, out)
    for t, nm in ((S, "S"), (z, "z"), (u, "u"), (out, "out")):
        _expect(t, torch.float32, nm, dim=2)
    for t, nm in ((sigma, "sigma"), (lo, "lo"), (hi, "hi")):
        _expect(t, torch.float32, nm, dim=1)
    ns, dof = S.shape[0], S.shape[1]
    if z is not None and z.shape[1] != dof or u is not None and u.shape[1] != dof:
        raise ValueError("z and u must have D columns (row stride D)")
    if z is not None and z.stride(0) != dof or u is not None and u.stride(0) != dof:
        raise ValueError("z and u must be contiguous (row stride D)")
    n_uniform = u.shape[0] if u is not None else 0
    total = ns * n_near + n_uniform
    ts = _tstream(stream)
    if out is None:
        out = _new((total, dof), torch.float32, S.device, ts)
    _check(L.fastron_active_samples(_ptr(S), ns, S.stride(0), dof, int(n_near), _ptr(z), _ptr(sigma), _ptr(u),
                                    n_uniform, _ptr(lo), _ptr(hi), _ptr(out), out.stride(0), ts.cuda_stream))
    return out


def fastron_label_capsules(pos, chain, boxes, radius: float, label=None, stream=None):
    """Capsule-vs-box labels (+1 = C_obs) of control-point positions pos (M, n, 4)."""
    torch = _torch()
    L = load_library()
    _require_cuda(pos, label)
    _expect_pos(pos, "pos")
    n = pos.shape[1]
    ts = _tstream(stream)
    if label is None:
        label = _new(n, torch.int8, pos.device, ts)
    _expect(label, torch.int8, "label", dim=1)
    ch = np.ascontiguousarray(np.asarray(chain, dtype=np.int32))
    bx = np.ascontiguousarray(np.asarray(boxes, dtype=np.float64).reshape(-1, 6))
    _check(L.fastron_label_capsules(_ptr(pos), pos.stride(0) // 4, n, ch.ctypes.data if len(ch) else None, len(ch),
                                    bx.ctypes.data if len(bx) else None, len(bx), float(radius), _ptr(label),
                                    ts.cuda_stream))
    return label


def fastron_kernel_matvec(K, alpha, F=None, stream=None):
    torch = _torch()
    L = load_library()
    _require_cuda(K, alpha, F)
    _expect(K, torch.float32, "K", dim=2)
    _expect(alpha, torch.float64, "alpha", dim=1)
    n = K.shape[0]
    ts = _tstream(stream)
    if F is None:
        F = _new(n, torch.float64, K.device, ts)
    _expect(F, torch.float64, "F", dim=1)
    _check(L.fastron_kernel_matvec(_ptr(K), n, K.stride(0), _ptr(alpha), _ptr(F), ts.cuda_stream))
    return F


def fastron_kernel_matvec_lazy(pos, alpha, kind: int, gamma: float, F=None, workspace=None, stream=None):
    """F = K alpha with the entries of K computed on the fly from control points pos
    (M, n, 4): the values and the order of fastron_kernel_matvec(fastron_gram(pos), alpha),
    without the Gram (the margins of a warm-started lazy Algorithm 1)."""
    torch = _torch()
    L = load_library()
    _require_cuda(pos, alpha, F)
    _expect_pos(pos, "pos")
    _expect(alpha, torch.float64, "alpha", dim=1)
    M, n = pos.shape[0], pos.shape[1]
    ts = _tstream(stream)
    if F is None:
        F = _new(n, torch.float64, pos.device, ts)
    _expect(F, torch.float64, "F", dim=1)
    need = L.fastron_kernel_matvec_lazy_workspace_bytes(n, M)
    if workspace is None or workspace.numel() < need:
        workspace = _workspace(need, pos.device, ts)
    _check(L.fastron_kernel_matvec_lazy(_ptr(pos), n, pos.stride(0) // 4, M, _kernel(kind, gamma), _ptr(alpha),
                                        _ptr(F), _ptr(workspace), workspace.numel(), ts.cuda_stream))
    return F


def train_result(res_tensor) -> dict:
    raw = bytes(res_tensor.cpu().numpy().tobytes())
    r = fastron_train_result.from_buffer_copy(raw)
    return dict(iterations=r.iterations, n_add=r.n_add, n_remove=r.n_remove, converged=bool(r.converged),
                n_support=r.n_support)


def fastron_edge_check(robot, qa, qb, n_interp: int, spos, alpha, kind: int, gamma: float, in_collision=None,
                       hit_index=None, want_hit_index=True, workspace=None, stream=None):
    torch = _torch()
    L = load_library()
    _require_cuda(qa, qb, spos, alpha, in_collision, hit_index)
    _expect(qa, torch.float32, "qa", dim=2)
    _expect(qb, torch.float32, "qb", dim=2)
    _expect_pos(spos, "spos")
    _expect(alpha, torch.float32, "alpha", dim=1)
    r = robot if isinstance(robot, fastron_robot) else make_robot_struct(robot)
    E = qa.shape[0]
    ns = spos.shape[1]
    if qa.shape != qb.shape or qa.stride(0) != qb.stride(0):
        raise ValueError("qa and qb must have the same shape and leading dimension")
    ts = _tstream(stream)
    if in_collision is None:
        in_collision = _new(E, torch.uint8, qa.device, ts)
    if want_hit_index and hit_index is None:
        hit_index = _new(E, torch.int32, qa.device, ts)
    _expect(in_collision, torch.uint8, "in_collision", dim=1)
    _expect(hit_index, torch.int32, "hit_index", dim=1)
    need = L.fastron_edge_workspace_bytes(E, ns, r.n_cp)
    if workspace is None or workspace.numel() < need:
        workspace = _workspace(need, qa.device, ts)
    lds = spos.stride(0) // 4 if ns > 0 else 0
    _check(L.fastron_edge_check(ctypes.byref(r), _ptr(qa), _ptr(qb), E, qa.stride(0), int(n_interp),
                                _ptr(spos) if ns else None, _ptr(alpha) if ns else None, ns, lds, _kernel(kind, gamma),
                                _ptr(in_collision), _ptr(hit_index), _ptr(workspace), workspace.numel(),
                                ts.cuda_stream))
    return in_collision, hit_index


def fastron_edge_check_packed(robot, qa, qb, n_interp: int, model: PackedModel, in_collision=None, hit_index=None,
                              want_hit_index=True, workspace=None, stream=None):
    """fastron_edge_check against a packed (e.g. broadcast) model."""
    torch = _torch()
    L = load_library()
    _require_cuda(qa, qb, in_collision, hit_index)
    _expect(qa, torch.float32, "qa", dim=2)
    _expect(qb, torch.float32, "qb", dim=2)
    r = robot if isinstance(robot, fastron_robot) else make_robot_struct(robot)
    if r.n_cp != model.n_cp:
        raise ValueError("robot and model control-point counts differ")
    E = qa.shape[0]
    if qa.shape != qb.shape or qa.stride(0) != qb.stride(0):
        raise ValueError("qa and qb must have the same shape and leading dimension")
    ts = _tstream(stream)
    if in_collision is None:
        in_collision = _new(E, torch.uint8, qa.device, ts)
    if want_hit_index and hit_index is None:
        hit_index = _new(E, torch.int32, qa.device, ts)
    _expect(in_collision, torch.uint8, "in_collision", dim=1)
    _expect(hit_index, torch.int32, "hit_index", dim=1)
    need = L.fastron_edge_packed_workspace_bytes(E, model.ns, r.n_cp)
    if workspace is None or workspace.numel() < need:
        workspace = _workspace(need, qa.device, ts)
    _check(L.fastron_edge_check_packed(ctypes.byref(r), _ptr(qa), _ptr(qb), E, qa.stride(0), int(n_interp),
                                       _ptr(model.buf), model.ns, r.n_cp, _kernel(model.kind, model.gamma),
                                       _ptr(in_collision), _ptr(hit_index), _ptr(workspace), workspace.numel(),
                                       ts.cuda_stream))
    return in_collision, hit_index


def fastron_query(robot, q, spos, alpha, kind: int, gamma: float, score=None, label=None, workspace=None,
                  stream=None):
    """FK + score; q / score / label may be host (CPU, ideally pinned) or device tensors."""
    torch = _torch()
    L = load_library()
    _require_cuda(spos, alpha)
    _expect(q, torch.float32, "q", dim=2)
    _expect_pos(spos, "spos")
    _expect(alpha, torch.float32, "alpha", dim=1)
    _expect(score, torch.float32, "score", dim=1)
    _expect(label, torch.int8, "label", dim=1)
    r = robot if isinstance(robot, fastron_robot) else make_robot_struct(robot)
    nq = q.shape[0]
    ns = spos.shape[1]
    ts = _tstream(stream)
    need = L.fastron_query_workspace_bytes(nq, ns, r.n_cp, r.dof)
    if workspace is None or workspace.numel() < need:
        workspace = _workspace(need, spos.device, ts)
    lds = spos.stride(0) // 4 if ns > 0 else 0
    _check(L.fastron_query(ctypes.byref(r), _ptr(q), nq, q.stride(0), _ptr(spos) if ns else None,
                           _ptr(alpha) if ns else None, ns, lds, _kernel(kind, gamma), _ptr(score), _ptr(label),
                           _ptr(workspace), workspace.numel(), ts.cuda_stream))
    return score, label


def fastron_query_packed(robot, q, model: PackedModel, score=None, label=None, want_score=True, want_label=True,
                         workspace=None, stream=None):
    """Configurations q (nq, >=D) float32 cuda against a packed model -> (score, label):
    one launch for small and mid-size batches (D-H chain fused into the scoring kernel)."""
    torch = _torch()
    L = load_library()
    _require_cuda(q, score, label)
    _expect(q, torch.float32, "q", dim=2)
    r = robot if isinstance(robot, fastron_robot) else make_robot_struct(robot)
    if r.n_cp != model.n_cp:
        raise ValueError("robot and model control-point counts differ")
    if q.shape[1] < r.dof:
        raise ValueError(f"q has {q.shape[1]} columns, the robot has {r.dof} joints")
    nq = q.shape[0]
    ts = _tstream(stream)
    if want_score and score is None:
        score = _new(nq, torch.float32, q.device, ts)
    if want_label and label is None:
        label = _new(nq, torch.int8, q.device, ts)
    _expect(score, torch.float32, "score", dim=1)
    _expect(label, torch.int8, "label", dim=1)
    need = L.fastron_query_packed_workspace_bytes(nq, model.ns, r.n_cp, r.dof)
    if workspace is None or workspace.numel() < need:
        workspace = _workspace(need, q.device, ts)
    _check(L.fastron_query_packed(ctypes.byref(r), _ptr(q), nq, q.stride(0), _ptr(model.buf), model.ns, r.n_cp,
                                  _kernel(model.kind, model.gamma), _ptr(score), _ptr(label), _ptr(workspace),
                                  workspace.numel(), ts.cuda_stream))
    return score, label


def fastron_fk64(robot, q, pos=None, stream=None):
    """q (n, >=D) float32 cuda -> pos (M, n, 4) float64 cuda: unrounded fp64 positions."""
    torch = _torch()
    L = load_library()
    _require_cuda(q, pos)
    _expect(q, torch.float32, "q", dim=2)
    r = robot if isinstance(robot, fastron_robot) else make_robot_struct(robot)
    n = q.shape[0]
    ts = _tstream(stream)
    if pos is None:
        pos = _new((r.n_cp, n, 4), torch.float64, q.device, ts)
    _expect(pos, torch.float64, "pos", dim=3)
    if pos.shape[0] != r.n_cp or pos.shape[2] != 4 or (n > 1 and pos.stride(1) != 4) or pos.data_ptr() % 32:
        raise ValueError("pos must be (M, n, 4) float64 with 32-byte aligned double4 records")
    _check(L.fastron_fk64(ctypes.byref(r), _ptr(q), n, q.stride(0), _ptr(pos), pos.stride(0) // 4, ts.cuda_stream))
    return pos


def fastron_score_precise(qpos64, spos64, alpha64, kind: int, gamma: float, score=None, label=None, stream=None):
    """fp64 scores (nq,) float64 and labels of fp64 positions against fp64 supports/weights."""
    torch = _torch()
    L = load_library()
    _require_cuda(qpos64, spos64, alpha64, score, label)
    for t, nm in ((qpos64, "qpos64"), (spos64, "spos64")):
        _expect(t, torch.float64, nm, dim=3)
        if t.shape[2] != 4 or (t.shape[1] > 1 and t.stride(1) != 4) or (t.numel() and t.data_ptr() % 32):
            raise ValueError(f"{nm} must be (M, n, 4) float64 with 32-byte aligned double4 records")
    _expect(alpha64, torch.float64, "alpha64", dim=1)
    M, nq = qpos64.shape[0], qpos64.shape[1]
    ns = spos64.shape[1]
    ts = _tstream(stream)
    if score is None:
        score = _new(nq, torch.float64, qpos64.device, ts)
    if label is None:
        label = _new(nq, torch.int8, qpos64.device, ts)
    _expect(score, torch.float64, "score", dim=1)
    _expect(label, torch.int8, "label", dim=1)
    _check(L.fastron_score_precise(_ptr(qpos64), nq, qpos64.stride(0) // 4, _ptr(spos64) if ns else None,
                                   _ptr(alpha64) if ns else None, ns, spos64.stride(0) // 4 if ns else 0, M,
                                   _kernel(kind, gamma), _ptr(score), _ptr(label), ts.cuda_stream))
    return score, label


def launch_count() -> int:
    return int(load_library().fastron_launch_count())


def set_validation(on: bool) -> None:
    """Content validation of every entry point's inputs (include/fastron.h conventions)."""
    load_library().fastron_set_validation(1 if on else 0)


def validation() -> bool:
    return bool(load_library().fastron_validation())


def version() -> str:
    return load_library().fastron_version().decode()
