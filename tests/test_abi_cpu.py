"""CPU-only checks of the C-ABI boundary: the library loads, exports every symbol
include/fastron.h declares, and rejects bad arguments before any CUDA work."""
import ctypes
import os
import re

import numpy as np
import pytest

import paper_1910_06451_b200 as fb
import workloads as W

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_functions():
    src = open(os.path.join(ROOT, "include", "fastron.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(fastron_\w+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    L = fb.load_library()
    declared = _declared_functions()
    assert len(declared) >= 14
    for name in declared:
        assert hasattr(L, name), name
    assert sorted(declared) == sorted(fb.EXPORTED)


def test_version_and_counter():
    assert "sm_100a" in fb.version()
    assert fb.launch_count() >= 0


def test_workspace_sizes_are_host_only():
    L = fb.load_library()
    # headline: 20k supports, M=8 -> 313 tiles of 64 x (4 pairs x 32 B + 4 B)
    ws = L.fastron_score_workspace_bytes(1_000_000, 20_000, 8)
    assert ws >= 313 * (64 * 4 * 32 + 64 * 4)
    assert L.fastron_score_workspace_bytes(-1, 10, 8) == 0
    assert L.fastron_gram_workspace_bytes(5000, 8) > 0
    assert L.fastron_edge_workspace_bytes(10_000, 3000, 8) > 0
    assert L.fastron_query_workspace_bytes(1 << 20, 20_000, 8, 7) > 0
    assert L.fastron_train_max_n() >= 20_000


def _robot():
    return fb.make_robot_struct(W.arm7(8))


def _err(status):
    return status, fb.load_library().fastron_last_error().decode()


def test_fk_argument_errors():
    L = fb.load_library()
    r = _robot()
    st, msg = _err(L.fastron_fk(None, 1, 10, 7, 16, 10, None))
    assert st == fb.FASTRON_ERR_INVALID_ARG and "robot" in msg
    bad = _robot()
    bad.dof = 0
    assert L.fastron_fk(ctypes.byref(bad), 16, 10, 7, 16, 10, None) == fb.FASTRON_ERR_INVALID_ARG
    bad = _robot()
    bad.cp_frame[3] = 9
    st, msg = _err(L.fastron_fk(ctypes.byref(bad), 16, 10, 7, 16, 10, None))
    assert st == fb.FASTRON_ERR_INVALID_ARG and "cp_frame" in msg
    bad = _robot()
    bad.dh[2][1] = float("nan")
    assert L.fastron_fk(ctypes.byref(bad), 16, 10, 7, 16, 10, None) == fb.FASTRON_ERR_INVALID_ARG
    assert L.fastron_fk(ctypes.byref(r), 16, 10, 6, 16, 10, None) == fb.FASTRON_ERR_INVALID_ARG  # ldq < dof
    assert L.fastron_fk(ctypes.byref(r), 16, 10, 7, 16, 9, None) == fb.FASTRON_ERR_INVALID_ARG  # ldpos < n
    assert L.fastron_fk(ctypes.byref(r), 16, 10, 7, 8, 10, None) == fb.FASTRON_ERR_INVALID_ARG  # misaligned pos
    assert L.fastron_fk(ctypes.byref(r), 16, -1, 7, 16, 10, None) == fb.FASTRON_ERR_INVALID_ARG
    assert L.fastron_fk(ctypes.byref(r), None, 0, 7, None, 0, None) == fb.FASTRON_OK  # empty is a no-op


def test_score_argument_errors():
    L = fb.load_library()
    k = fb.fastron_kernel(0, 5.0)
    assert L.fastron_score(16, 10, 10, 16, 16, 5, 5, 8, fb.fastron_kernel(0, 0.0), 16, None, 256, 1 << 20,
                           None) == fb.FASTRON_ERR_INVALID_ARG
    assert L.fastron_score(16, 10, 10, 16, 16, 5, 5, 8, fb.fastron_kernel(0, float("inf")), 16, None, 256, 1 << 20,
                           None) == fb.FASTRON_ERR_INVALID_ARG
    assert L.fastron_score(16, 10, 10, 16, 16, 5, 5, 8, fb.fastron_kernel(7, 1.0), 16, None, 256, 1 << 20,
                           None) == fb.FASTRON_ERR_INVALID_ARG
    assert L.fastron_score(16, 10, 10, 16, 16, 5, 5, 0, k, 16, None, 256, 1 << 20, None) == fb.FASTRON_ERR_INVALID_ARG
    assert L.fastron_score(16, 10, 10, 16, 16, 5, 5, 33, k, 16, None, 256, 1 << 20, None) == fb.FASTRON_ERR_INVALID_ARG
    assert L.fastron_score(16, 10, 9, 16, 16, 5, 5, 8, k, 16, None, 256, 1 << 20, None) == fb.FASTRON_ERR_INVALID_ARG
    assert L.fastron_score(16, 10, 10, 16, 16, 5, 4, 8, k, 16, None, 256, 1 << 20, None) == fb.FASTRON_ERR_INVALID_ARG
    assert L.fastron_score(16, 10, 10, None, 16, 5, 5, 8, k, 16, None, 256, 1 << 20, None) == fb.FASTRON_ERR_INVALID_ARG
    assert L.fastron_score(16, 10, 10, 16, 16, 5, 5, 8, k, None, None, 256, 1 << 20, None) == fb.FASTRON_ERR_INVALID_ARG
    st, msg = _err(L.fastron_score(16, 10, 10, 16, 16, 5, 5, 8, k, 16, None, 256, 8, None))
    assert st == fb.FASTRON_ERR_WORKSPACE and "workspace" in msg
    assert L.fastron_score(16, 0, 0, None, None, 0, 0, 8, k, None, None, None, 0, None) == fb.FASTRON_OK


def test_gram_train_edge_query_argument_errors():
    L = fb.load_library()
    k = fb.fastron_kernel(1, 2.0)
    assert L.fastron_gram(16, 10, 9, 8, k, 16, 10, 256, 1 << 20, None) == fb.FASTRON_ERR_INVALID_ARG
    assert L.fastron_gram(16, 10, 10, 8, k, 16, 10, 256, 4, None) == fb.FASTRON_ERR_WORKSPACE
    assert L.fastron_gram(None, 0, 0, 8, k, None, 0, None, 0, None) == fb.FASTRON_OK
    # train: beta < 1, too large n, NULL result
    assert L.fastron_train(16, 10, 10, 16, 0.5, 10, 10, 16, 16, None, None, 16, None) == fb.FASTRON_ERR_INVALID_ARG
    assert L.fastron_train(16, 10, 10, 16, float("nan"), 10, 10, 16, 16, None, None, 16, None) == fb.FASTRON_ERR_INVALID_ARG
    assert L.fastron_train(16, 10, 10, 16, 1.0, 10, 10, 16, 16, None, None, None, None) == fb.FASTRON_ERR_INVALID_ARG
    big = L.fastron_train_max_n() + 1
    assert L.fastron_train(16, big, big, 16, 1.0, 10, 10, 16, 16, None, None, 16, None) == fb.FASTRON_ERR_UNSUPPORTED
    assert L.fastron_train(16, 10, 9, 16, 1.0, 10, 10, 16, 16, None, None, 16, None) == fb.FASTRON_ERR_INVALID_ARG
    r = _robot()
    assert L.fastron_edge_check(ctypes.byref(r), 16, 16, 10, 7, 0, 16, 16, 5, 5, k, 16, None, 256, 1 << 24,
                                None) == fb.FASTRON_ERR_INVALID_ARG  # n_interp < 1
    assert L.fastron_edge_check(ctypes.byref(r), 16, 16, 10, 7, 64, 16, 16, 5, 5, k, 16, None, 256, 16,
                                None) == fb.FASTRON_ERR_WORKSPACE
    assert L.fastron_edge_check(ctypes.byref(r), None, None, 0, 7, 64, None, None, 0, 0, k, None, None, None, 0,
                                None) == fb.FASTRON_OK
    assert L.fastron_query(ctypes.byref(r), 16, 10, 6, 16, 16, 5, 5, k, 16, None, 256, 1 << 24,
                           None) == fb.FASTRON_ERR_INVALID_ARG


def test_robot_marshalling_roundtrip():
    robot = W.arm7(16)
    r = fb.make_robot_struct(robot)
    assert r.dof == 7 and r.n_cp == 16
    assert np.allclose(np.array([[r.dh[i][c] for c in range(4)] for i in range(7)]), robot.dh)
    assert [r.cp_frame[m] for m in range(16)] == robot.cp_frame.tolist()
    with pytest.raises(ValueError):
        fb.make_robot_struct(W.make_robot("x", np.zeros((17, 4)), [1], [[0, 0, 0]]))


def test_product_package_never_imports_the_oracle():
    """The product path must not route through the oracle (no CPU fallback)."""
    pkg = os.path.join(ROOT, "paper_1910_06451_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                src = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in src and "from oracle" not in src and "liboracle" not in src, f


def test_validation_switch():
    """fastron_set_validation / fastron_validation (include/fastron.h conventions)."""
    before = fb.validation()
    fb.set_validation(True)
    assert fb.validation()
    fb.set_validation(False)
    assert not fb.validation()
    fb.set_validation(before)


def test_round2_entry_points_argument_errors():
    """The round-2 calls reject bad arguments before any CUDA work: n_cp mismatches,
    misaligned float4/double4/packed pointers, short workspaces, unsupported n_cp."""
    L = fb.load_library()
    r = _robot()
    k = fb.fastron_kernel(0, 5.0)
    A = 1 << 20  # an aligned, never dereferenced address
    # fastron_query_packed: n_cp must match the robot; packed 256-byte aligned
    st, msg = _err(L.fastron_query_packed(ctypes.byref(r), A, 10, 7, A, 100, 16, k, A, None, A, 1 << 20, None))
    assert st == fb.FASTRON_ERR_INVALID_ARG and "n_cp" in msg
    assert L.fastron_query_packed(ctypes.byref(r), None, 0, 7, None, 0, 8, k, None, None, None, 0, None) == fb.FASTRON_OK
    # fastron_edge_check_packed
    st, msg = _err(L.fastron_edge_check_packed(ctypes.byref(r), A, A, 10, 7, 64, A, 100, 4, k, A, None, A, 1 << 20, None))
    assert st == fb.FASTRON_ERR_INVALID_ARG and "n_cp" in msg
    st, msg = _err(L.fastron_edge_check_packed(ctypes.byref(r), A, A, 10, 7, 64, A + 16, 100, 8, k, A, None, A,
                                               1 << 24, None))
    assert st == fb.FASTRON_ERR_INVALID_ARG and "aligned" in msg
    assert L.fastron_edge_check_packed(ctypes.byref(r), A, A, 10, 7, 0, A, 100, 8, k, A, None, A, 1 << 24,
                                       None) == fb.FASTRON_ERR_INVALID_ARG  # n_interp < 1
    # fastron_score_packed: packed and qpos alignment
    st, msg = _err(L.fastron_score_packed(A, 10, 10, A + 16, 100, 8, k, A, None, A, 1 << 24, None))
    assert st == fb.FASTRON_ERR_INVALID_ARG and "packed" in msg
    st, msg = _err(L.fastron_score_packed(A + 8, 10, 10, A, 100, 8, k, A, None, A, 1 << 24, None))
    assert st == fb.FASTRON_ERR_INVALID_ARG and "qpos" in msg
    # fastron_kernel_matvec_lazy: n_cp range, workspace size and alignment
    assert L.fastron_kernel_matvec_lazy(A, 10, 10, 0, k, A, A, A, 1 << 20, None) == fb.FASTRON_ERR_INVALID_ARG
    st, msg = _err(L.fastron_kernel_matvec_lazy(A, 1000, 1000, 8, k, A, A, A, 16, None))
    assert st == fb.FASTRON_ERR_WORKSPACE
    assert L.fastron_kernel_matvec_lazy(A + 8, 10, 10, 8, k, A, A, A, 1 << 20, None) == fb.FASTRON_ERR_INVALID_ARG
    # fastron_fk64 / fastron_score_precise: double4 alignment, n_cp <= 16
    assert L.fastron_fk64(ctypes.byref(r), A, 10, 7, A + 16, 10, None) == fb.FASTRON_ERR_INVALID_ARG
    st, msg = _err(L.fastron_score_precise(A, 10, 10, A, A, 5, 5, 17, k, A, None, None))
    assert st == fb.FASTRON_ERR_UNSUPPORTED and "n_cp" in msg
    assert L.fastron_score_precise(A + 16, 10, 10, A, A, 5, 5, 8, k, A, None, None) == fb.FASTRON_ERR_INVALID_ARG
    assert L.fastron_score_precise(A, 10, 10, A, A, 5, 4, 8, k, A, None, None) == fb.FASTRON_ERR_INVALID_ARG
    assert L.fastron_score_precise(None, 0, 0, None, None, 0, 0, 8, k, None, None, None) == fb.FASTRON_OK
    # workspace sizes: host-only queries
    assert L.fastron_query_packed_workspace_bytes(1 << 20, 20_000, 8, 7) > 0
    assert L.fastron_edge_packed_workspace_bytes(10_000, 3000, 8) > 0
    assert L.fastron_kernel_matvec_lazy_workspace_bytes(20_000, 16) > 0
    assert L.fastron_train_lazy_max_n(16) == 32_768
