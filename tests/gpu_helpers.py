"""Shared helpers of the -m gpu parity tests (GPU path through the C ABI vs the oracle)."""
import numpy as np
import pytest

try:
    import torch
except Exception:  # pragma: no cover
    torch = None


def require_gpu():
    if torch is None or not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")


def dev(a, dtype=None):
    t = torch.as_tensor(np.ascontiguousarray(a))
    if dtype is not None:
        t = t.to(dtype)
    return t.cuda()


def soa_from_oracle(pos64):
    """oracle (N, M, 3) float64 -> (M, N, 4) float32 device tensor (rounded once)."""
    n, M, _ = pos64.shape
    out = np.zeros((M, n, 4), dtype=np.float32)
    out[:, :, :3] = np.transpose(pos64, (1, 0, 2)).astype(np.float32)
    return dev(out)


def positions_np(pos_dev):
    """(M, N, 4) device -> (N, M, 3) float64 numpy."""
    p = pos_dev.cpu().numpy()
    return np.transpose(p[:, :, :3], (1, 0, 2)).astype(np.float64)


def assert_score_parity(f_gpu, f_ref, label_gpu=None, rel=1e-4, floor=1e-5, what=""):
    """BASELINE.json north_star tolerance (R16): |f_gpu - f_ref| <= max(rel |f_ref|, floor)
    for every checked query; labels equal wherever |f_ref| > 1e-4."""
    f_gpu = np.asarray(f_gpu, dtype=np.float64)
    err = np.abs(f_gpu - f_ref)
    tol = np.maximum(rel * np.abs(f_ref), floor)
    bad = np.flatnonzero(err > tol)
    assert bad.size == 0, (f"{what}: {bad.size} of {f_ref.size} outside tolerance; worst idx {bad[:5]} "
                           f"gpu {f_gpu[bad[:5]]} ref {f_ref[bad[:5]]} max err {err.max():.3g}")
    if label_gpu is not None:
        lab = np.asarray(label_gpu)
        sure = np.abs(f_ref) > 1e-4
        ref_lab = np.where(f_ref > 0, 1, -1)
        mism = np.flatnonzero(sure & (lab != ref_lab))
        assert mism.size == 0, f"{what}: {mism.size} label mismatches at {mism[:5]}"
        # the label is the sign of the GPU's own score (R8), everywhere
        assert np.array_equal(lab, np.where(f_gpu > 0, 1, -1)) or np.all(
            (lab == np.where(f_gpu > 0, 1, -1)) | (np.abs(f_gpu) < 1e-30))
    return float(err.max()) if err.size else 0.0
