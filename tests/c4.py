"""The GPU-vs-oracle parity protocol of SURVEY.md §8(c) C4, shared by the -m gpu tests and
tests/tools/parity_report.py (test infrastructure; expected values come only from oracle/).

Tolerance (BASELINE.json north_star, R16): a score passes iff
    |f_gpu - f_ref| <= max(1e-4 |f_ref|, 1e-5),
and labels must agree wherever |f_ref| > 1e-4. Sampling at full sizes: a seeded uniform
subsample plus every query whose GPU score lies within 1e-2 of zero (the label boundary,
where the 1e-5 floor binds), up to 10,000 of them.
"""
import numpy as np

REL, FLOOR, LABEL_SURE = 1e-4, 1e-5, 1e-4


def c4_sample(s_gpu, n_uniform, seed, band=1e-2, band_max=10_000):
    """Indices: n_uniform seeded uniform queries plus every |s_gpu| <= band (at most band_max,
    a seeded subset if there are more). Returns (idx, n_band)."""
    s_gpu = np.asarray(s_gpu)
    rng = np.random.default_rng(seed)
    n = len(s_gpu)
    uni = rng.choice(n, min(n_uniform, n), replace=False) if n_uniform < n else np.arange(n)
    near = np.flatnonzero(np.abs(s_gpu) <= band)
    if near.size > band_max:
        near = rng.choice(near, band_max, replace=False)
    return np.unique(np.concatenate([uni, near])), int(near.size)


def score_stats(f_gpu, f_ref, label_gpu=None):
    """Max / 99.99th-percentile / rms error, R16 violations, label mismatches, and the same
    restricted to the near-zero queries (|f_ref| < 0.1, where the absolute floor binds)."""
    f_gpu = np.asarray(f_gpu, dtype=np.float64)
    f_ref = np.asarray(f_ref, dtype=np.float64)
    err = np.abs(f_gpu - f_ref)
    tol = np.maximum(REL * np.abs(f_ref), FLOOR)
    near = np.abs(f_ref) < 0.1
    out = dict(checked=int(err.size), max_err=float(err.max()) if err.size else 0.0,
               p9999_err=float(np.quantile(err, 0.9999)) if err.size else 0.0,
               rms_err=float(np.sqrt(np.mean(err ** 2))) if err.size else 0.0,
               violations=int(np.sum(err > tol)), max_err_over_tol=float(np.max(err / tol)) if err.size else 0.0,
               near_zero=int(near.sum()), near_zero_max_err=float(err[near].max()) if near.any() else 0.0)
    if label_gpu is not None:
        lab = np.asarray(label_gpu)
        sure = np.abs(f_ref) > LABEL_SURE
        out["label_mismatches"] = int(np.sum(sure & (lab != np.where(f_ref > 0, 1, -1))))
        out["label_ambiguous"] = int(np.sum(~sure))
    return out


def assert_stats(st, what):
    assert st["violations"] == 0, f"{what}: {st}"
    assert st.get("label_mismatches", 0) == 0, f"{what}: {st}"
