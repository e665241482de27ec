"""SURVEY.md §8(f) rank 4 (certified early exit): how many queries could
stop scoring early with a certified label? Supports are streamed in |alpha|-descending
order; after a prefix of p supports the unseen terms are bounded because every kernel
value lies in (0, 1] (Eq. 3/4 are means of terms in (0, 1]), so the sign of f is certain
once the partial sum exceeds the unseen mass of the opposite sign. A second, tighter bound
uses k >= k_min, the smallest kernel value over all sampled (query, support) pairs (not a
guarantee for unseen pairs; an upper estimate of what certification could ever save).

Models: the Algorithm 1 model trained on cfg3 (its real alpha: |S| = 2,48x, entries of both
signs up to ~200) and the headline's alpha ~ N(0, 1) over 20,000 supports.
Test infrastructure: every kernel value comes from oracle/ (oracle.score with one support
and alpha = 1). Writes profiles/r02/f4_certification.json.
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import oracle  # noqa: E402
import workloads as W  # noqa: E402

PREFIXES = (0.01, 0.05, 0.10, 0.25, 0.50, 0.75, 0.90, 1.0)


def kernel_matrix(kind, gamma, qp, sp):
    """k(q, s_i) for all queries (rows) and supports (columns), one oracle call per support."""
    out = np.empty((qp.shape[0], sp.shape[0]))
    one = np.ones(1, np.float32)
    for i in range(sp.shape[0]):
        out[:, i], _ = oracle.score(kind, gamma, qp, sp[i:i + 1], one)
    return out


def certify(alpha, Kq):
    """Per query: the first prefix length at which the label is certified (|S| + 1 = never),
    with the (0, 1] bound and with the [k_min, 1] estimate."""
    order = np.argsort(-np.abs(alpha), kind="stable")
    a = alpha[order].astype(np.float64)
    Kq = Kq[:, order]
    n = len(a)
    pos_after = np.concatenate([np.cumsum(np.where(a > 0, a, 0.0)[::-1])[::-1][1:], [0.0]])   # unseen + mass
    neg_after = np.concatenate([np.cumsum(np.where(a < 0, -a, 0.0)[::-1])[::-1][1:], [0.0]])  # unseen - mass
    kmin = float(Kq.min())
    first01 = np.full(Kq.shape[0], n + 1)
    firstk = np.full(Kq.shape[0], n + 1)
    S = np.zeros(Kq.shape[0])
    for p in range(n):
        S += a[p] * Kq[:, p]
        ok01 = (S > neg_after[p]) | (S < -pos_after[p])
        okk = (S + kmin * pos_after[p] - neg_after[p] > 0) | (S + pos_after[p] - kmin * neg_after[p] < 0)
        first01 = np.where((first01 > n) & ok01, p + 1, first01)
        firstk = np.where((firstk > n) & okk, p + 1, firstk)
    f = S
    res = {"supports": n, "queries": int(Kq.shape[0]), "k_min_sampled": kmin,
           "max_abs_alpha": float(np.abs(a).max()), "sum_abs_alpha": float(np.abs(a).sum()),
           "median_abs_f": float(np.median(np.abs(f)))}
    for name, first in (("bound_k_in_0_1", first01), ("estimate_k_in_kmin_1", firstk)):
        res[name] = {
            "certified_fraction_at_prefix": {f"{int(q * 100)}%": float(np.mean(first <= max(1, int(round(q * n)))))
                                             for q in PREFIXES},
            "mean_fraction_of_supports_scored": float(np.mean(np.minimum(first, n)) / n),
        }
    return res


def main():
    out = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "profiles", "r02", "f4_certification.json")
    nq = int(os.environ.get("NQ", "2000"))
    rep = {}
    # (1) the cfg3-trained model
    tw = W.train_workload()
    P = oracle.fk(tw.robot, tw.X)
    y = W.capsule_aabb_labels(W.chain_points(P), tw.cubes, tw.radius)
    K = oracle.gram(tw.kind, tw.gamma, P)
    r = oracle.train(K, y, tw.beta, tw.iter_max)
    sup = r["support"]
    alpha = r["alpha"][sup]
    q = W.uniform_configs(np.random.default_rng(77), nq, 7)
    qp = oracle.fk(tw.robot, q)
    rep["cfg3_trained_model"] = certify(alpha, kernel_matrix(tw.kind, tw.gamma, qp, P[sup]))
    rep["cfg3_trained_model"]["training"] = {k: r[k] for k in ("iterations", "n_add", "n_remove", "converged",
                                                                "n_support")}
    print(json.dumps(rep["cfg3_trained_model"]), flush=True)
    # (2) the headline model (alpha ~ N(0,1), 20k supports)
    wl = W.score_workload("headline", n_queries=nq // 4)
    rep["headline_random_alpha"] = certify(wl.alpha.astype(np.float64),
                                           kernel_matrix(wl.kind, wl.gamma, oracle.fk(wl.robot, wl.queries),
                                                         oracle.fk(wl.robot, wl.supports)))
    print(json.dumps(rep["headline_random_alpha"]), flush=True)
    os.makedirs(os.path.dirname(out), exist_ok=True)
    with open(out, "w") as fh:
        json.dump(rep, fh, indent=1)


if __name__ == "__main__":
    main()
