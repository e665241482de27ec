"""Parity statistics of the GPU path against the fp64 oracle under the C4 protocol of
SURVEY.md §8(c) (tests/c4.py), per BASELINE.json config and kernel shape. Writes one
JSON file (default profiles/r02/parity.json). Test infrastructure: expected values come
only from oracle/; the GPU side is called through the binding of the C ABI.

    python tests/tools/parity_report.py [OUT.json] [--only cfg1,cfg2,headline,cfg5,cfg4,gram,trained]
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_1910_06451_b200 as fb  # noqa: E402
import workloads as W  # noqa: E402
from c4 import c4_sample, score_stats  # noqa: E402

KINDS = {0: "gaussian", 1: "rq"}


def gpu_scores(robot, sup, alpha, q, kind, gamma):
    spos = fb.fastron_fk(robot, torch.from_numpy(sup).cuda())
    qpos = fb.fastron_fk(robot, torch.from_numpy(q).cuda())
    s, l = fb.fastron_score(qpos, spos, torch.from_numpy(alpha).cuda(), kind, gamma)
    torch.cuda.synchronize()
    return s.cpu().numpy().astype(np.float64), l.cpu().numpy()


def score_case(name, kind, n_uniform=None, seed=0):
    wl = W.score_workload(name, kind=kind)
    t0 = time.time()
    s, l = gpu_scores(wl.robot, wl.supports, wl.alpha, wl.queries, kind, wl.gamma)
    if n_uniform is None:  # every query
        idx, n_band = np.arange(len(s)), int(np.sum(np.abs(s) <= 1e-2))
    else:
        idx, n_band = c4_sample(s, n_uniform, seed)
    f, _ = oracle.score(kind, wl.gamma, oracle.fk(wl.robot, wl.queries[idx]), oracle.fk(wl.robot, wl.supports),
                        wl.alpha)
    st = score_stats(s[idx], f, l[idx])
    st.update(queries=len(s), supports=len(wl.supports), M=wl.robot.n_cp, sample="all" if n_uniform is None else
              f"{n_uniform} uniform + {n_band} with |f_gpu| <= 1e-2", seconds=round(time.time() - t0, 1))
    return st


def edge_case(kind):
    wl = W.edge_workload(kind=kind)
    spos = fb.fastron_fk(wl.robot, torch.from_numpy(wl.supports).cuda())
    hit, idx = fb.fastron_edge_check(wl.robot, torch.from_numpy(wl.qa).cuda(), torch.from_numpy(wl.qb).cuda(),
                                     wl.n_interp, spos, torch.from_numpy(wl.alpha).cuda(), kind, wl.gamma)
    torch.cuda.synchronize()
    hit, idx = hit.cpu().numpy(), idx.cpu().numpy()
    ref, fmax, fall = oracle.edge(wl.robot, wl.qa, wl.qb, wl.n_interp, kind, wl.gamma,
                                  oracle.fk(wl.robot, wl.supports), wl.alpha, with_all=True)
    sure = np.abs(fmax) > 1e-4
    bad_hit_point = sum(1 for e in np.flatnonzero(hit) if fall[e, idx[e]] <= -1e-4)
    return dict(edges=len(hit), checked=len(hit), in_collision=int(hit.sum()),
                label_mismatches=int(np.sum(sure & (hit != ref))), ambiguous=int(np.sum(~sure)),
                hit_points_with_f_ref_below_minus_1e4=int(bad_hit_point))


def gram_case(kind):
    tw = W.train_workload()
    pos = fb.fastron_fk(tw.robot, torch.from_numpy(tw.X).cuda())
    K = fb.fastron_gram(pos, kind, tw.gamma).cpu().numpy().astype(np.float64)
    Kref = oracle.gram(kind, tw.gamma, oracle.fk(tw.robot, tw.X))
    err = np.abs(K - Kref)
    tol = np.maximum(1e-4 * np.abs(Kref), 1e-5)
    return dict(n=len(K), entries=int(K.size), max_err=float(err.max()), violations=int(np.sum(err > tol)),
                symmetric=bool(np.array_equal(K, K.T)), unit_diagonal=bool(np.all(np.diag(K) == 1.0)))


def trained_case(kind):
    """Queries against a model trained by Algorithm 1 on cfg3 (alpha of both signs and
    magnitude ~10-100): R16 on every query, plus the count of queries whose sum is
    ill-conditioned (kappa = sum_i |alpha_i| k_i / |f| > 1e4), reported separately."""
    from paper_1910_06451_b200.model import FastronModel
    tw = W.train_workload()
    y = W.capsule_aabb_labels(W.chain_points(oracle.fk(tw.robot, tw.X)), tw.cubes, tw.radius)
    m = FastronModel(tw.robot, kind=kind, gamma=tw.gamma, iter_max=tw.iter_max)
    res = m.fit(torch.from_numpy(tw.X).cuda(), torch.from_numpy(y).cuda())
    q = W.uniform_configs(np.random.default_rng(77), 50_000, 7)
    s, l = m.query(torch.from_numpy(q).cuda())
    torch.cuda.synchronize()
    s, l = s.cpu().numpy().astype(np.float64), l.cpu().numpy()
    a32 = m.alpha.float().cpu().numpy()
    sup = m.supports.cpu().numpy()
    qp, sp = oracle.fk(tw.robot, q), oracle.fk(tw.robot, sup)
    f, _ = oracle.score(kind, tw.gamma, qp, sp, a32)
    cond, _ = oracle.score(kind, tw.gamma, qp, sp, np.abs(a32))
    st = score_stats(s, f, l)
    kappa = cond / np.maximum(np.abs(f), 1e-300)
    st.update(n_support=int(res["n_support"]), max_abs_alpha=float(np.abs(a32).max()),
              ill_conditioned_kappa_gt_1e4=int(np.sum(kappa > 1e4)),
              max_err_over_condition=float(np.max(np.abs(s - f) / cond)))
    ok = kappa <= 1e4
    st["non_cancelling_queries"] = score_stats(s[ok], f[ok], l[ok])
    # the same model on the fp64 path (fastron_fk64 + fastron_score_precise, fp64 alpha)
    import paper_1910_06451_b200 as fbm
    s64, l64 = fbm.fastron_score_precise(fbm.fastron_fk64(tw.robot, torch.from_numpy(q).cuda()),
                                         fbm.fastron_fk64(tw.robot, m.supports), m.alpha, kind, tw.gamma)
    torch.cuda.synchronize()
    f64, _ = oracle.score(kind, tw.gamma, qp, sp, m.alpha.cpu().numpy(), exact_alpha=True)
    st["fp64_path_every_query"] = score_stats(s64.cpu().numpy(), f64, l64.cpu().numpy())
    return st


def main():
    out = next((a for a in sys.argv[1:] if a.endswith(".json")), os.path.join(ROOT, "profiles", "r02", "parity.json"))
    only = None
    if "--only" in sys.argv:
        only = set(sys.argv[sys.argv.index("--only") + 1].split(","))
    want = (lambda k: only is None or k in only)
    rep = {"protocol": "SURVEY.md §8(c) C4; tolerance max(1e-4|f|, 1e-5), labels where |f_ref| > 1e-4",
           "library": fb.LIB_PATH if hasattr(fb, "LIB_PATH") else "", "oracle_threads": oracle.num_threads()}
    for kind in (0, 1):
        k = KINDS[kind]
        if want("cfg1"):
            rep[f"cfg1_{k}"] = score_case("cfg1", kind)
        if want("cfg2"):
            rep[f"cfg2_{k}"] = score_case("cfg2", kind)
        if want("headline"):
            rep[f"headline_{k}"] = score_case("headline", kind, n_uniform=50_000, seed=10 + kind)
        if want("cfg5"):
            rep[f"cfg5_{k}"] = score_case("cfg5", kind, n_uniform=10_000, seed=20 + kind)
        if want("cfg4"):
            rep[f"cfg4_edges_{k}"] = edge_case(kind)
        if want("gram"):
            rep[f"cfg3_gram_{k}"] = gram_case(kind)
        if want("trained"):
            rep[f"cfg3_trained_model_{k}"] = trained_case(kind)
        print(json.dumps({kk: v for kk, v in rep.items() if kk.endswith(k)}), flush=True)
    os.makedirs(os.path.dirname(out), exist_ok=True)
    with open(out, "w") as fh:
        json.dump(rep, fh, indent=1)
    print("wrote", out)


if __name__ == "__main__":
    main()
