"""Time fastron_train on cfg3 (N=5000, 20k iterations) for several cluster sizes and
check every run gives the same trace (the kernel is deterministic for any C)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1910_06451_b200 as fb, workloads as W
N = int(os.environ.get("TRAIN_N", "5000"))
tw = W.train_workload(N)
pos = fb.fastron_fk(tw.robot, torch.from_numpy(tw.X).cuda())
P = np.transpose(pos.cpu().numpy()[:, :, :3], (1, 0, 2)).astype(np.float64)
y = torch.from_numpy(W.capsule_aabb_labels(W.chain_points(P), tw.cubes, tw.radius)).cuda()
K = fb.fastron_gram(pos, 0, tw.gamma)
ref = None
for C in [int(c) for c in (sys.argv[1:] or ["1", "2", "4", "8", "16"])]:
    os.environ["FASTRON_TRAIN_CLUSTER"] = str(C)
    out = fb.fastron_train(K, y, 1.0, tw.iter_max)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        out = fb.fastron_train(K, y, 1.0, tw.iter_max)
    e1.record(); e1.synchronize()
    ms = e0.elapsed_time(e1) / 3
    res = fb.train_result(out["result"])
    tr = out["trace"].cpu().numpy()[:res["iterations"]]
    same = ref is None or np.array_equal(tr, ref)
    al = out["alpha"].cpu().numpy()
    sup = out["support_idx"].cpu().numpy()[:res["n_support"]]
    if ref is None:
        ref, aref = tr, al
    print(json.dumps({"C": C, "ms": ms, "us_per_iter": ms * 1e3 / max(1, res["iterations"]), "same_trace": bool(same),
                      "nnz_alpha": int(np.count_nonzero(al)), "alpha_maxdiff": float(np.abs(al - aref).max()),
                      "support_ok": bool(np.array_equal(sup, np.flatnonzero(al))), **res}), flush=True)
