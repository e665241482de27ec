"""fastron_train_lazy at cfg5 scale (N = 20,000, M = 16, 20,000 iterations) for the column
cache sizes given on the command line (default 4096 8192); one JSON line each. With a
-DFASTRON_TRAIN_PROF build the kernel also prints the computed columns and their cost."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1910_06451_b200 as fb, workloads as W
tw = W.train_workload()
robot5, X5, _, moved5 = W.cfg5_gram_workload()
pos5 = fb.fastron_fk(robot5, torch.from_numpy(X5).cuda())
n5 = len(X5)
P8 = np.transpose(fb.fastron_fk(tw.robot, torch.from_numpy(X5).cuda()).cpu().numpy()[:, :, :3], (1, 0, 2))
y5 = torch.from_numpy(W.capsule_aabb_labels(W.chain_points(P8.astype(np.float64)), moved5, 0.05)).cuda()
ref = None
for cc in [int(c) for c in (sys.argv[1:] or ["4096", "8192"])]:
    ws = torch.empty(fb.load_library().fastron_train_lazy_workspace_bytes(n5, 16, cc), dtype=torch.uint8, device="cuda")
    out = fb.fastron_train_lazy(pos5, y5, 0, 5.0, 1.0, 20_000, cache_cols=cc, workspace=ws)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); out = fb.fastron_train_lazy(pos5, y5, 0, 5.0, 1.0, 20_000, cache_cols=cc, workspace=ws); e1.record()
    e1.synchronize()
    res = fb.train_result(out["result"])
    tr = out["trace"].cpu().numpy()[:res["iterations"]]
    same = ref is None or np.array_equal(tr, ref); ref = tr if ref is None else ref
    print(json.dumps({"cache_cols": cc, "us_per_iter": e0.elapsed_time(e1) * 1e3 / max(1, res["iterations"]),
                      "distinct_columns": int(len(np.unique(np.abs(tr)))), "same_trace": bool(same), **res}), flush=True)
    del ws
