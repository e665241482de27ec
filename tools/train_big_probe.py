"""Algorithm 1 at N > 2,048 (the cluster path) for several cluster sizes: the update
cycle's 8,446-point set size and 20,000. Traces must agree across C."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1910_06451_b200 as fb, workloads as W
robot = W.arm7(8)
cubes = W.train_workload().cubes
for N in [int(x) for x in os.environ.get("NS", "8446").split(",")]:
    X = W.cfg5_gram_workload(N)[1]
    pos = fb.fastron_fk(robot, torch.from_numpy(X).cuda())
    P = np.transpose(pos.cpu().numpy()[:, :, :3], (1, 0, 2)).astype(np.float64)
    y = torch.from_numpy(W.capsule_aabb_labels(W.chain_points(P), cubes, 0.05)).cuda()
    K = fb.fastron_gram(pos, 0, 5.0)
    ref = None
    for C in [int(c) for c in sys.argv[1:]]:
        os.environ["FASTRON_TRAIN_CLUSTER"] = str(C)
        out = fb.fastron_train(K, y, 1.0, 20000)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        out = fb.fastron_train(K, y, 1.0, 20000)
        e1.record(); e1.synchronize()
        res = fb.train_result(out["result"])
        tr = out["trace"].cpu().numpy()[:res["iterations"]]
        same = ref is None or np.array_equal(tr, ref)
        ref = tr if ref is None else ref
        print(json.dumps({"N": N, "C": C, "us_per_iter": e0.elapsed_time(e1) * 1e3 / max(1, res["iterations"]),
                          "iterations": res["iterations"], "same_trace": bool(same)}), flush=True)
