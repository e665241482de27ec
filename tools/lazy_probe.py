"""Time fastron_train_lazy (Algorithm 1 with K columns computed on demand) on cfg3 for the
cluster sizes given on the command line; traces must agree across C."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1910_06451_b200 as fb, workloads as W
tw = W.train_workload()
pos = fb.fastron_fk(tw.robot, torch.from_numpy(tw.X).cuda())
P = np.transpose(pos.cpu().numpy()[:, :, :3], (1, 0, 2)).astype(np.float64)
y = torch.from_numpy(W.capsule_aabb_labels(W.chain_points(P), tw.cubes, tw.radius)).cuda()
ref = None
for C in [int(c) for c in sys.argv[1:]]:
    os.environ["FASTRON_TRAIN_CLUSTER"] = str(C)
    out = fb.fastron_train_lazy(pos, y, 0, tw.gamma, 1.0, tw.iter_max, cache_cols=4096)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); out = fb.fastron_train_lazy(pos, y, 0, tw.gamma, 1.0, tw.iter_max, cache_cols=4096); e1.record(); e1.synchronize()
    tr = out["trace"].cpu().numpy()
    same = ref is None or np.array_equal(tr, ref); ref = tr if ref is None else ref
    print(json.dumps({"C": C, "us": e0.elapsed_time(e1) * 1e3 / 20000, "same": bool(same)}), flush=True)
