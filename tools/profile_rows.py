"""Runs the secondary rows once each (after one warm-up) for ncu captures:
cfg3 Gram (5000^2) + Algorithm 1 (20k iterations), cfg4 edge check, cfg1 score."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1910_06451_b200 as fb, workloads as W

which = sys.argv[1:] or ["gram", "train", "edge", "cfg1"]
tw = W.train_workload()
pos = fb.fastron_fk(tw.robot, torch.from_numpy(tw.X).cuda())
P = np.transpose(pos.cpu().numpy()[:, :, :3], (1, 0, 2)).astype(np.float64)
y = torch.from_numpy(W.capsule_aabb_labels(W.chain_points(P), tw.cubes, tw.radius)).cuda()
K = torch.empty((len(tw.X), len(tw.X)), device="cuda")
for rep in range(2):
    if "gram" in which or "train" in which:
        fb.fastron_gram(pos, 0, tw.gamma, K=K)
    if "train" in which:
        out = fb.fastron_train(K, y, 1.0, tw.iter_max)
    if "edge" in which:
        ew = W.edge_workload()
        sp = fb.fastron_fk(ew.robot, torch.from_numpy(ew.supports).cuda())
        fb.fastron_edge_check(ew.robot, torch.from_numpy(ew.qa).cuda(), torch.from_numpy(ew.qb).cuda(), 64, sp,
                              torch.from_numpy(ew.alpha).cuda(), 0, ew.gamma)
    if "cfg1" in which:
        wl = W.score_workload("cfg1")
        sp = fb.fastron_fk(wl.robot, torch.from_numpy(wl.supports).cuda())
        qp = fb.fastron_fk(wl.robot, torch.from_numpy(wl.queries).cuda())
        fb.fastron_score(qp, sp, torch.from_numpy(wl.alpha).cuda(), 0, wl.gamma)
if "gram5" in which:
    robot5, X5, _, _ = W.cfg5_gram_workload(8192)
    pos5 = fb.fastron_fk(robot5, torch.from_numpy(X5).cuda())
    for rep in range(2):
        fb.fastron_gram(pos5, 0, 5.0)
torch.cuda.synchronize()
if "train" in which:
    print(fb.train_result(out["result"]))
print("ok")
