"""Exercise every C-ABI entry point on small inputs (for compute-sanitizer runs)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1910_06451_b200 as fb, workloads as W

wl = W.score_workload("cfg2", n_queries=3001, n_supports=333)
spos = fb.fastron_fk(wl.robot, torch.from_numpy(wl.supports).cuda())
qpos = fb.fastron_fk(wl.robot, torch.from_numpy(wl.queries).cuda())
al = torch.from_numpy(wl.alpha).cuda()
for kind in (0, 1):
    fb.fastron_score(qpos, spos, al, kind, 5.0)
    m = fb.fastron_model_pack(spos, al, kind, 5.0)
    fb.fastron_score_packed(qpos, m)
wl5 = W.score_workload("cfg5", n_queries=700, n_supports=130)
sp5 = fb.fastron_fk(wl5.robot, torch.from_numpy(wl5.supports).cuda())
qp5 = fb.fastron_fk(wl5.robot, torch.from_numpy(wl5.queries).cuda())
fb.fastron_score(qp5, sp5, torch.from_numpy(wl5.alpha).cuda(), 0, 5.0)
tw = W.train_workload(300)
pos = fb.fastron_fk(tw.robot, torch.from_numpy(tw.X).cuda())
K = fb.fastron_gram(pos, 0, 5.0)
P = np.transpose(pos.cpu().numpy()[:, :, :3], (1, 0, 2)).astype(np.float64)
y = torch.from_numpy(W.capsule_aabb_labels(W.chain_points(P), tw.cubes, tw.radius)).cuda()
fb.fastron_train(K, y, 1.0, 2000)
fb.fastron_train(K, y, 1.0, 2000, s_max=20)
ew = W.edge_workload(n_edges=70, n_supports=200)
sp = fb.fastron_fk(ew.robot, torch.from_numpy(ew.supports).cuda())
for n_interp in (1, 40, 64):
    fb.fastron_edge_check(ew.robot, torch.from_numpy(ew.qa).cuda(), torch.from_numpy(ew.qb).cuda(), n_interp, sp,
                          torch.from_numpy(ew.alpha).cuda(), 0, 5.0)
qh = torch.from_numpy(wl.queries).pin_memory()
sh = torch.empty(len(wl.queries), dtype=torch.float32).pin_memory()
fb.fastron_query(wl.robot, qh, spos, al, 0, 5.0, score=sh)
torch.cuda.synchronize()
print("sanitize workload ok")
