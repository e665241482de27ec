"""cfg1 (10k queries x 1k supports, M = 4) through fastron_query_packed, a few calls (for
ncu launch lists of the fused one-launch query vs FK + score + finalize)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1910_06451_b200 as fb, workloads as W
name = os.environ.get("WL", "cfg1")
nq = int(os.environ.get("NQ", "0")) or None
wl = W.score_workload(name, n_queries=nq)
robot = fb.make_robot_struct(wl.robot)
model = fb.fastron_model_pack(fb.fastron_fk(robot, torch.from_numpy(wl.supports).cuda()),
                              torch.from_numpy(wl.alpha).cuda(), wl.kind, wl.gamma)
q = torch.from_numpy(wl.queries).cuda()
for _ in range(int(os.environ.get("REPS", "5"))):
    fb.fastron_query_packed(robot, q, model)
torch.cuda.synchronize()
print("ok")
