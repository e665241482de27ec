"""Per-query throughput of the headline score launch vs the query count, to measure the
last-wave (tail) loss: nq = 1,000,000 gives 8.8 waves; 1,022,976 gives exactly 9."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1910_06451_b200 as fb, workloads as W
wl = W.score_workload("headline")
robot = fb.make_robot_struct(wl.robot)
spos = fb.fastron_fk(robot, torch.from_numpy(wl.supports).cuda())
model = fb.fastron_model_pack(spos, torch.from_numpy(wl.alpha).cuda(), wl.kind, wl.gamma)
out = {}
for nq in (900_000, 1_000_000, 1_022_976, 1_100_000, 2_045_952):
    q = torch.from_numpy(W.uniform_configs(np.random.default_rng(9), nq, 7)).cuda()
    qpos = fb.fastron_fk(robot, q)
    sc = torch.empty(nq, device="cuda"); lb = torch.empty(nq, dtype=torch.int8, device="cuda")
    for _ in range(2):
        fb.fastron_score_packed(qpos, model, sc, lb)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        fb.fastron_score_packed(qpos, model, sc, lb)
    e1.record(); e1.synchronize()
    ms = e0.elapsed_time(e1) / 5
    out[nq] = {"ms": round(ms, 3), "frac": nq * 2e4 * 8 / (ms * 1e-3) / (148 * 16 * 1.965e9)}
print(json.dumps(out), flush=True)
