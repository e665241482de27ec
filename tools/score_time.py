"""Time FK + packed scoring on a score workload (WL env: headline, cfg1, cfg2, cfg5; NQ
overrides the query count; KIND 0/1) and hash the scores; one JSON line. FASTRON_LIB
selects the library build (A/B probing: same hash = bit-identical scores)."""
import hashlib, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1910_06451_b200 as fb, workloads as W
name = os.environ.get("WL", "headline")
nq = int(os.environ["NQ"]) if os.environ.get("NQ") else None
wl = W.score_workload(name, n_queries=nq, kind=int(os.environ.get("KIND", "0")))
robot = fb.make_robot_struct(wl.robot)
M = wl.robot.n_cp
spos = fb.fastron_fk(robot, torch.from_numpy(wl.supports).cuda())
model = fb.fastron_model_pack(spos, torch.from_numpy(wl.alpha).cuda(), wl.kind, wl.gamma)
q = torch.from_numpy(wl.queries).cuda()
qpos = torch.empty((M, len(q), 4), device="cuda")
sc = torch.empty(len(q), device="cuda")
lb = torch.empty(len(q), dtype=torch.int8, device="cuda")
def step():
    fb.fastron_fk(robot, q, pos=qpos); fb.fastron_score_packed(qpos, model, sc, lb)
for _ in range(3): step()
torch.cuda.synchronize()
reps = max(1, min(50, int(2e11 / (len(q) * len(wl.alpha) * M))))
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); [step() for _ in range(reps)]; e1.record(); e1.synchronize()
ms = e0.elapsed_time(e1) / reps
print(json.dumps({"lib": os.environ.get("FASTRON_LIB", "default"), "wl": name, "kind": wl.kind, "nq": len(q),
                  "ms": ms, "frac": len(q) * len(wl.alpha) * M / (ms * 1e-3) / (148 * 16 * 1.965e9),
                  "sha": hashlib.sha1(sc.cpu().numpy().tobytes()).hexdigest()[:12]}), flush=True)
