"""Time the headline step and measure score error stats for one library build
(FASTRON_LIB env selects the .so). Prints one JSON line."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_1910_06451_b200 as fb, workloads as W, oracle
wl = W.score_workload("headline", kind=int(os.environ.get("KIND", "0")))
robot = fb.make_robot_struct(wl.robot)
spos = fb.fastron_fk(robot, torch.from_numpy(wl.supports).cuda())
model = fb.fastron_model_pack(spos, torch.from_numpy(wl.alpha).cuda(), wl.kind, wl.gamma)
q = torch.from_numpy(wl.queries).cuda()
qpos = torch.empty((8, len(q), 4), device="cuda"); sc = torch.empty(len(q), device="cuda"); lb = torch.empty(len(q), dtype=torch.int8, device="cuda")
def step():
    fb.fastron_fk(robot, q, pos=qpos); fb.fastron_score_packed(qpos, model, sc, lb)
for _ in range(3): step()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); [step() for _ in range(5)]; e1.record(); e1.synchronize()
ms = e0.elapsed_time(e1) / 5
s = sc.cpu().numpy().astype(np.float64)
if os.environ.get("NO_ORACLE"):  # timing + output hash only (A/B of bit-identical variants)
    import hashlib
    print(json.dumps({"lib": os.environ.get("FASTRON_LIB", "default"), "kind": wl.kind, "ms": ms,
                      "frac": 1e6 * 2e4 * 8 / (ms * 1e-3) / (148 * 16 * 1.965e9),
                      "sha": hashlib.sha1(sc.cpu().numpy().tobytes()).hexdigest()[:12]}), flush=True)
    sys.exit(0)
rng = np.random.default_rng(1)
idx = np.unique(np.concatenate([rng.choice(len(s), 3000, replace=False), np.argsort(np.abs(s))[:1000]]))
f, _ = oracle.score(wl.kind, wl.gamma, oracle.fk(wl.robot, wl.queries[idx]), oracle.fk(wl.robot, wl.supports), wl.alpha)
err = np.abs(s[idx] - f); tol = np.maximum(1e-4 * np.abs(f), 1e-5)
print(json.dumps({"lib": os.environ.get("FASTRON_LIB", "default"), "kind": wl.kind, "ms": ms,
                  "frac": 1e6 * 2e4 * 8 / (ms * 1e-3) / (148 * 16 * 1.965e9),
                  "err_rms": float(np.sqrt(np.mean(err ** 2))), "err_max": float(err.max()),
                  "violations": int(np.sum(err > tol)), "checked": int(len(idx))}), flush=True)
