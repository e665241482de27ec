"""Gram time vs N at M = 8 (cfg3 robot, uniform configurations): efficiency against the MUFU
roofline as the triangle deepens (wave quantisation vs steady-state efficiency)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1910_06451_b200 as fb, workloads as W
robot = W.train_workload().robot
rng = np.random.default_rng(11)
for n in [int(x) for x in os.environ.get("NS", "1280,2560,5000,7680,10240,20000").split(",")]:
    X = rng.uniform(-np.pi, np.pi, size=(n, 7)).astype(np.float32)
    pos = fb.fastron_fk(robot, torch.from_numpy(X).cuda())
    K = torch.empty((n, n), device="cuda")
    ws = torch.empty(max(256, fb.load_library().fastron_gram_workspace_bytes(n, robot.n_cp)), dtype=torch.uint8,
                     device="cuda")
    fb.fastron_gram(pos, 0, 5.0, K=K, workspace=ws)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 20
    e0.record()
    for _ in range(reps):
        fb.fastron_gram(pos, 0, 5.0, K=K, workspace=ws)
    e1.record(); e1.synchronize()
    ms = e0.elapsed_time(e1) / reps
    nb = (n + 127) // 128
    mufu = nb * (nb + 1) // 2 * 128 * 128 * robot.n_cp
    exact = n * (n + 1) // 2 * robot.n_cp
    print(json.dumps({"n": n, "tiles": nb * (nb + 1) // 2, "us": round(ms * 1e3, 2),
                      "frac_tiles": round(mufu / (ms * 1e-3) / (148 * 16 * 1.965e9), 3),
                      "frac_pairs": round(exact / (ms * 1e-3) / (148 * 16 * 1.965e9), 3)}), flush=True)
