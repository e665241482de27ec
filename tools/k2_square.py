"""K2 (fastron_score_packed) on an n x n problem (n queries against the same n supports, M = 8):
the Gram's work shape through the scoring kernel, for comparing per-CTA efficiency."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1910_06451_b200 as fb, workloads as W
robot = W.train_workload().robot
rng = np.random.default_rng(11)
for n in [int(x) for x in os.environ.get("NS", "5000,20000").split(",")]:
    X = rng.uniform(-np.pi, np.pi, size=(n, 7)).astype(np.float32)
    pos = fb.fastron_fk(robot, torch.from_numpy(X).cuda())
    model = fb.fastron_model_pack(pos, torch.from_numpy(rng.standard_normal(n).astype(np.float32)).cuda(), 0, 5.0)
    sc = torch.empty(n, device="cuda"); lb = torch.empty(n, dtype=torch.int8, device="cuda")
    ws = torch.empty(max(256, fb.load_library().fastron_score_packed_workspace_bytes(n, n, 8)), dtype=torch.uint8, device="cuda")
    fb.fastron_score_packed(pos, model, sc, lb, workspace=ws)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        fb.fastron_score_packed(pos, model, sc, lb, workspace=ws)
    e1.record(); e1.synchronize()
    us = e0.elapsed_time(e1) / 20 * 1e3
    print(json.dumps({"k2_square_n": n, "us": round(us, 2), "frac_full_square": round(n * n * 8 / (us * 1e-6) / 4.653e12, 3)}))
