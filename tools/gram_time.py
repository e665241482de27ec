"""Time fastron_gram on cfg3 (N=5000, M=8) and a 20k M=16 case (cfg5 size); one JSON line."""
import hashlib, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1910_06451_b200 as fb, workloads as W
out = {"lib": os.environ.get("FASTRON_LIB", "default")}
for name, (robot, X) in {"cfg3": (W.train_workload().robot, W.train_workload().X),
                         "cfg5": W.cfg5_gram_workload()[:2]}.items():
    pos = fb.fastron_fk(robot, torch.from_numpy(X).cuda())
    n = len(X)
    K = torch.empty((n, n), device="cuda")
    ws = torch.empty(fb.load_library().fastron_gram_workspace_bytes(n, robot.n_cp), dtype=torch.uint8, device="cuda")
    fb.fastron_gram(pos, 0, 5.0, K=K, workspace=ws)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 20 if n <= 5000 else 3
    e0.record()
    for _ in range(reps):
        fb.fastron_gram(pos, 0, 5.0, K=K, workspace=ws)
    e1.record(); e1.synchronize()
    ms = e0.elapsed_time(e1) / reps
    nb = (n + 127) // 128
    mufu = nb * (nb + 1) // 2 * 128 * 128 * robot.n_cp
    out[name] = {"ms": ms, "mufu_frac": mufu / (ms * 1e-3) / (148 * 16 * 1.965e9), "write_GBps": n * n * 4 / ms * 1e-6,
                 "sha": hashlib.sha1(K.cpu().numpy().tobytes()).hexdigest()[:12]}
print(json.dumps(out), flush=True)
