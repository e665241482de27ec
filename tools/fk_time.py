"""Time fastron_fk (K1) on the headline batch (1M x 7 joints, M = 8) and cfg5's M = 16;
one JSON line (FASTRON_LIB selects the library build)."""
import hashlib, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1910_06451_b200 as fb, workloads as W
out = {"lib": os.environ.get("FASTRON_LIB", "default")}
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for name, n_cp in (("m8", 8), ("m16", 16)):
    robot = fb.make_robot_struct(W.arm7(n_cp))
    q = torch.from_numpy(W.uniform_configs(np.random.default_rng(1), 1_000_000, 7)).cuda()
    pos = torch.empty((n_cp, len(q), 4), device="cuda")
    for _ in range(3):
        fb.fastron_fk(robot, q, pos=pos)
    ts = []
    for _ in range(10):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fb.fastron_fk(robot, q, pos=pos); e1.record(); e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = float(np.median(ts))
    byts = len(q) * (4 * 7 + 16 * n_cp)
    out[name] = {"us": ms * 1e3, "GBps": byts / ms * 1e-6, "hbm_frac": byts / ms * 1e-6 / 6554.6,
                 "sha": hashlib.sha1(pos.cpu().numpy().tobytes()).hexdigest()[:12]}
print(json.dumps(out), flush=True)
