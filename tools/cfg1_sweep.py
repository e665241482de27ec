"""cfg1 (10k x 1k, M = 4) one-launch query vs FK + score: CUDA-graph replay time over
forced split counts (FASTRON_SCORE_SPLITS) and the one-query-per-thread limit
(FASTRON_ONEQ_MAX). (fastron_query_packed = FK + score for these sizes.)"""
import hashlib, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1910_06451_b200 as fb, workloads as W
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from query_probe_lib import graphed, timed

name = os.environ.get("WL", "cfg1")
nq = int(os.environ.get("NQ", "0")) or None
wl = W.score_workload(name, n_queries=nq)
robot = fb.make_robot_struct(wl.robot)
model = fb.fastron_model_pack(fb.fastron_fk(robot, torch.from_numpy(wl.supports).cuda()),
                              torch.from_numpy(wl.alpha).cuda(), wl.kind, wl.gamma)
q = torch.from_numpy(wl.queries).cuda()
n = len(q)
sc = torch.empty(n, device="cuda"); lb = torch.empty(n, dtype=torch.int8, device="cuda")
L = fb.load_library()
ws = torch.empty(max(256, L.fastron_query_packed_workspace_bytes(n, len(wl.supports), robot.n_cp, robot.dof)),
                 dtype=torch.uint8, device="cuda")
for oq in os.environ.get("ONEQ", "128 16384").split():
    for sp in os.environ.get("SPLITS", "0 4 8 16").split():
        os.environ["FASTRON_ONEQ_MAX"] = oq
        os.environ["FASTRON_SCORE_SPLITS"] = sp
        f = lambda: fb.fastron_query_packed(robot, q, model, sc, lb, workspace=ws)
        g = graphed(f, 200)
        t = timed(f, 200)
        h = hashlib.sha1(sc.cpu().numpy().tobytes()).hexdigest()[:10]
        terms = n * len(wl.supports) * robot.n_cp
        print(json.dumps({"wl": name, "nq": n, "fused": os.environ.get("FASTRON_QUERY_FUSED", "1"), "oneq_max": oq,
                          "splits": sp, "graph_us": g, "stream_us": t, "frac_R": terms / (g * 1e-6) / (148 * 16 * 1.965e9),
                          "sha": h}), flush=True)
