"""Time fastron_query_packed (configurations in, scores out) against FK + score_packed,
stream launches and CUDA-graph replays, over batch sizes (the fused one-launch query vs the
two-kernel path; FASTRON_QUERY_FUSED=0 disables the fused kernel). One JSON line per case;
hashes of the scores show the paths agree bit for bit."""
import hashlib, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1910_06451_b200 as fb, workloads as W

def timed(fn, reps):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); e1.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3

def graphed(fn, reps):
    side = torch.cuda.Stream(); side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side): fn()
    torch.cuda.current_stream().wait_stream(side); torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g): fn()
    return timed(g.replay, reps)

cases = [("cfg1", 10_000, None), ("cfg1", 37_888, None), ("cfg2", 37_888, None)] + \
    [("headline", n, None) for n in (33, 128, 1000, 2048, 4096, 16384, 37_888, 65536)] + \
    [("headline", n, 303) for n in (33, 1000, 10_000, 37_888)] + [("cfg5", n, None) for n in (512, 4096, 37_888)]
kind = int(os.environ.get("KIND", "0"))
for name, nq, ns in cases:
    wl = W.score_workload(name, n_queries=nq, n_supports=ns, kind=kind)
    robot = fb.make_robot_struct(wl.robot)
    model = fb.fastron_model_pack(fb.fastron_fk(robot, torch.from_numpy(wl.supports).cuda()),
                                  torch.from_numpy(wl.alpha).cuda(), kind, wl.gamma)
    q = torch.from_numpy(wl.queries).cuda()
    sc = torch.empty(nq, device="cuda"); lb = torch.empty(nq, dtype=torch.int8, device="cuda")
    L = fb.load_library()
    wsq = torch.empty(max(256, L.fastron_query_packed_workspace_bytes(nq, len(wl.supports), robot.n_cp, robot.dof)),
                      dtype=torch.uint8, device="cuda")
    qpos = torch.empty((robot.n_cp, nq, 4), device="cuda")
    wss = torch.empty(max(256, L.fastron_score_packed_workspace_bytes(nq, len(wl.supports), robot.n_cp)),
                      dtype=torch.uint8, device="cuda")
    f1 = lambda: fb.fastron_query_packed(robot, q, model, sc, lb, workspace=wsq)
    def f2():
        fb.fastron_fk(robot, q, pos=qpos); fb.fastron_score_packed(qpos, model, sc, lb, workspace=wss)
    reps = max(3, min(200, int(2e6 / nq)))
    out = {"wl": name, "nq": nq, "ns": len(wl.supports), "M": robot.n_cp, "kind": kind,
           "slab_max": os.environ.get("FASTRON_SLAB_MAX", "default")}
    out["query_packed_us"] = timed(f1, reps); out["query_packed_graph_us"] = graphed(f1, reps)
    h1 = hashlib.sha1(sc.cpu().numpy().tobytes()).hexdigest()[:10]
    out["fk_score_us"] = timed(f2, reps); out["fk_score_graph_us"] = graphed(f2, reps)
    h2 = hashlib.sha1(sc.cpu().numpy().tobytes()).hexdigest()[:10]
    out["same_bits"] = h1 == h2
    terms = nq * len(wl.supports) * robot.n_cp
    out["frac_R_query_graph"] = terms / (out["query_packed_graph_us"] * 1e-6) / (148 * 16 * 1.965e9)
    print(json.dumps(out), flush=True)
