"""cfg1 (10k queries x 1k supports, M = 4) and nearby mid-size batches: device time per call of
  * query_packed  — fastron_query_packed (configurations in: one launch + a ticket memset),
  * fk+score      — fastron_fk + fastron_score_packed (positions),
each as (a) one call per CUDA-graph replay, replays back to back (the bench row's method:
host launch rate included when the call is short) and (b) a graph of REPS calls replayed
once (device time per call, launch gaps included, host excluded). One JSON line per case.
FASTRON_RES_MAXQ=0 in the environment selects the tile-kernel path (A/B)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1910_06451_b200 as fb, workloads as W

REPS = 20


def graph_of(fn, calls):
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        fn()
    torch.cuda.current_stream().wait_stream(side)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(calls):
            fn()
    return g


def timed(fn, reps):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3  # us


cases = [("cfg1", None, None)] + [("cfg1", int(n), None) for n in os.environ.get("NQS", "").split(",") if n]
if os.environ.get("M8"):
    cases += [("cfg2", 4096, 303), ("cfg2", 10000, 1000)]
for name, nq, ns in cases:
    wl = W.score_workload(name, n_queries=nq, n_supports=ns)
    robot = fb.make_robot_struct(wl.robot)
    spos = fb.fastron_fk(robot, torch.from_numpy(wl.supports).cuda())
    model = fb.fastron_model_pack(spos, torch.from_numpy(wl.alpha).cuda(), wl.kind, wl.gamma)
    q = torch.from_numpy(wl.queries).cuda()
    n = len(wl.queries)
    sc = torch.empty(n, device="cuda")
    lb = torch.empty(n, dtype=torch.int8, device="cuda")
    L = fb.load_library()
    wq = torch.empty(max(256, L.fastron_query_packed_workspace_bytes(n, model.ns, robot.n_cp, robot.dof)),
                     dtype=torch.uint8, device="cuda")
    ws = torch.empty(max(256, L.fastron_score_packed_workspace_bytes(n, model.ns, robot.n_cp)), dtype=torch.uint8,
                     device="cuda")
    qpos = torch.empty((robot.n_cp, n, 4), device="cuda")
    out = {"case": name, "nq": n, "ns": model.ns, "M": robot.n_cp, "res_maxq": os.environ.get("FASTRON_RES_MAXQ")}
    fns = {"query_packed": lambda: fb.fastron_query_packed(robot, q, model, sc, lb, workspace=wq),
           "fk+score": lambda: (fb.fastron_fk(robot, q, pos=qpos), fb.fastron_score_packed(qpos, model, sc, lb,
                                                                                           workspace=ws))}
    for k, fn in fns.items():
        g1 = graph_of(fn, 1)
        gR = graph_of(fn, REPS)
        out[k] = {"stream_us": round(timed(fn, 50), 2), "graph_replay_us": round(timed(g1.replay, 50), 2),
                  "graph_per_call_us": round(timed(gR.replay, 5) / REPS, 2)}
    print(json.dumps(out), flush=True)
