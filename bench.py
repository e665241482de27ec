#!/usr/bin/env python
"""bench.py — headline benchmark of the Fastron FK hot path on B200.

Step = one pass of the proxy-collision-check path over one batch: batched FK of Q
query configurations (fastron_fk, K1) + FK-kernel scores and labels against the packed
support set (fastron_score_packed, K2). Workload (BASELINE.json north_star, DESIGN.md
R14): cfg2's 7-DOF arm, M = 8 control points, |S| = 20,000 supports (alpha ~ N(0,1)),
Q = 1,000,000 uniform queries per GPU, gamma = 5, Gaussian term. Metric: collision
checks/s (and kernel evaluations/s = checks/s x |S|); roofline = MUFU (SFU) throughput.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--rows]

Multi-GPU (torchrun, one rank per GPU): every rank scores its own 1M-query batch against
the replicated model — queries are independent units, so there is no data-path
collective ("scaling": "weak"); timing is the max over ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import workloads as W  # noqa: E402

METRIC = "7-DOF FK-kernel proxy collision checks/sec (1M queries x 20k supports, M=8)"
UNIT = "checks/s"
MUFU_PER_CLK_PER_SM = 16  # B200 SFU: 16 ex2/rcp per clock per SM (tools/pipe_peaks.cu measured 15.8)
MUFU_MEASURED_PER_CLK_PER_SM = 15.82  # profiles/r01/pipe_peaks.json (mufu_ex2)


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except Exception:
        return {}


def _parity(kind: int):
    """The committed parity statistics of this workload (tests/tools/parity_report.py, which
    compares the GPU path with oracle/ under SURVEY §8(c) C4; bench.py only reads its file)."""
    path = os.path.join(ROOT, "profiles", "r02", "parity.json")
    try:
        with open(path) as f:
            rep = json.load(f)
    except Exception:
        return None
    k = "gaussian" if kind == 0 else "rq"
    keep = ("checked", "sample", "max_err", "p9999_err", "rms_err", "violations", "max_err_over_tol",
            "near_zero", "near_zero_max_err", "label_mismatches")
    out = {"source": "profiles/r02/parity.json", "tolerance": "max(1e-4 |f|, 1e-5); labels where |f_ref| > 1e-4"}
    for name in ("headline", "cfg2", "cfg5", "cfg1"):
        st = rep.get(f"{name}_{k}")
        if st:
            out[name] = {kk: st[kk] for kk in keep if kk in st}
    return out


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []
        self.thread = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            if self.thread:
                self.thread.join(timeout=2)

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx.append(float(parts[2]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": float(max(mx)), "reasons": sorted(reasons),
                "samples": len(sm)}


def _dist():
    from paper_1910_06451_b200 import dist as fd
    return fd.world()


def _cpu_model() -> str:
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_baseline(wl, target_s=12.0):
    """The oracle as it stands, on this host's cores, on a bounded sample of the workload:
    the first Qs queries of the batch against all supports (FK + fp64 score)."""
    import oracle
    oracle.set_num_threads(os.cpu_count() or 1)  # all host cores (torchrun sets OMP_NUM_THREADS=1)
    spos = oracle.fk(wl.robot, wl.supports)

    def run(nq):
        t = time.perf_counter()
        f, _ = oracle.score(wl.kind, wl.gamma, oracle.fk(wl.robot, wl.queries[:nq]), spos, wl.alpha)
        return time.perf_counter() - t

    t64 = run(64)
    nq = int(min(len(wl.queries), max(64, 64 * target_s / max(t64, 1e-6))))
    dt = run(nq)
    cores = oracle.num_threads()
    # one thread, on a smaller sample (~target_s / 4 of CPU), for the per-core figure
    oracle.set_num_threads(1)
    try:
        t1 = run(16)
        n1 = int(min(len(wl.queries), max(16, 16 * target_s / 4 / max(t1, 1e-6))))
        dt1 = run(n1)
    finally:
        oracle.set_num_threads(cores)
    return {"value": nq / dt, "unit": UNIT, "cores": cores, "kind": "oracle", "cpu_model": _cpu_model(),
            "host_cpus": os.cpu_count(),
            "sample": f"first {nq} of the {len(wl.queries)} headline queries x all {len(wl.supports)} supports "
                      f"(fp64 FK + score, OpenMP), {dt:.1f} s",
            "kernel_evals_per_s": nq * len(wl.supports) / dt,
            "single_thread": {"value": n1 / dt1, "unit": UNIT, "sample": f"first {n1} queries, {dt1:.1f} s"}}


def run_reference(args):
    ws, rank, _ = _dist()
    if rank != 0:
        return 0
    import oracle
    oracle.set_num_threads(os.cpu_count() or 1)  # all host cores (torchrun sets OMP_NUM_THREADS=1)
    wl = W.score_workload("headline", kind=args.kind)
    spos = oracle.fk(wl.robot, wl.supports)
    # each step: a bounded sample of the batch (a different slice per step)
    t0 = time.perf_counter()
    oracle.score(wl.kind, wl.gamma, oracle.fk(wl.robot, wl.queries[:64]), spos, wl.alpha)
    per_q = (time.perf_counter() - t0) / 64
    nq = int(max(64, min(20000, 2.0 / max(per_q, 1e-9))))  # ~2 s of CPU per step
    for s in range(args.warmup):
        oracle.score(wl.kind, wl.gamma, oracle.fk(wl.robot, wl.queries[:64]), spos, wl.alpha)
    t = time.perf_counter()
    for s in range(args.steps):
        sl = slice(s * nq, (s + 1) * nq)
        oracle.score(wl.kind, wl.gamma, oracle.fk(wl.robot, wl.queries[sl]), spos, wl.alpha)
    dt = (time.perf_counter() - t) / args.steps
    value = nq / dt
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "headline", "n_supports": len(wl.supports), "queries_per_step": nq,
                       "n_cp": wl.robot.n_cp, "dof": wl.robot.dof, "gamma": wl.gamma,
                       "kernel": "gaussian" if wl.kind == 0 else "rq"},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": oracle.num_threads(), "kind": "oracle",
                             "cpu_model": _cpu_model(),
                             "sample": f"{nq} queries x {len(wl.supports)} supports per step"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def _time_rows(fb, torch, kind):
    """Secondary §8(a) rows, each timed on its own (not part of the headline step)."""
    rows = {}
    st = torch.cuda.current_stream()
    R_MUFU = 148 * 16 * 1.965e9  # MUFU roofline, ops/s

    def timed(fn, reps):
        fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(reps):
            fn()
        e1.record(st)
        e1.synchronize()
        return e0.elapsed_time(e1) / reps

    def graphed(fn, reps, calls=1):
        """The same calls captured once into a CUDA graph and replayed (SURVEY §8(d):
        separates launch overhead from kernel time). calls > 1 captures that many calls
        back to back in one graph and returns the time per call: the device time of a call
        in a stream of calls, with no host launch in between (one replay per `calls` calls;
        a graph of one short call replayed from Python is bound by the host's launch rate)."""
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
        return timed(g.replay, max(1, reps // calls)) / calls

    # cfg1: 3-DOF, 10k queries x 1k supports, M=4 (launch-latency scale)
    wl = W.score_workload("cfg1")
    spos = fb.fastron_fk(wl.robot, torch.from_numpy(wl.supports).cuda())
    model = fb.fastron_model_pack(spos, torch.from_numpy(wl.alpha).cuda(), kind, wl.gamma)
    q = torch.from_numpy(wl.queries).cuda()
    qpos = torch.empty((wl.robot.n_cp, len(wl.queries), 4), device="cuda")
    sc = torch.empty(len(wl.queries), device="cuda")
    lb = torch.empty(len(wl.queries), dtype=torch.int8, device="cuda")
    wsb = torch.empty(max(256, fb.load_library().fastron_score_packed_workspace_bytes(len(wl.queries), len(wl.supports),
                                                                                    wl.robot.n_cp)),
                      dtype=torch.uint8, device="cuda")

    def step1():
        fb.fastron_fk(wl.robot, q, pos=qpos)
        fb.fastron_score_packed(qpos, model, sc, lb, workspace=wsb)

    ms = timed(step1, 50)
    gms = graphed(step1, 50)
    dms = graphed(step1, 200, calls=20)
    rows["cfg1_score"] = {"ms": ms, "checks_per_s": len(wl.queries) / ms * 1e3,
                          "kernel_evals_per_s": len(wl.queries) * len(wl.supports) / ms * 1e3,
                          "graph_replay_ms": gms, "graph_checks_per_s": len(wl.queries) / gms * 1e3,
                          "graph_device_ms": dms, "graph_device_mufu_frac":
                              len(wl.queries) * len(wl.supports) * wl.robot.n_cp / (dms * 1e-3) / R_MUFU}
    # cfg2: 1M x 2k, M=8
    wl = W.score_workload("cfg2")
    spos = fb.fastron_fk(wl.robot, torch.from_numpy(wl.supports).cuda())
    model = fb.fastron_model_pack(spos, torch.from_numpy(wl.alpha).cuda(), kind, wl.gamma)
    q = torch.from_numpy(wl.queries).cuda()
    qpos = torch.empty((8, len(wl.queries), 4), device="cuda")
    sc = torch.empty(len(wl.queries), device="cuda")
    lb = torch.empty(len(wl.queries), dtype=torch.int8, device="cuda")

    def step2():
        fb.fastron_fk(wl.robot, q, pos=qpos)
        fb.fastron_score_packed(qpos, model, sc, lb)

    ms = timed(step2, 10)
    rows["cfg2_score"] = {"ms": ms, "checks_per_s": len(wl.queries) / ms * 1e3,
                          "kernel_evals_per_s": len(wl.queries) * len(wl.supports) / ms * 1e3}
    # cfg3: Gram 5000^2 + Algorithm 1 (labels from the product FK + the workload labeller)
    tw = W.train_workload()
    X = torch.from_numpy(tw.X).cuda()
    pos = fb.fastron_fk(tw.robot, X)
    P = np.transpose(pos.cpu().numpy()[:, :, :3], (1, 0, 2)).astype(np.float64)
    y = torch.from_numpy(W.capsule_aabb_labels(W.chain_points(P), tw.cubes, tw.radius)).cuda()
    K = torch.empty((len(tw.X), len(tw.X)), device="cuda")
    gws = torch.empty(fb.load_library().fastron_gram_workspace_bytes(len(tw.X), 8), dtype=torch.uint8, device="cuda")
    ms = timed(lambda: fb.fastron_gram(pos, tw.kind, tw.gamma, K=K, workspace=gws), 10)
    gms = graphed(lambda: fb.fastron_gram(pos, tw.kind, tw.gamma, K=K, workspace=gws), 10)
    dms = graphed(lambda: fb.fastron_gram(pos, tw.kind, tw.gamma, K=K, workspace=gws), 100, calls=10)
    n = len(tw.X)
    pair_ops = n * (n + 1) // 2 * 8  # MUFU ops of the unique pairs (the algorithmic work)
    rows["cfg3_gram"] = {"ms": ms, "unique_pairs": n * (n + 1) // 2,
                         "mufu_tops": pair_ops / ms * 1e-9, "mufu_frac_pairs": pair_ops / (ms * 1e-3) / R_MUFU,
                         "write_GBps": n * n * 4 / ms * 1e-6, "graph_replay_ms": gms, "graph_device_ms": dms,
                         "graph_device_mufu_frac_pairs": pair_ops / (dms * 1e-3) / R_MUFU}
    out = {}

    def train():
        out.update(fb.fastron_train(K, y, tw.beta, tw.iter_max))

    ms = timed(train, 3)
    res = fb.train_result(out["result"])
    rows["cfg3_train"] = {"ms": ms, **res, "us_per_iteration": ms * 1e3 / max(res["iterations"], 1),
                          "positive_fraction": float((y > 0).float().mean().item())}
    # the same Algorithm 1 with lazily computed, cached K columns (no Gram)
    lz = {}
    lws = torch.empty(fb.load_library().fastron_train_lazy_workspace_bytes(len(tw.X), 8, 4096), dtype=torch.uint8,
                      device="cuda")

    def train_lazy():
        lz.update(fb.fastron_train_lazy(pos, y, tw.kind, tw.gamma, tw.beta, tw.iter_max, cache_cols=4096,
                                        workspace=lws))

    ms = timed(train_lazy, 3)
    resl = fb.train_result(lz["result"])
    rows["cfg3_train_lazy"] = {"ms": ms, **resl, "us_per_iteration": ms * 1e3 / max(resl["iterations"], 1),
                               "same_as_full_gram": resl == res}
    # cfg5: M = 16 scoring (1M of the 10M queries x 20k supports) and the 20k x 20k Gram rebuild (R21)
    wl = W.score_workload("cfg5")  # the full BASELINE size: 10M queries x 20k supports, M = 16
    spos = fb.fastron_fk(wl.robot, torch.from_numpy(wl.supports).cuda())
    model = fb.fastron_model_pack(spos, torch.from_numpy(wl.alpha).cuda(), kind, wl.gamma)
    q = torch.from_numpy(wl.queries).cuda()
    qpos = torch.empty((16, len(wl.queries), 4), device="cuda")
    sc = torch.empty(len(wl.queries), device="cuda")
    lb = torch.empty(len(wl.queries), dtype=torch.int8, device="cuda")

    def step5():
        fb.fastron_fk(wl.robot, q, pos=qpos)
        fb.fastron_score_packed(qpos, model, sc, lb)

    ms = timed(step5, 2)
    terms = len(wl.queries) * len(wl.supports) * 16
    rows["cfg5_score_10M"] = {"ms": ms, "checks_per_s": len(wl.queries) / ms * 1e3,
                             "kernel_evals_per_s": len(wl.queries) * len(wl.supports) / ms * 1e3,
                             "mufu_frac": terms / (ms * 1e-3) / (148 * 16 * 1.965e9)}
    del qpos, q, sc, lb
    robot5, X5, _, _ = W.cfg5_gram_workload()
    pos5 = fb.fastron_fk(robot5, torch.from_numpy(X5).cuda())
    n5 = len(X5)
    K5 = torch.empty((n5, n5), device="cuda")
    gws5 = torch.empty(fb.load_library().fastron_gram_workspace_bytes(n5, 16), dtype=torch.uint8, device="cuda")
    ms = timed(lambda: fb.fastron_gram(pos5, kind, 5.0, K=K5, workspace=gws5), 3)
    nb = (n5 + 127) // 128
    rows["cfg5_gram"] = {"ms": ms, "n": n5, "mufu_frac_pairs": n5 * (n5 + 1) // 2 * 16 / (ms * 1e-3) / R_MUFU,
                         "write_GBps": n5 * n5 * 4 / ms * 1e-6}
    # Algorithm 1 at cfg5 scale (N = 20,000, M = 16; labels by the moved cubes, R21): on the
    # 1.6 GB Gram and with lazily computed columns (no Gram; the point planes of the 16
    # slices exceed shared memory and live in L2) — the same run bit for bit
    _, _, _, moved5 = W.cfg5_gram_workload()
    P8 = np.transpose(fb.fastron_fk(tw.robot, torch.from_numpy(X5).cuda()).cpu().numpy()[:, :, :3], (1, 0, 2))
    y5 = torch.from_numpy(W.capsule_aabb_labels(W.chain_points(P8.astype(np.float64)), moved5, 0.05)).cuda()
    o5 = {}
    ms = timed(lambda: o5.update(fb.fastron_train(K5, y5, 1.0, 20_000)), 2)
    r5 = fb.train_result(o5["result"])
    rows["cfg5_train"] = {"ms": ms, **r5, "us_per_iteration": ms * 1e3 / max(r5["iterations"], 1)}
    del K5
    torch.cuda.empty_cache()
    l5 = {}
    # column cache of 8,192 columns (655 MB): every column the run needs (6,586) is computed once
    lws5 = torch.empty(fb.load_library().fastron_train_lazy_workspace_bytes(n5, 16, 8192), dtype=torch.uint8,
                       device="cuda")
    ms = timed(lambda: l5.update(fb.fastron_train_lazy(pos5, y5, kind, 5.0, 1.0, 20_000, cache_cols=8192,
                                                       workspace=lws5)), 2)
    rl5 = fb.train_result(l5["result"])
    rows["cfg5_train_lazy"] = {"ms": ms, **rl5, "us_per_iteration": ms * 1e3 / max(rl5["iterations"], 1),
                               "cache_cols": 8192,
                               "same_as_full_gram": rl5 == r5 and bool(torch.equal(l5["alpha"], o5["alpha"]))}
    del lws5
    torch.cuda.empty_cache()
    # the model-update cycle (Table I "update time" 55.8 ms incl. FCL labelling):
    # fit on cfg3, move 3 of the 6 cubes by 0.1 m (R21), then 2 draws near every support point +
    # 1,000 uniform draws, GPU capsule labelling, Gram, warm-started Algorithm 1
    from paper_1910_06451_b200.model import CapsuleScene, FastronModel
    chain = [-1, 0, 1, 2, 3, 4, 5, 6, 7]
    mdl = FastronModel(tw.robot, tw.kind, tw.gamma, tw.beta, tw.iter_max)
    mdl.fit(X, y)
    ns0 = mdl.supports.shape[0]
    rng = np.random.default_rng(11)
    moved = tw.cubes.copy()
    for j in rng.choice(len(moved), 3, replace=False):
        v = rng.standard_normal(3)
        moved[j] += 0.1 * v / np.linalg.norm(v)
    scene = CapsuleScene(np.array(chain), moved, tw.radius)
    z = torch.from_numpy(rng.standard_normal((2 * ns0, 7)).astype(np.float32)).cuda()
    u = torch.from_numpy(rng.uniform(0, 1, (1000, 7)).astype(np.float32)).cuda()
    sig = torch.full((7,), 0.05 * 2 * np.pi, device="cuda")
    lo_t, hi_t = torch.full((7,), -np.pi, device="cuda"), torch.full((7,), np.pi, device="cuda")
    snap = (mdl.supports.clone(), mdl.alpha.clone(), mdl.model)
    upd = {}

    def cycle():
        mdl.supports, mdl.alpha, mdl.model = snap[0], snap[1], snap[2]
        upd["res"] = mdl.update(scene, z, u, sig, lo_t, hi_t, 2)[0]

    ms = timed(cycle, 3)
    rows["cfg3_update_cycle"] = {"ms": ms, "n_dataset": 3 * ns0 + 1000, **upd["res"],
                                 "paper_update_ms": 55.8, "note": "samples + FK + GPU labelling + Gram + warm-started Alg. 1"}
    # Table I context: Fastron FK (|S| = 303, M = 8) vs the joint-space "Fastron RBF" kernel
    # (|S| = 2369), the paper's mean support-set sizes, 1M queries each
    hw = W.score_workload("headline", n_queries=1_000_000)
    qd = torch.from_numpy(hw.queries).cuda()
    res_t1 = {}
    for name, ns in (("fk", 303), ("rbf_joint", 2369)):
        sup = torch.from_numpy(hw.supports[:ns]).cuda()
        al = torch.from_numpy(hw.alpha[:ns]).cuda()
        if name == "fk":
            sp = fb.fastron_fk(hw.robot, sup)
            mdl = fb.fastron_model_pack(sp, al, kind, hw.gamma)
            qp = torch.empty((8, len(hw.queries), 4), device="cuda")
            fn = lambda: (fb.fastron_fk(hw.robot, qd, pos=qp), fb.fastron_score_packed(qp, mdl))
        else:
            wsj = torch.empty(fb.load_library().fastron_score_joint_workspace_bytes(len(hw.queries), ns, 7),
                              dtype=torch.uint8, device="cuda")
            fn = lambda: fb.fastron_score_joint(qd, sup, al, kind, 0.5, workspace=wsj)
        ms = timed(fn, 5)
        res_t1[name] = {"n_supports": ns, "ms": ms, "checks_per_s": len(hw.queries) / ms * 1e3,
                        "us_per_check_batched": ms * 1e3 / len(hw.queries)}
    res_t1["fk_speedup_vs_rbf"] = res_t1["rbf_joint"]["ms"] / res_t1["fk"]["ms"]
    res_t1["paper_query_us"] = {"fk": 2.5, "rbf": 4.6, "note": "PAPER.md:290-291, single queries, unstated CPU"}
    rows["table1_query_sizes"] = res_t1
    # small batches (a planner asking a few configurations at a time): per-call latency of
    # FK + score for nq queries, stream launches vs a captured CUDA graph, at the Table I
    # FK model size (|S| = 303) and the headline model (|S| = 20,000)
    lat = {}
    robot_c = fb.make_robot_struct(hw.robot)
    for ns in (303, 20_000):
        sp = fb.fastron_fk(hw.robot, torch.from_numpy(hw.supports[:ns]).cuda())
        mdl = fb.fastron_model_pack(sp, torch.from_numpy(hw.alpha[:ns]).cuda(), kind, hw.gamma)
        for nq in (1, 64, 4096):
            qs = qd[:nq].contiguous()
            qp = torch.empty((8, nq, 4), device="cuda")
            sc = torch.empty(nq, device="cuda")
            lb = torch.empty(nq, dtype=torch.int8, device="cuda")
            wsl = torch.empty(max(256, fb.load_library().fastron_score_packed_workspace_bytes(nq, ns, 8)),
                              dtype=torch.uint8, device="cuda")
            fn = lambda: (fb.fastron_fk(hw.robot, qs, pos=qp), fb.fastron_score_packed(qp, mdl, sc, lb, workspace=wsl))
            lat[f"S{ns}_q{nq}"] = {"stream_us": timed(fn, 200) * 1e3, "graph_us": graphed(fn, 200) * 1e3,
                                   "graph_device_us": graphed(fn, 400, calls=20) * 1e3}
            if nq <= 32:  # fastron_query on device buffers: one fused launch for small batches
                sp_ = sp.contiguous()
                al_ = torch.from_numpy(hw.alpha[:ns]).cuda()
                qws_ = torch.empty(fb.load_library().fastron_query_workspace_bytes(nq, ns, 8, 7), dtype=torch.uint8,
                                   device="cuda")
                fq = lambda: fb.fastron_query(robot_c, qs, sp_, al_, kind, hw.gamma, score=sc, label=lb,
                                              workspace=qws_)
                lat[f"S{ns}_q{nq}"]["query_stream_us"] = timed(fq, 200) * 1e3
                lat[f"S{ns}_q{nq}"]["query_graph_us"] = graphed(fq, 200) * 1e3
            # fastron_query_packed: the planner's call (model packed once; one launch at nq <= 32)
            pws = torch.empty(max(256, fb.load_library().fastron_query_packed_workspace_bytes(nq, ns, 8, 7)),
                              dtype=torch.uint8, device="cuda")
            fqp = lambda: fb.fastron_query_packed(robot_c, qs, mdl, sc, lb, workspace=pws)
            lat[f"S{ns}_q{nq}"]["query_packed_stream_us"] = timed(fqp, 200) * 1e3
            lat[f"S{ns}_q{nq}"]["query_packed_graph_us"] = graphed(fqp, 200) * 1e3
            lat[f"S{ns}_q{nq}"]["query_packed_device_us"] = graphed(fqp, 400, calls=20) * 1e3
    rows["small_batch_latency"] = lat
    # cfg4: 10k edges x 64 points, 3k supports, early exit
    ew = W.edge_workload()
    spos = fb.fastron_fk(ew.robot, torch.from_numpy(ew.supports).cuda())
    qa, qb = torch.from_numpy(ew.qa).cuda(), torch.from_numpy(ew.qb).cuda()
    al = torch.from_numpy(ew.alpha).cuda()
    res = {}

    def edges():
        res["hit"], res["idx"] = fb.fastron_edge_check(ew.robot, qa, qb, ew.n_interp, spos, al, kind, ew.gamma)

    ms = timed(edges, 5)
    idx = res["idx"].cpu().numpy()
    hit = res["hit"].cpu().numpy()
    order = [2 * o for o in range(32)] + [2 * o + 1 for o in range(32)]
    pos_of = {k: o for o, k in enumerate(order)}
    rounds = np.array([1 if (h and pos_of[int(k)] < 32) else 2 for h, k in zip(hit, idx)])
    evaluated = int(np.sum(rounds * 32))
    rows["cfg4_edges"] = {"ms": ms, "edges_per_s": len(ew.qa) / ms * 1e3, "in_collision_fraction": float(hit.mean()),
                          "configs_evaluated": evaluated,
                          "evaluated_kernel_evals_per_s": evaluated * len(ew.supports) / ms * 1e3,
                          "mufu_frac_evaluated": evaluated * len(ew.supports) * ew.robot.n_cp / (ms * 1e-3)
                          / (148 * 16 * 1.965e9)}
    return rows


def run_ours(args):
    import torch
    import paper_1910_06451_b200 as fb
    ws, rank, local = _dist()
    torch.cuda.set_device(local)
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    fb.load_library()
    wl = W.score_workload("headline", kind=args.kind)
    from paper_1910_06451_b200 import dist as fd
    if args.strong:  # strong scaling: the one 1M-query batch cut into contiguous shards
        queries = np.ascontiguousarray(fd.shard(wl.queries, rank, ws))
    else:  # weak scaling: every rank its own batch of the workload's size
        queries = fd.shard_queries(wl.queries, rank)
    Q_total = len(wl.queries) if args.strong else ws * len(wl.queries)
    Q, S, M = len(queries), len(wl.supports), wl.robot.n_cp
    robot = fb.make_robot_struct(wl.robot)
    st = torch.cuda.current_stream()

    # model (support set): FK + pack once per model update, on rank 0; replicated to the
    # other ranks by one broadcast of the packed buffer, outside the timed region
    spos = fb.fastron_fk(robot, torch.from_numpy(wl.supports).cuda())
    model = fb.fastron_model_pack(spos, torch.from_numpy(wl.alpha).cuda(), wl.kind, wl.gamma)
    if ws > 1:
        if rank != 0:
            model.buf.zero_()
        fd.broadcast_model(model.buf, src=0)
        torch.cuda.synchronize()
    q = torch.from_numpy(queries).cuda()
    qpos = torch.empty((M, Q, 4), device="cuda")
    score = torch.empty(Q, device="cuda")
    label = torch.empty(Q, dtype=torch.int8, device="cuda")
    wsb = torch.empty(max(256, fb.load_library().fastron_score_packed_workspace_bytes(Q, S, M)), dtype=torch.uint8,
                      device="cuda")
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(args.steps)]

    def step(e=None):
        if e:
            e[0].record(st)
        fb.fastron_fk(robot, q, pos=qpos)
        if e:
            e[1].record(st)
        fb.fastron_score_packed(qpos, model, score, label, workspace=wsb)
        if e:
            e[2].record(st)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if ws > 1:
        torch.distributed.barrier()
    launches0 = fb.launch_count()
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record(st)
        for s in range(args.steps):
            step(ev[s])
        t1.record(st)
        torch.cuda.synchronize()
        if ws > 1:
            torch.distributed.barrier()
    launches = fb.launch_count() - launches0
    ms_total = t0.elapsed_time(t1)
    fk_ms = float(np.mean([e[0].elapsed_time(e[1]) for e in ev]))
    sc_ms = float(np.mean([e[1].elapsed_time(e[2]) for e in ev]))
    step_each = np.array([e[0].elapsed_time(e[2]) for e in ev])  # per-step FK start -> score end
    ms_step = fd.max_over_ranks(ms_total / args.steps, device="cuda")
    value = Q_total / (ms_step * 1e-3)  # all ranks' queries / the slowest rank's time
    clocks = clk.summary()

    # ---- end to end through the public API with host buffers (pinned), rank-local ----
    qh = torch.from_numpy(queries).pin_memory()
    sh = torch.empty(Q, dtype=torch.float32).pin_memory()
    lh = torch.empty(Q, dtype=torch.int8).pin_memory()
    qws = torch.empty(fb.load_library().fastron_query_workspace_bytes(Q, S, M, wl.robot.dof), dtype=torch.uint8,
                      device="cuda")

    def e2e_step():
        fb.fastron_query(robot, qh, spos, model_alpha, wl.kind, wl.gamma, score=sh, label=lh, workspace=qws)

    model_alpha = torch.from_numpy(wl.alpha).cuda()
    for _ in range(max(1, args.warmup)):
        e2e_step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(args.steps):
        e2e_step()
    e1.record(st)
    e1.synchronize()
    e2e_ms = fd.max_over_ranks(e0.elapsed_time(e1) / args.steps, device="cuda")
    assert np.array_equal(sh.numpy(), score.cpu().numpy()), "fastron_query disagrees with fk + score_packed"

    # ---- sharded edge checks (cfg4, strong scaling): the 10k edges cut into contiguous
    #      shards, each rank checks its shard against the broadcast packed model ----
    ew = W.edge_workload(kind=args.kind)
    emodel = fb.fastron_model_pack(fb.fastron_fk(robot, torch.from_numpy(ew.supports).cuda()),
                                   torch.from_numpy(ew.alpha).cuda(), ew.kind, ew.gamma)
    if ws > 1:
        fd.broadcast_model(emodel.buf, src=0)
    eqa, eqb = torch.from_numpy(ew.qa).cuda(), torch.from_numpy(ew.qb).cuda()
    eshard = lambda a, b: fb.fastron_edge_check_packed(robot, a, b, ew.n_interp, emodel)
    for _ in range(args.warmup):
        fd.sharded_map(eshard, len(ew.qa), eqa, eqb, gather=False)
    torch.cuda.synchronize()
    if ws > 1:
        torch.distributed.barrier()
    ee0, ee1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ee0.record(st)
    for _ in range(args.steps):
        fd.sharded_map(eshard, len(ew.qa), eqa, eqb, gather=False)
    ee1.record(st)
    ee1.synchronize()
    edge_ms = fd.max_over_ranks(ee0.elapsed_time(ee1) / args.steps, device="cuda")
    hit_all = fd.sharded_map(eshard, len(ew.qa), eqa, eqb)[0]  # gathered in edge order on every rank
    edges = {"workload": "cfg4 (10k edges x 64 points, 3k supports)", "scaling": "strong",
             "edges_per_s": len(ew.qa) / (edge_ms * 1e-3), "ms": edge_ms, "edges_per_gpu": len(fd.shard(ew.qa, rank, ws)),
             "in_collision_fraction": float(hit_all.float().mean().item())}

    # ---- roofline of the dominant kernel (the score launch) ----
    peaks = _peaks()
    sm_max = float(peaks.get("sm_max_mhz", 1965.0))
    sms = torch.cuda.get_device_properties(local).multi_processor_count
    peak = sms * MUFU_PER_CLK_PER_SM * sm_max * 1e6  # MUFU ops/s at the max SM clock
    achieved = Q * S * M / (sc_ms * 1e-3)
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "score_traffic.json")) as f:
            traffic = json.load(f).get("dram_bytes_per_launch")
    except Exception:
        pass
    roof = {"bound": "alu", "pipe": "MUFU (SFU) ex2" if wl.kind == 0 else "MUFU (SFU) rcp",
            "achieved": achieved * 1e-12, "peak": peak * 1e-12, "unit": "Tops/s", "frac": achieved / peak,
            "traffic": traffic, "kernel": "fastron_score_packed (score_kernel<8,kind,pos> + finalize" + (")" if wl.kind == 0 else "; RQ: pass 1 fast term + pass 2 refinement of |f| < 0.5)"),
            "peak_source": f"{sms} SMs x {MUFU_PER_CLK_PER_SM} MUFU/clk x {sm_max:.0f} MHz (MEASURED_PEAKS sm_max_mhz)",
            "frac_at_run_clock": (achieved / (sms * MUFU_PER_CLK_PER_SM * clocks["sm_mhz"] * 1e6)
                                  if clocks.get("sm_mhz") else None),
            # against the microbenchmarked MUFU rate (tools/pipe_peaks.cu: 15.82 ex2/clk/SM)
            "frac_vs_measured_mufu": achieved / (sms * MUFU_MEASURED_PER_CLK_PER_SM * sm_max * 1e6),
            "kernel_ms": sc_ms, "fk_ms": fk_ms,
            "fk_hbm_GBps": Q * (wl.robot.dof * 4 + M * 16) / (fk_ms * 1e-3) * 1e-9,
            "fk_hbm_frac": Q * (wl.robot.dof * 4 + M * 16) / (fk_ms * 1e-3) * 1e-9 / float(peaks.get("hbm_gbs", 6554.6))}

    rows = None
    if args.rows and rank == 0:
        rows = _time_rows(fb, torch, args.kind)

    base = None
    if rank == 0 and ws == 1 and not args.no_cpu:
        base = cpu_baseline(W.score_workload("headline", kind=args.kind))

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
                "scaling": "strong" if args.strong else "weak",
                "vs_baseline": None, "dtype": "f32 (fp64 FK and accumulation)", "data": "synthetic",
                "config": {"workload": "headline", "robot": "cfg2 7-DOF arm, M=8", "global_batch": Q_total,
                           "queries_per_gpu": Q, "n_supports": S, "n_cp": M, "dof": wl.robot.dof,
                           "gamma": wl.gamma, "kernel": "gaussian" if wl.kind == 0 else "rq",
                           "parallelism": f"dp{ws} ({'contiguous shards of one batch' if args.strong else 'a batch per rank'}"
                                          ", replicated model)",
                           "l2": "inputs larger than L2 (28 MB queries + 128 MB positions per step > 126 MB)"},
                "kernel_evals_per_s": value * S,
                "step_ms": {"min": float(step_each.min()), "median": float(np.median(step_each)),
                            "max": float(step_each.max())},
                "roofline": roof,
                "cpu_baseline": base,
                "e2e": {"value": Q_total / (e2e_ms * 1e-3), "unit": UNIT, "h2d_bytes_per_step": Q * wl.robot.dof * 4,
                        "d2h_bytes_per_step": Q * 5, "ms_per_step": e2e_ms,
                        "api": "fastron_query with pinned host q/score/label"},
                "gpu_launches": launches,
                "edge_check": edges,
                "parity": _parity(args.kind),
                "clocks": clocks}
        if rows is not None:
            line["rows"] = rows
        print(json.dumps(line), flush=True)
    if ws > 1:
        torch.distributed.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--kind", type=int, default=0, help="0 = Gaussian (north star), 1 = RQ (PAPER.md Eq. 3)")
    ap.add_argument("--rows", action="store_true", help="also time cfg1/cfg2/cfg3/cfg4 rows")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--strong", action="store_true",
                    help="strong scaling: split the one 1M-query batch over the ranks (default: weak, 1M per rank)")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # `python bench.py --gpus N` without a launcher: start one rank per GPU ourselves,
        # exactly as the driver does (torchrun, rendezvous on 127.0.0.1)
        import socket
        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        os.execv(sys.executable, [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                                  f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1", "--master-port",
                                  str(port), os.path.abspath(__file__)] + sys.argv[1:])
    ws_env = int(os.environ.get("WORLD_SIZE", "1"))
    if ws_env != args.gpus:
        print(f"note: --gpus {args.gpus} but WORLD_SIZE={ws_env}; reporting n_gpus={ws_env}", file=sys.stderr)
    if args.warmup < 3 and args.impl == "ours":
        print("note: warmup raised to 3 (timing rules)", file=sys.stderr)
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
