"""CPU emulation of the scoring kernel's fp32 arithmetic for the RQ term (Eq. 3) at the
headline size, against the fp64 oracle, splitting the error by source (R24).
Test infrastructure: it reads only oracle/ and workloads/."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import oracle, workloads as W

NQ = int(os.environ.get("NQ", "300"))
wl = W.score_workload("headline", kind=W.RQ, n_queries=NQ)
qp, sp = oracle.fk(wl.robot, wl.queries), oracle.fk(wl.robot, wl.supports)
g, a, f32 = wl.gamma, wl.alpha.astype(np.float64), np.float32
c = f32(np.sqrt(g / 2))
S = (sp.astype(f32) * c).astype(f32)


def lanes32(r):  # even / odd lanes: acc = fma(r, r, acc) in fp32 (one rounding), then promoted
    r = r.astype(np.float64)
    l0, l1 = (r[:, 0] * r[:, 0]).astype(f32), (r[:, 1] * r[:, 1]).astype(f32)
    for m in range(2, r.shape[1], 2):
        l0 = (r[:, m] * r[:, m] + l0.astype(np.float64)).astype(f32)
        l1 = (r[:, m + 1] * r[:, m + 1] + l1.astype(np.float64)).astype(f32)
    return l0.astype(np.float64) + l1.astype(np.float64)


err = {k: [] for k in ("fp32 positions + pre-scale", "+ fp32 term arithmetic (fp64 sums)",
                       "+ fp32 lane sums (kernel)")}
for i in range(NQ):
    ref = (a * (1.0 / (1.0 + g / 2 * ((qp[i][None] - sp) ** 2).sum(-1)) ** 2).mean(-1)).sum()
    Q = (qp[i].astype(f32) * c).astype(f32)
    d = Q[None].astype(np.float64) - S.astype(np.float64)
    err["fp32 positions + pre-scale"].append((a * (1 / (1 + (d ** 2).sum(-1)) ** 2).mean(-1)).sum() - ref)
    d = (Q[None] - S).astype(f32)
    d2 = (d[..., 0] * d[..., 0]).astype(f32)
    d2 = (d2 + (d[..., 1] * d[..., 1]).astype(f32)).astype(f32)
    d2 = (d2 + (d[..., 2] * d[..., 2]).astype(f32)).astype(f32)
    w = (f32(1) + d2).astype(f32)
    r = (f32(1) / w).astype(f32)  # the kernel: r = rcp(1 + d2), terms r^2 fused into the lane sums
    M = r.shape[1]
    t = (r.astype(np.float64) ** 2).astype(f32)
    err["+ fp32 term arithmetic (fp64 sums)"].append((a * t.astype(np.float64).sum(-1)).sum() / M - ref)
    err["+ fp32 lane sums (kernel)"].append((a * lanes32(r)).sum() / M - ref)
for k, v in err.items():
    v = np.abs(np.array(v))
    print(f"{k:40s} rms {np.sqrt((v ** 2).mean()):.2e}  max {v.max():.2e}")
