"""Time fastron_edge_check on cfg4 (10k edges x 64 points, 3k supports, M = 8); one JSON
line (FASTRON_LIB selects the library build)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1910_06451_b200 as fb, workloads as W
ew = W.edge_workload(kind=int(os.environ.get("KIND", "0")))
spos = fb.fastron_fk(ew.robot, torch.from_numpy(ew.supports).cuda())
al = torch.from_numpy(ew.alpha).cuda()
qa, qb = torch.from_numpy(ew.qa).cuda(), torch.from_numpy(ew.qb).cuda()
run = lambda: fb.fastron_edge_check(ew.robot, qa, qb, ew.n_interp, spos, al, ew.kind, ew.gamma)
hit, idx = run()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    hit, idx = run()
e1.record(); e1.synchronize()
ms = e0.elapsed_time(e1) / 10
h = hit.cpu().numpy()
ix = idx.cpu().numpy()
nround2 = int((h == 0).sum() + ((h == 1) & (ix % 2 == 1)).sum())  # edges that needed round 2 (odd points)
evaluated = 32 * len(h) + 32 * nround2
print(json.dumps({"lib": os.environ.get("FASTRON_LIB", "default"), "ms": ms, "hits": int(h.sum()),
                  "evaluated": evaluated, "frac": evaluated * len(ew.supports) * 8 / (ms * 1e-3) / (148 * 16 * 1.965e9),
                  "idx_sum": int(ix.sum())}), flush=True)
