"""Where the model-update cycle's time goes (bench row cfg3_update_cycle): each stage of
FastronModel.update timed with events (a synchronise per stage, so the sum exceeds the
pipelined cycle). One JSON line."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1910_06451_b200 as fb, workloads as W
from paper_1910_06451_b200.model import CapsuleScene, FastronModel
tw = W.train_workload()
X = torch.from_numpy(tw.X).cuda()
pos = fb.fastron_fk(tw.robot, X)
P = np.transpose(pos.cpu().numpy()[:, :, :3], (1, 0, 2)).astype(np.float64)
y = torch.from_numpy(W.capsule_aabb_labels(W.chain_points(P), tw.cubes, tw.radius)).cuda()
mdl = FastronModel(tw.robot, tw.kind, tw.gamma, tw.beta, tw.iter_max)
mdl.fit(X, y)
ns0 = mdl.supports.shape[0]
rng = np.random.default_rng(11)
moved = tw.cubes.copy()
for j in rng.choice(len(moved), 3, replace=False):
    v = rng.standard_normal(3); moved[j] += 0.1 * v / np.linalg.norm(v)
scene = CapsuleScene(np.array([-1, 0, 1, 2, 3, 4, 5, 6, 7]), moved, tw.radius)
z = torch.from_numpy(rng.standard_normal((2 * ns0, 7)).astype(np.float32)).cuda()
u = torch.from_numpy(rng.uniform(0, 1, (1000, 7)).astype(np.float32)).cuda()
sig = torch.full((7,), 0.05 * 2 * np.pi, device="cuda")
lo_t, hi_t = torch.full((7,), -np.pi, device="cuda"), torch.full((7,), np.pi, device="cuda")
snap = (mdl.supports.clone(), mdl.alpha.clone(), mdl.model)
out = {}
def stage(name, fn, reps=3):
    fn(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        r = fn()
    torch.cuda.synchronize()
    out[name] = round((time.perf_counter() - t0) / reps * 1e3, 3)
    return r
def whole():
    mdl.supports, mdl.alpha, mdl.model = snap
    return mdl.update(scene, z, u, sig, lo_t, hi_t, 2)
stage("cycle_ms", whole)
mdl.supports, mdl.alpha, mdl.model = snap
samples = stage("samples", lambda: fb.fastron_active_samples(mdl.supports, 2, z, sig, u, lo_t, hi_t))
Xn = stage("cat", lambda: torch.cat([mdl.supports, samples], dim=0).contiguous())
posn = stage("fk", lambda: fb.fastron_fk(mdl.robot_c, Xn))
yn = stage("label", lambda: fb.fastron_label_capsules(posn, scene.chain, scene.flat_boxes(), scene.radius))
def mk_alpha():
    a = torch.zeros(Xn.shape[0], dtype=torch.float64, device="cuda"); a[:ns0] = snap[1]; return a
a0 = stage("alpha0", mk_alpha)
K = stage("gram", lambda: fb.fastron_gram(posn, mdl.kind, mdl.gamma))
F0 = stage("matvec", lambda: fb.fastron_kernel_matvec(K, a0))
tr = stage("train", lambda: fb.fastron_train(K, yn, mdl.beta, mdl.iter_max, Xn.shape[0], alpha=a0.clone(), F=F0.clone()))
res = stage("result_readback", lambda: fb.train_result(tr["result"]))
def post():
    sup = tr["support_idx"][:res["n_support"]].long()
    s2 = Xn[sup].contiguous(); al = tr["alpha"][sup].contiguous(); lb = yn[sup].contiguous()
    sp = fb.fastron_fk(mdl.robot_c, s2)
    return fb.fastron_model_pack(sp, al.float(), mdl.kind, mdl.gamma)
stage("gather_pack", post)
out["n"] = int(Xn.shape[0]); out["iterations"] = res["iterations"]
print(json.dumps(out))
