"""FastronModel — host orchestration of the C-ABI calls into the paper's workflow:
fit (Algorithm 1 on a labelled dataset), query (the proxy collision check) and update
(the two-stage active-learning cycle of PAPER.md:272 followed by a warm-started
Algorithm 1). Every arithmetic step runs in the library's kernels; this
module only allocates device tensors and sequences the calls.
"""
from __future__ import annotations

import dataclasses
from typing import Optional

import numpy as np

from . import (fastron_active_samples, fastron_fk, fastron_fk64, fastron_gram, fastron_kernel_matvec,
               fastron_kernel_matvec_lazy, fastron_score_precise,
               fastron_label_capsules, fastron_model_pack, fastron_query_packed, fastron_score_packed, fastron_train,
               fastron_train_lazy,
               make_robot_struct, train_result)


@dataclasses.dataclass
class CapsuleScene:
    """Geometric checker of the update cycle (the paper's FCL; here capsules vs boxes, R12)."""

    chain: np.ndarray  # int32 control-point indices (-1 = base origin)
    boxes: np.ndarray  # (n, 2, 3) or (n, 6) float64 lo/hi corners
    radius: float

    def flat_boxes(self) -> np.ndarray:
        return np.asarray(self.boxes, dtype=np.float64).reshape(-1, 6)


class FastronModel:
    def __init__(self, robot, kind: int = 0, gamma: float = 5.0, beta: float = 1.0, iter_max: int = 20000,
                 s_max: Optional[int] = None, lazy: bool = False, cache_cols: int = 4096, precise: bool = False):
        self.robot = robot
        self.robot_c = make_robot_struct(robot)
        self.kind, self.gamma, self.beta = int(kind), float(gamma), float(beta)
        self.iter_max, self.s_max, self.lazy, self.cache_cols = int(iter_max), s_max, bool(lazy), int(cache_cols)
        # precise: queries are scored on the fp64 path (unrounded positions, fp64 weights and
        # terms) — for trained models whose cancelling sums the fp32 path cannot resolve to
        # 1e-5 near the decision boundary (R25)
        self.precise = bool(precise)
        self.supports = None  # (|S|, D) device float32 configurations
        self.alpha = None  # (|S|,) device float64
        self.last = None  # result dict of the last training run

    # ---- Algorithm 1 on a dataset ----
    def _train(self, X, y, alpha0=None, F0=None):
        import torch
        pos = fastron_fk(self.robot_c, X)
        n = X.shape[0]
        s_max = n if self.s_max is None else self.s_max
        if self.lazy:
            if alpha0 is not None and F0 is None:  # margins of the loaded model: F = K alpha (as the full mode)
                F0 = fastron_kernel_matvec_lazy(pos, alpha0, self.kind, self.gamma)
            out = fastron_train_lazy(pos, y, self.kind, self.gamma, self.beta, self.iter_max, s_max, alpha=alpha0, F=F0,
                                     cache_cols=min(self.cache_cols, n))
        else:
            K = fastron_gram(pos, self.kind, self.gamma)
            if alpha0 is not None and F0 is None:
                F0 = fastron_kernel_matvec(K, alpha0)
            out = fastron_train(K, y, self.beta, self.iter_max, s_max, alpha=alpha0, F=F0)
        res = train_result(out["result"])
        sup = out["support_idx"][:res["n_support"]].long()
        self.supports = X[sup].contiguous()
        self.alpha = out["alpha"][sup].contiguous()
        self.labels = y[sup].contiguous()
        self.last = dict(res, n=n)
        self._pack()
        return self.last

    def _pack(self):
        spos = fastron_fk(self.robot_c, self.supports)
        self.model = fastron_model_pack(spos, self.alpha.float(), self.kind, self.gamma)
        self.spos64 = fastron_fk64(self.robot_c, self.supports) if self.precise else None

    def fit(self, X, y):
        """X: (N, D) float32 device configurations, y: (N,) int8 device labels (+1 = C_obs)."""
        return self._train(X, y)

    # ---- checkpoint / resume (loadPreviousModel) ----
    def state_dict(self) -> dict:
        """The trained model: support configurations, their fp64 weights and labels, and the
        kernel/training settings (the robot is the caller's; it is stored as its D-H table)."""
        import torch
        return {"supports": self.supports.cpu(), "alpha": self.alpha.cpu(), "labels": self.labels.cpu(),
                "kind": self.kind, "gamma": self.gamma, "beta": self.beta,
                "robot_dh": torch.as_tensor(np.asarray(self.robot.dh, dtype=np.float32)),
                "robot_cp_frame": torch.as_tensor(np.asarray(self.robot.cp_frame, dtype=np.int32)),
                "robot_cp_offset": torch.as_tensor(np.asarray(self.robot.cp_offset, dtype=np.float32)),
                "robot_base": torch.as_tensor(np.asarray(self.robot.base, dtype=np.float32))}

    def save(self, path: str) -> None:
        import torch
        torch.save(self.state_dict(), path)

    def load_state_dict(self, st: dict, device="cuda") -> None:
        """Restore a saved model (its robot must match this model's) and re-pack it."""
        # every part of the robot the scores depend on (D-H table, control-point frames and
        # offsets, base pose), compared after the same fp32 rounding the checkpoint applied
        mine = {"robot_dh": np.asarray(self.robot.dh, dtype=np.float32),
                "robot_cp_frame": np.asarray(self.robot.cp_frame, dtype=np.int32),
                "robot_cp_offset": np.asarray(self.robot.cp_offset, dtype=np.float32).reshape(-1, 3),
                "robot_base": np.asarray(self.robot.base, dtype=np.float32)}
        for key, v in mine.items():
            if key not in st or st[key].numpy().shape != v.shape or not np.array_equal(st[key].numpy(), v):
                raise ValueError(f"the saved model belongs to a different robot ({key} differs)")
        self.kind, self.gamma, self.beta = int(st["kind"]), float(st["gamma"]), float(st["beta"])
        self.supports = st["supports"].to(device).contiguous()
        self.alpha = st["alpha"].to(device).contiguous()
        self.labels = st["labels"].to(device).contiguous()
        self._pack()

    def load(self, path: str, device="cuda") -> None:
        import torch
        self.load_state_dict(torch.load(path, weights_only=True), device)

    # ---- proxy collision check ----
    def query(self, q):
        """Configurations q (n, D) device float32 -> (score, label): fastron_query_packed
        (one launch for small batches); precise models: fastron_fk64 + fastron_score_precise
        (fp64 scores)."""
        if self.precise:
            return fastron_score_precise(fastron_fk64(self.robot_c, q), self.spos64, self.alpha, self.kind, self.gamma)
        return fastron_query_packed(self.robot_c, q, self.model)

    def query_graph(self, nq: int):
        """A fixed-size query captured once as a CUDA graph (fastron_query_packed on static
        buffers): for planners that ask the same number of configurations again and again,
        a replay skips the per-call host work. Returns fn(q) -> (score, label); the outputs
        are reused buffers, so copy them before the next call. Valid until the model
        changes (fit / update / load)."""
        import torch
        from . import load_library
        dev = self.supports.device
        q_static = torch.zeros((nq, self.robot_c.dof), dtype=torch.float32, device=dev)
        score = torch.empty(nq, dtype=torch.float32, device=dev)
        label = torch.empty(nq, dtype=torch.int8, device=dev)
        ws = torch.empty(max(256, load_library().fastron_query_packed_workspace_bytes(
            nq, self.model.ns, self.model.n_cp, self.robot_c.dof)), dtype=torch.uint8, device=dev)
        model = self.model
        if self.precise:  # fp64 path: static fp64 positions and scores
            score = torch.empty(nq, dtype=torch.float64, device=dev)
            qpos64 = torch.empty((self.robot_c.n_cp, nq, 4), dtype=torch.float64, device=dev)
            spos64 = self.spos64

            def body():
                fastron_fk64(self.robot_c, q_static, pos=qpos64)
                fastron_score_precise(qpos64, spos64, self.alpha, self.kind, self.gamma, score=score, label=label)
            ws = (ws, qpos64, spos64)
        else:
            def body():
                fastron_query_packed(self.robot_c, q_static, model, score, label, workspace=ws)

        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            body()  # warm-up outside the capture (function attributes, occupancy cache)
        torch.cuda.current_stream().wait_stream(side)
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            body()

        keep = (q_static, score, label, ws, model)  # every buffer the graph touches stays alive

        def run(q):
            q_static.copy_(q, non_blocking=True)
            graph.replay()
            return score, label

        run.buffers = keep  # (freed buffers would be reused by the allocator while replays write them)
        return run

    # ---- the update cycle ----
    def update(self, scene: CapsuleScene, z, u, sigma, lo, hi, n_near: int):
        """Stage 1: n_near draws around every support point (z ~ N(0,1) inputs, scale sigma);
        stage 2: uniform draws (u ~ U[0,1) inputs). The support points and the new samples
        are labelled by the geometric check, then Algorithm 1 restarts from the previous
        alpha (loadPreviousModel) on that dataset."""
        import torch
        samples = fastron_active_samples(self.supports, n_near, z, sigma, u, lo, hi)
        X = torch.cat([self.supports, samples], dim=0).contiguous()
        pos = fastron_fk(self.robot_c, X)
        y = fastron_label_capsules(pos, scene.chain, scene.flat_boxes(), scene.radius)
        # loadPreviousModel: the support points keep their alpha, new samples start at 0
        alpha0 = torch.zeros(X.shape[0], dtype=torch.float64, device=X.device)
        alpha0[:self.supports.shape[0]] = self.alpha
        a_in = alpha0.clone()
        return self._train(X, y, alpha0=alpha0), X, y, a_in
