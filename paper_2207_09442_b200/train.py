"""End-to-end learning of the cost weights through the solver (BASELINE.json configs C4/C5: "learnable cost
weights trained end-to-end via implicit differentiation"; Eq. 2 :74-79 outer loop, Listing 1
:104-131 with torch.optim.Adam, :168 robust PGO learning).

Outer loop: phi = log w (one learnable weight per Between edge, shared by the batch), inner loop = the
TheseusLayer-style ``pose_graph_layer`` (K Gauss-Newton iterations on the GPU, implicit backward through the
cached factor), outer loss = mean over the batch of || theta*(w) - theta_gt ||^2 on the pose matrices.
With outlier loop closures (SURVEY.md §8(d) "outlier variant") the loss pushes the outliers' weights down.

    python -m paper_2207_09442_b200.train [--poses 1024] [--batch 256] [--epochs 20]
"""
from __future__ import annotations

import argparse
import json
import time

import numpy as np
import torch

from . import dnls as D
from .layer import PoseGraphSolver, pose_graph_layer


def learn_cost_weights(topo, data, epochs: int = 20, lr: float = 0.05, iterations: int = 10,
                       backward_mode: str = "implicit", device: int = 0, group=None):
    """Adam over log-weights.  Returns a history dict: loss, mean weight of outlier / inlier edges per epoch,
    device time per epoch (CUDA events around forward + backward + optimizer step)."""
    dev = torch.device("cuda", device)
    group = group if group is not None else (D.SE3 if topo.dim == 3 else D.SE2)
    solver = PoseGraphSolver(group, topo.num_poses, topo.edges, topo.prior_vars, device=device,
                             max_iterations=iterations)
    t = {k: torch.from_numpy(np.ascontiguousarray(v)).to(dev) for k, v in data.items() if k != "gt"}
    gt = torch.from_numpy(np.ascontiguousarray(data["gt"])).to(dev)[None]     # [1][N][r][r+1]
    logw = torch.zeros(topo.num_edges, dtype=torch.float64, device=dev, requires_grad=True)
    opt = torch.optim.Adam([logw], lr=lr)
    out = torch.from_numpy(topo.outlier).to(dev)
    hist = {"loss": [], "w_outlier": [], "w_inlier": [], "epoch_ms": [], "status_failed": []}
    for _ in range(epochs):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        opt.zero_grad()
        w = torch.exp(logw)
        poses, obj, st, it = pose_graph_layer(solver, t["poses0"], t["meas"], t["prior_meas"], w, t["w_prior"],
                                              backward_mode=backward_mode)
        loss = ((poses - gt) ** 2).sum(dim=(1, 2, 3)).mean()
        loss.backward()
        opt.step()
        b.record()
        torch.cuda.synchronize()
        with torch.no_grad():
            w = torch.exp(logw)
            hist["loss"].append(float(loss))
            hist["w_outlier"].append(float(w[out].mean()) if bool(out.any()) else float("nan"))
            hist["w_inlier"].append(float(w[~out].mean()))
            hist["epoch_ms"].append(a.elapsed_time(b))
            hist["status_failed"].append(int(((st & D.ST_CODE_MASK) == D.ST_NOT_SPD).sum()))
    hist["final_weights"] = torch.exp(logw).detach().cpu().numpy().tolist()
    return hist


def main():
    import synth
    ap = argparse.ArgumentParser()
    ap.add_argument("--poses", type=int, default=1024)
    ap.add_argument("--batch", type=int, default=256)
    ap.add_argument("--epochs", type=int, default=20)
    ap.add_argument("--iterations", type=int, default=10)
    ap.add_argument("--lr", type=float, default=0.05)
    ap.add_argument("--outliers", type=float, default=0.1)
    ap.add_argument("--backward", default="implicit", choices=["implicit", "dlm", "unroll"])
    args = ap.parse_args()
    topo = synth.cube_topology(args.poses, dim=3, p=0.2, seed=0, outlier_ratio=args.outliers)
    data = synth.cube_batch(topo, args.batch, seed=0)
    t0 = time.perf_counter()
    h = learn_cost_weights(topo, data, args.epochs, args.lr, args.iterations, args.backward)
    wall = time.perf_counter() - t0
    summary = {"poses": args.poses, "batch": args.batch, "edges": topo.num_edges,
               "outlier_edges": int(topo.outlier.sum()), "epochs": args.epochs, "backward": args.backward,
               "loss_first": h["loss"][0], "loss_last": h["loss"][-1],
               "w_outlier": h["w_outlier"], "w_inlier": h["w_inlier"],
               "epoch_ms_median": float(np.median(h["epoch_ms"][1:] or h["epoch_ms"])),
               "wall_s_total": wall}
    print(json.dumps(summary))


if __name__ == "__main__":
    main()
