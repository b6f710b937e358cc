"""Per-stage device times of the hot path (stage-level C-ABI entry points, CUDA events).

usage: python tools/stage_times.py [C2|C4|...] [reps]
Prints linearize / factorize / solve / forward(K) / backward times in microseconds for the
bench configs, so the fused k_forward time can be attributed to its phases.
"""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import synth  # noqa: E402
from bench import CONFIGS  # noqa: E402
from paper_2207_09442_b200 import dnls as D  # noqa: E402
from paper_2207_09442_b200.layer import PoseGraphSolver  # noqa: E402


def timeit(fn, reps):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e3


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "C2"
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
    cfg = CONFIGS[name]
    B = cfg["B"] if cfg["scaling"] == "weak" else cfg["B"]
    topo = synth.cube_topology(cfg["N"], dim=cfg["dim"], p=cfg["p"], mode=cfg["mode"], seed=0)
    data = synth.cube_batch(topo, B, seed=0)
    dev = torch.device("cuda", 0)
    t = {k: torch.from_numpy(np.ascontiguousarray(v)).to(dev) for k, v in data.items()}
    group = D.SE3 if cfg["dim"] == 3 else D.SE2
    solver = PoseGraphSolver(group, topo.num_poses, topo.edges, topo.prior_vars, device=0, max_iterations=cfg["K"])
    g = solver.graph
    ws = solver.workspace(B)
    poses = t["poses0"].clone()
    obj = torch.zeros(B, dtype=torch.float64, device=dev)
    st = torch.zeros(B, dtype=torch.int32, device=dev)
    pr = D.make_problem(poses, t["meas"], t["prior_meas"], t["w_edge"], t["w_prior"], obj, st)
    n = topo.num_poses * g.d
    rhs = torch.randn(B, n, dtype=torch.float64, device=dev)
    x = torch.zeros_like(rhs)
    out = {"config": name, "B": B, "stats": {k: solver.stats[k] for k in
                                             ("nnz_L", "storage_doubles", "num_supernodes", "num_levels")}}
    out["linearize_us"] = timeit(lambda: D.dnls_linearize(g, B, pr, None, 0, ws), reps)
    D.dnls_linearize(g, B, pr, None, 0, ws)

    def fact():
        D.dnls_linearize(g, B, pr, None, 0, ws)
        D.dnls_factorize(g, B, ws, st)
    out["linearize+factorize_us"] = timeit(fact, reps)
    out["factorize_us"] = out["linearize+factorize_us"] - out["linearize_us"]
    out["solve_us"] = timeit(lambda: D.dnls_solve_factored(g, B, ws, rhs, x), reps)
    opt = solver.options
    opt.backward_mode = D.BWD_IMPLICIT

    def fwd():
        poses.copy_(t["poses0"])
        D.dnls_forward(g, B, opt, pr, ws)
    out["forward_us"] = timeit(fwd, reps)
    v = torch.randn(B, topo.num_poses, g.d, dtype=torch.float64, device=dev)
    ge = torch.zeros(topo.num_edges, dtype=torch.float64, device=dev)
    gp = torch.zeros(1, dtype=torch.float64, device=dev)
    out["backward_us"] = timeit(lambda: D.dnls_backward_implicit(g, B, pr, v, D.GRAD_TANGENT, ge, gp, 0, ws), reps)
    K = cfg["K"]
    out["forward_model_us"] = (K + 1) * (out["linearize_us"] + out["factorize_us"]) + K * out["solve_us"]
    print(json.dumps(out))


if __name__ == "__main__":
    main()
