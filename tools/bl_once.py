"""One batch-interleaved forward (+ implicit backward) of a bench config, for ncu launch lists:
  python tools/bl_once.py C5 [K] [interleave]"""
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

name = sys.argv[1] if len(sys.argv) > 1 else "C5"
K = int(sys.argv[2]) if len(sys.argv) > 2 else 1
il = int(sys.argv[3]) if len(sys.argv) > 3 else 32
cfg = CONFIGS[name]
B = cfg["B"]
topo = synth.cube_topology(cfg["N"], dim=cfg["dim"], p=cfg["p"], mode=cfg["mode"], seed=0)
data = synth.cube_batch(topo, B, seed=0)
dev = torch.device("cuda", 0)
t = {k: torch.from_numpy(np.ascontiguousarray(v)).to(dev) for k, v in data.items() if k != "gt"}
solver = PoseGraphSolver(D.SE3 if cfg["dim"] == 3 else D.SE2, topo.num_poses, topo.edges, topo.prior_vars, device=0,
                         max_iterations=K, batch_interleave=il)
v = torch.randn(B, topo.num_poses, 6, dtype=torch.float64, device=dev)
for _ in range(2):
    P, obj, st, it = solver.forward(t["poses0"], t["meas"], t["prior_meas"], t["w_edge"], t["w_prior"], implicit=True)
    solver.backward(P, t["meas"], t["prior_meas"], t["w_edge"], t["w_prior"], v, D.GRAD_TANGENT)
torch.cuda.synchronize()
print("done", name, B, K)
