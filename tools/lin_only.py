"""Run dnls_linearize repeatedly (profiling target: ncu -k regex:k_linearize)."""
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

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
B = int(sys.argv[2]) if len(sys.argv) > 2 else 128
cfg = CONFIGS[name]
topo = synth.cube_topology(cfg["N"], dim=cfg["dim"], p=cfg["p"], mode=cfg["mode"], seed=0)
data = synth.cube_batch(topo, B, seed=0)
dev = torch.device("cuda", 0)
t = {k: torch.from_numpy(np.ascontiguousarray(v)).to(dev) for k, v in data.items()}
solver = PoseGraphSolver(D.SE3 if cfg["dim"] == 3 else D.SE2, topo.num_poses, topo.edges, topo.prior_vars, device=0)
g = solver.graph
ws = solver.workspace(B)
pr = D.make_problem(t["poses0"], t["meas"], t["prior_meas"], t["w_edge"], t["w_prior"])
for _ in range(4):
    D.dnls_linearize(g, B, pr, None, 0, ws)
torch.cuda.synchronize()
print("done")
