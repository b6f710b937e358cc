"""Small forward + backward runs for compute-sanitizer (memcheck / racecheck / synccheck / initcheck):
  python tools/sanitize_case.py <case>   case in c1 | c2 | cluster | lm | unroll | dlm | bl | bll
(bll: the batch-interleaved large-batch schedule forced on a small batch -- bl_subtree with a tight work cap, the
filtered chunked per-level items + bl_factor_red, the bl_lsolve tail solves in shared memory, PDL launches)
SURVEY.md §5 "race detection": the fused kernels rely on named barriers, mbarrier/TMA proxy ordering and
cluster barriers; these cases exercise each path once."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
from paper_2207_09442_b200 import dnls as D  # noqa: E402
from paper_2207_09442_b200.layer import PoseGraphSolver  # noqa: E402

case = sys.argv[1] if len(sys.argv) > 1 else "c2"
cfg = {"c1": (16, 2, 4, {}), "c2": (256, 3, 4, {}), "cluster": (1024, 3, 2, {"cluster_ctas": 2}),
       "lm": (64, 3, 3, {"optimizer": D.LM}), "unroll": (64, 3, 3, {}), "dlm": (64, 3, 3, {}),
       "bl": (64, 3, 40, {"batch_interleave": 32}), "bll": (256, 3, 40, {"batch_interleave": 32})}[case]
if case == "bll":
    os.environ.update(DNLS_BL_UPD="1", DNLS_BL_PERSIST="4", DNLS_BL_SUBW="20", DNLS_BL_LCH="2")
N, dim, B, opts = cfg
topo = synth.cube_topology(N, dim=dim, p=0.3, seed=0)
data = synth.cube_batch(topo, B, seed=0)
dev = torch.device("cuda", 0)
t = {k: torch.from_numpy(np.ascontiguousarray(v)).to(dev) for k, v in data.items() if k != "gt"}
group = D.SE3 if dim == 3 else D.SE2
solver = PoseGraphSolver(group, N, topo.edges, topo.prior_vars, device=0, max_iterations=3, **opts)
v = torch.randn(B, N, group, dtype=torch.float64, device=dev)
mode = {"unroll": D.BWD_UNROLL, "dlm": D.BWD_NONE}.get(case, D.BWD_IMPLICIT)
P, obj, st, it = solver.forward(t["poses0"], t["meas"], t["prior_meas"], t["w_edge"], t["w_prior"], backward_mode=mode)
bmode = {"unroll": "unroll", "dlm": "dlm"}.get(case, "implicit")
ge, gp = solver.backward(P, t["meas"], t["prior_meas"], t["w_edge"], t["w_prior"], v, D.GRAD_TANGENT, mode=bmode)
torch.cuda.synchronize()
print(case, "ok", obj.cpu().numpy()[:2], float(ge.abs().max()))
