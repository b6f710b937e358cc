import sys, numpy as np, torch
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
from gpu_helpers import make_case, to_dev, D
from paper_2207_09442_b200.layer import PoseGraphSolver
topo, data = make_case(64, dim=3, p=0.3, seed=72, B=3)
t = to_dev(data)
for K in (1, 2, 4):
    res = {}
    for cl in (1, 8):
        s = PoseGraphSolver(D.SE3, topo.num_poses, topo.edges, topo.prior_vars, device=0, max_iterations=K, cluster_ctas=cl)
        for rep in range(3):
            p, o, st, it = s.forward(t["poses0"], t["meas"], t["prior_meas"], t["w_edge"], t["w_prior"], implicit=False)
            torch.cuda.synchronize()
            res[(cl, rep)] = (p.cpu().numpy(), o.cpu().numpy())
    for rep in range(3):
        d = np.abs(res[(8, rep)][0] - res[(1, 0)][0]).reshape(3, -1).max(axis=1)
        do = np.abs(res[(8, rep)][1] - res[(1, 0)][1])
        print("K", K, "rep", rep, "pose diff per element", d, "obj diff", do, flush=True)
