import sys, numpy as np, torch
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
from gpu_helpers import make_case, to_dev, D
from paper_2207_09442_b200.layer import PoseGraphSolver
topo, data = make_case(64, dim=3, p=0.3, seed=72, B=3)
t = to_dev(data)
out = {}
for cl in (1, 2, 8):
    s = PoseGraphSolver(D.SE3, topo.num_poses, topo.edges, topo.prior_vars, device=0, max_iterations=8, cluster_ctas=cl)
    p, o, st, it = s.forward(t["poses0"], t["meas"], t["prior_meas"], t["w_edge"], t["w_prior"], implicit=True)
    ws = s.workspace(3)
    n = topo.num_poses * 6
    dense = torch.zeros(3, n, n, dtype=torch.float64, device="cuda")
    D.dnls_export_factor(s.graph, 3, ws, dense)
    torch.cuda.synchronize()
    out[cl] = (p.cpu().numpy(), dense.cpu().numpy())
for cl in (2, 8):
    dp = np.abs(out[cl][0] - out[1][0]).max()
    dl = np.abs(out[cl][1] - out[1][1])
    print("cl", cl, "pose diff", dp, "factor diff max", dl.max(), "n bad", (dl > 1e-9).sum(), "of", dl.size)
    idx = np.argwhere(dl > 1e-9)[:10]
    print(idx)
v = torch.from_numpy(np.random.default_rng(4).standard_normal((3, 64, 6))).to("cuda")
gs = {}
for cl in (1, 8):
    s = PoseGraphSolver(D.SE3, topo.num_poses, topo.edges, topo.prior_vars, device=0, max_iterations=8, cluster_ctas=cl)
    p, o, st, it = s.forward(t["poses0"], t["meas"], t["prior_meas"], t["w_edge"], t["w_prior"], implicit=True)
    ge, gp = s.backward(p, t["meas"], t["prior_meas"], t["w_edge"], t["w_prior"], v, D.GRAD_TANGENT, per_element=True)
    torch.cuda.synchronize()
    gs[cl] = ge.cpu().numpy()
    print(cl, "status", st.tolist(), it.tolist())
print("grad diff", np.abs(gs[8] - gs[1]).max(), np.abs(gs[1]).max())
