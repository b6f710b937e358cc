import sys, numpy as np, torch
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
from gpu_helpers import make_case, to_dev, D, oracle_results, oracle_problem, oimp, rel_vec_err, pose_err
from paper_2207_09442_b200.layer import PoseGraphSolver
for seed in (72, 66):
    topo, data = make_case(64, dim=3, p=0.3, seed=seed, B=3)
    t = to_dev(data)
    res = oracle_results(topo, data, max_iterations=8, implicit=True)
    v = np.random.default_rng(4).standard_normal((3, 64, 6))
    for cl in (1, 8):
        s = PoseGraphSolver(D.SE3, topo.num_poses, topo.edges, topo.prior_vars, device=0, max_iterations=8, cluster_ctas=cl)
        p, o, st, it = s.forward(t["poses0"], t["meas"], t["prior_meas"], t["w_edge"], t["w_prior"], implicit=True)
        ge, gp = s.backward(p, t["meas"], t["prior_meas"], t["w_edge"], t["w_prior"], torch.from_numpy(v).to("cuda"), D.GRAD_TANGENT, per_element=True)
        P = p.cpu().numpy()
        for b, r in enumerate(res):
            a, c, _ = oimp.implicit_weight_grads(oracle_problem(topo, data, b), r.x, v[b].reshape(-1), L_K=r.L_final)
            print(seed, cl, b, "pose", pose_err(P[b], r.x), "grad", rel_vec_err(np.concatenate([ge[b].cpu().numpy(), gp[b].cpu().numpy()]), np.concatenate([a, c])), "S", r.objective)
