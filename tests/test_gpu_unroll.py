"""-m gpu parity of the Unroll / Truncated backward (
include/dnls.h dnls_backward_unroll) against the oracle (oracle/unroll.py, pinned by FD of the unrolled
K-step map): weight gradients (batch-summed and per element) and the theta_init gradient at the
north_star gradient tolerance 1e-6, theta_K at 1e-9; truncation windows; the history-state contract."""
import numpy as np
import pytest
import torch

from gpu_helpers import DEV, TOL_GRAD, TOL_POSE, D, make_case, olie, oracle_problem, pose_err, rel_vec_err, to_dev
from oracle import unroll as ounroll
from paper_2207_09442_b200._lib import DnlsError
from paper_2207_09442_b200.layer import PoseGraphSolver, pose_graph_layer

pytestmark = pytest.mark.gpu


def run_unroll(topo, data, K, mode, steps=0, alpha=1.0, seed=0):
    group = D.SE3 if topo.dim == 3 else D.SE2
    solver = PoseGraphSolver(group, topo.num_poses, topo.edges, topo.prior_vars, device=0, max_iterations=K,
                             step_size=alpha)
    t = to_dev(data)
    B = data["poses0"].shape[0]
    P, obj, st, it = solver.forward(t["poses0"], t["meas"], t["prior_meas"], t["w_edge"], t["w_prior"],
                                    backward_mode=mode, backward_steps=steps)
    v = np.random.default_rng(seed).standard_normal((B, topo.num_poses, group))
    g0 = torch.zeros(B, topo.num_poses, group, dtype=torch.float64, device=DEV)
    ge, gp = solver.backward(P, t["meas"], t["prior_meas"], t["w_edge"], t["w_prior"],
                             torch.from_numpy(v).to(DEV), D.GRAD_TANGENT, per_element=True, mode="unroll",
                             grad_poses0=g0)
    torch.cuda.synchronize()
    return P.cpu().numpy(), ge.cpu().numpy(), gp.cpu().numpy(), g0.cpu().numpy(), v, st.cpu().numpy()


@pytest.mark.parametrize("N,dim,B,K,mode,steps,alpha", [
    (16, 2, 4, 4, D.BWD_UNROLL, 0, 1.0),           # C1-sized SE2
    (27, 3, 3, 3, D.BWD_UNROLL, 0, 1.0),
    (27, 3, 2, 4, D.BWD_UNROLL, 0, 0.7),           # damped step alpha
    (30, 3, 3, 5, D.BWD_TRUNCATED, 2, 1.0),        # truncated window < K: biased, no theta_init gradient
    (20, 2, 2, 3, D.BWD_TRUNCATED, 7, 1.0),        # window >= K: identical to unroll
])
def test_unroll_matches_oracle(N, dim, B, K, mode, steps, alpha):
    topo, data = make_case(N, dim=dim, p=0.4, seed=N + K, B=B, sigma_t=0.2, sigma_r=0.1)
    P, ge, gp, g0, v, st = run_unroll(topo, data, K, mode, steps, alpha)
    assert np.all((st & D.ST_CODE_MASK) == D.ST_OK)
    trunc = None if mode == D.BWD_UNROLL else steps
    for b in range(B):
        prob = oracle_problem(topo, data, b)
        TK, gw_o, gp_o, g0_o = ounroll.unroll_weight_grads(prob, olie.to_homog(data["poses0"][b]), K, v[b], alpha,
                                                            truncate=trunc)
        assert pose_err(P[b], TK) <= TOL_POSE
        g_gpu = np.concatenate([ge[b], gp[b]])
        g_ora = np.concatenate([gw_o, gp_o])
        assert rel_vec_err(g_gpu, g_ora) <= TOL_GRAD, (b, rel_vec_err(g_gpu, g_ora))
        if trunc is None or trunc >= K:
            assert rel_vec_err(g0[b].reshape(-1), g0_o.reshape(-1)) <= TOL_GRAD
        else:
            assert np.all(g0[b] == 0)


def test_unroll_layer_autograd_and_state():
    topo, data = make_case(16, dim=3, p=0.4, seed=3, B=2)
    solver = PoseGraphSolver(D.SE3, topo.num_poses, topo.edges, topo.prior_vars, device=0, max_iterations=3)
    t = to_dev(data)
    w = t["w_edge"].clone().requires_grad_(True)
    P, obj, st, it = pose_graph_layer(solver, t["poses0"], t["meas"], t["prior_meas"], w, t["w_prior"],
                                      backward_mode="unroll")
    (P ** 2).sum().backward()
    assert w.grad is not None and torch.isfinite(w.grad).all() and w.grad.abs().max() > 0
    # a backward without an unroll forward on the workspace: DNLS_E_STATE
    solver.forward(t["poses0"], t["meas"], t["prior_meas"], t["w_edge"], t["w_prior"], implicit=True)
    with pytest.raises(DnlsError) as ei:
        solver.backward(P, t["meas"], t["prior_meas"], t["w_edge"], t["w_prior"], torch.zeros_like(P),
                        mode="unroll")
    assert ei.value.status == 5
    # LM is not supported in the unroll modes
    bad = PoseGraphSolver(D.SE3, topo.num_poses, topo.edges, topo.prior_vars, device=0, optimizer=D.LM)
    with pytest.raises(DnlsError) as ei:
        bad.forward(t["poses0"], t["meas"], t["prior_meas"], t["w_edge"], t["w_prior"], backward_mode=D.BWD_UNROLL)
    assert ei.value.status == 8
