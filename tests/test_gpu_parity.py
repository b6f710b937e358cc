"""-m gpu parity tests: the CUDA path (through the C-ABI) against the fp64 CPU oracle on the
same seeded inputs.  Tolerances from north_star: 1e-9 relative on solutions / objectives,
1e-6 relative on implicit gradients; factor entries vs chol(P H P^T) (Cholesky uniqueness,
SURVEY.md pin P6) at 1e-12."""
import numpy as np
import pytest
import torch

import synth

from gpu_helpers import (DEV, TOL_GRAD, TOL_OBJ, TOL_POSE, D, graph_for, make_case, oimp, olie, onls,
                         oracle_problem, oracle_results, perm_matrix_indices, pose_err, rel_vec_err, to_dev)
from paper_2207_09442_b200._lib import DnlsError
from paper_2207_09442_b200.layer import PoseGraphSolver, pose_graph_layer

pytestmark = pytest.mark.gpu


def run_forward(topo, data, implicit=False, w_edge=None, **opts):
    group = D.SE3 if topo.dim == 3 else D.SE2
    solver = PoseGraphSolver(group, topo.num_poses, topo.edges, topo.prior_vars, device=0, **opts)
    t = to_dev(data)
    we = t["w_edge"] if w_edge is None else w_edge
    poses, obj, st, it = solver.forward(t["poses0"], t["meas"], t["prior_meas"], we, t["w_prior"],
                                        implicit=implicit)
    torch.cuda.synchronize()
    return solver, t, poses, obj, st, it


# ------------------------------------------------------------------ factor / solve (minimum slice)
@pytest.mark.parametrize("N,dim,mode", [(16, 2, "local"), (64, 3, "local"), (48, 3, "random"), (200, 2, "random")])
def test_factor_matches_dense_cholesky(N, dim, mode):
    topo, data = make_case(N, dim=dim, p=0.3, mode=mode, seed=N, B=3)
    g = graph_for(topo)
    idx = perm_matrix_indices(g)
    Hs = []
    for b in range(3):
        prob = oracle_problem(topo, data, b)
        _, H, _ = prob.linearize(olie.to_homog(data["poses0"][b]))
        Hs.append(H)
    H = np.stack(Hs)
    n = H.shape[1]
    ws = D.alloc_workspace(g, 3)
    Hd = torch.from_numpy(H).to(DEV)
    D.dnls_import_matrix(g, 3, Hd, ws)
    st = torch.full((3,), -1, dtype=torch.int32, device=DEV)
    D.dnls_factorize(g, 3, ws, st)
    Ld = torch.zeros(3, n, n, dtype=torch.float64, device=DEV)
    D.dnls_export_factor(g, 3, ws, Ld)
    # solve with the factor
    rhs = np.random.default_rng(N).standard_normal((3, n))
    x = torch.zeros(3, n, dtype=torch.float64, device=DEV)
    D.dnls_solve_factored(g, 3, ws, torch.from_numpy(rhs).to(DEV), x)
    torch.cuda.synchronize()
    assert st.tolist() == [0, 0, 0]
    L = Ld.cpu().numpy()
    for b in range(3):
        Hp = H[b][np.ix_(idx, idx)]
        Lref = np.linalg.cholesky(Hp)
        err = np.max(np.abs(L[b] - Lref)) / np.max(np.abs(Lref))
        assert err <= 1e-12, err
        xr = np.linalg.solve(H[b], rhs[b])
        assert rel_vec_err(x[b].cpu().numpy(), xr) <= 1e-10


def test_factor_flags_not_spd_per_element():
    topo, data = make_case(20, dim=3, p=0.3, seed=5, B=2)
    g = graph_for(topo)
    prob = oracle_problem(topo, data, 0)
    _, H, _ = prob.linearize(olie.to_homog(data["poses0"][0]))
    Hbad = H.copy()
    Hbad[6, 6] = -1.0                                 # indefinite element 1
    ws = D.alloc_workspace(g, 2)
    D.dnls_import_matrix(g, 2, torch.from_numpy(np.stack([H, Hbad])).to(DEV), ws)
    st = torch.full((2,), -1, dtype=torch.int32, device=DEV)
    D.dnls_factorize(g, 2, ws, st)
    torch.cuda.synchronize()
    assert st.tolist() == [D.ST_OK, D.ST_NOT_SPD]


# ------------------------------------------------------------------ linearisation (a1 + a2)
@pytest.mark.parametrize("dim,noise", [(3, {}), (2, {}), (3, {"sigma_r": 0.8, "sigma_t": 1.0, "init_sigma_r": 0.7}),
                                       (2, {"sigma_r": 1.2, "init_sigma_r": 1.0})])
def test_linearize_matches_oracle(dim, noise):
    topo, data = make_case(40, dim=dim, p=0.4, seed=7, B=3, **noise)
    g = graph_for(topo)
    idx = perm_matrix_indices(g)
    t = to_dev(data)
    ws = D.alloc_workspace(g, 3)
    obj = torch.zeros(3, dtype=torch.float64, device=DEV)
    pr = D.make_problem(t["poses0"], t["meas"], t["prior_meas"], t["w_edge"], t["w_prior"], obj)
    D.dnls_linearize(g, 3, pr, None, D.DAMP_MARQUARDT, ws)
    n = topo.num_poses * g.d
    Hd = torch.zeros(3, n, n, dtype=torch.float64, device=DEV)
    bd = torch.zeros(3, n, dtype=torch.float64, device=DEV)
    D.dnls_export_factor(g, 3, ws, Hd)
    D.dnls_export_rhs(g, 3, ws, bd)
    torch.cuda.synchronize()
    for b in range(3):
        prob = oracle_problem(topo, data, b)
        S, H, bb = prob.linearize(olie.to_homog(data["poses0"][b]))
        Hp = np.tril(H[np.ix_(idx, idx)])
        Hg = Hd[b].cpu().numpy()
        pat = Hg != 0
        assert np.max(np.abs(Hg - Hp)) <= 1e-12 * np.max(np.abs(Hp))
        assert not np.any(Hp[~pat] != 0)
        assert rel_vec_err(bd[b].cpu().numpy(), bb) <= 1e-12
        assert abs(obj[b].item() - S) <= 1e-12 * S


def test_linearize_lm_damping():
    topo, data = make_case(30, dim=3, p=0.3, seed=8, B=2)
    g = graph_for(topo)
    idx = perm_matrix_indices(g)
    t = to_dev(data)
    ws = D.alloc_workspace(g, 2)
    lam = torch.tensor([0.5, 2.0], dtype=torch.float64, device=DEV)
    n = topo.num_poses * 6
    for damping, mode in [(D.DAMP_MARQUARDT, "marquardt"), (D.DAMP_IDENTITY, "identity")]:
        pr = D.make_problem(t["poses0"], t["meas"], t["prior_meas"], t["w_edge"], t["w_prior"])
        D.dnls_linearize(g, 2, pr, lam, damping, ws)
        Hd = torch.zeros(2, n, n, dtype=torch.float64, device=DEV)
        D.dnls_export_factor(g, 2, ws, Hd)
        torch.cuda.synchronize()
        for b in range(2):
            _, H, _ = oracle_problem(topo, data, b).linearize(olie.to_homog(data["poses0"][b]))
            Hl = onls.linalg.damp(H, lam[b].item(), mode)
            Hp = np.tril(Hl[np.ix_(idx, idx)])
            assert np.max(np.abs(Hd[b].cpu().numpy() - Hp)) <= 1e-12 * np.max(np.abs(Hp))


# ------------------------------------------------------------------ forward GN / LM
@pytest.mark.parametrize("N,dim,B,K,p,mode", [
    (16, 2, 4, 10, 0.2, "local"),       # BASELINE.json configs[0] (C1)
    (64, 3, 8, 10, 0.2, "local"),
    (40, 3, 5, 6, 0.3, "random"),
    (150, 2, 3, 8, 0.3, "random"),
])
def test_forward_gn_matches_oracle(N, dim, B, K, p, mode):
    topo, data = make_case(N, dim=dim, p=p, mode=mode, seed=N, B=B)
    _, _, poses, obj, st, it = run_forward(topo, data, max_iterations=K)
    res = oracle_results(topo, data, max_iterations=K)
    P = poses.cpu().numpy()
    for b, r in enumerate(res):
        assert pose_err(P[b], r.x) <= TOL_POSE
        assert abs(obj[b].item() - r.objective) <= TOL_OBJ * r.objective + 1e-20
        assert (st[b].item() & 0xff) == r.status and it[b].item() == r.iterations


def lm_has_tie(r, rel=1e-10):
    # DESIGN.md reading A13: an accept/reject decision whose trial objective equals the current one
    # to rounding can flip between two correct implementations; those runs are compared on the
    # converged iterate (objective 1e-9, poses 1e-7) instead of iterate-wise.
    return any(st is not None and abs(st - s) <= rel * s for s, st, _ in r.trials)


@pytest.mark.parametrize("K,seed", [(6, 3), (10, 3), (8, 4)])
def test_forward_lm_matches_oracle(K, seed):
    topo, data = make_case(32, dim=3, p=0.4, seed=seed, B=4, init_sigma_t=0.6, init_sigma_r=0.4)
    opts = dict(optimizer=D.LM, max_iterations=K, lambda0=1e-4)
    _, _, poses, obj, st, it = run_forward(topo, data, **opts)
    res = oracle_results(topo, data, optimizer="lm", max_iterations=K, lambda0=1e-4)
    P = poses.cpu().numpy()
    n_strict = 0
    for b, r in enumerate(res):
        assert abs(obj[b].item() - r.objective) <= TOL_OBJ * r.objective + 1e-20
        if lm_has_tie(r):
            assert pose_err(P[b], r.x) <= 1e-7
        else:
            n_strict += 1
            assert pose_err(P[b], r.x) <= TOL_POSE
            assert (st[b].item() & 0xff) == r.status and it[b].item() == r.iterations
    if K <= 6:
        assert n_strict == len(res)      # far from convergence no ties occur: strict iterate parity


def test_forward_step_size_and_early_stop():
    topo, data = make_case(24, dim=2, p=0.3, seed=4, B=3)
    opts = dict(max_iterations=12, step_size=0.5, early_stop=1, abs_tol=1e-12, rel_tol=1e-6)
    _, _, poses, obj, st, it = run_forward(topo, data, **opts)
    res = oracle_results(topo, data, max_iterations=12, step_size=0.5, early_stop=True, abs_tol=1e-12, rel_tol=1e-6)
    for b, r in enumerate(res):
        assert pose_err(poses[b].cpu().numpy(), r.x) <= TOL_POSE
        assert (st[b].item() & 0xff) == r.status and it[b].item() == r.iterations


def test_not_spd_without_prior_is_per_element_status():
    topo, data = make_case(10, dim=2, p=0.0, seed=1, B=2)
    # drop the prior: H singular (gauge freedom) -> status NOT_SPD, poses unchanged
    g = D.dnls_graph_create(D.SE2, 10, topo.edges, [], 0)
    t = to_dev(data)
    poses = t["poses0"].clone()
    st = torch.full((2,), -1, dtype=torch.int32, device=DEV)
    it = torch.full((2,), -1, dtype=torch.int32, device=DEV)
    obj = torch.zeros(2, dtype=torch.float64, device=DEV)
    ws = D.alloc_workspace(g, 2)
    pr = D.make_problem(poses, t["meas"], None, t["w_edge"], None, obj, st, it)
    D.dnls_forward(g, 2, D.dnls_options_default(max_iterations=3), pr, ws)
    torch.cuda.synchronize()
    assert st.tolist() == [D.ST_NOT_SPD] * 2 and it.tolist() == [0, 0]
    assert torch.equal(poses, t["poses0"])


def test_zero_noise_is_fixed_point():
    topo, data = make_case(27, dim=3, p=0.3, seed=2, B=2, zero_noise=True)
    _, t, poses, obj, st, it = run_forward(topo, data, max_iterations=3)
    assert obj.abs().max().item() < 1e-25
    assert torch.allclose(poses, t["poses0"], atol=1e-13, rtol=0)


def test_determinism_and_batch_permutation():
    topo, data = make_case(48, dim=3, p=0.3, seed=9, B=6)
    _, t, p1, o1, _, _ = run_forward(topo, data, max_iterations=5)
    _, _, p2, o2, _, _ = run_forward(topo, data, max_iterations=5)
    assert torch.equal(p1, p2) and torch.equal(o1, o2)          # bitwise reproducible
    perm = np.array([3, 0, 5, 1, 4, 2])
    dperm = {k: (v[perm] if k in ("poses0", "meas", "prior_meas") else v) for k, v in data.items()}
    _, _, p3, o3, _, _ = run_forward(topo, dperm, max_iterations=5)
    assert torch.equal(p3, p1[torch.from_numpy(perm).to(DEV)])
    assert torch.equal(o3, o1[torch.from_numpy(perm).to(DEV)])


def test_per_element_weights():
    topo, data = make_case(30, dim=3, p=0.3, seed=6, B=3)
    rng = np.random.default_rng(1)
    W = 0.5 + rng.random((3, topo.num_edges))
    d2 = dict(data)
    d2["w_edge"] = W
    _, t, poses, obj, _, _ = run_forward(topo, d2, max_iterations=6)
    res = oracle_results(topo, d2, max_iterations=6)
    for b, r in enumerate(res):
        assert pose_err(poses[b].cpu().numpy(), r.x) <= TOL_POSE


# ------------------------------------------------------------------ implicit backward
@pytest.mark.parametrize("dim,kind", [(3, D.GRAD_TANGENT), (3, D.GRAD_MATRIX), (2, D.GRAD_MATRIX)])
def test_implicit_backward_matches_oracle(dim, kind):
    N, B, K = 36, 4, 8
    topo, data = make_case(N, dim=dim, p=0.3, seed=11, B=B)
    solver, t, poses, obj, st, it = run_forward(topo, data, implicit=True, max_iterations=K)
    rng = np.random.default_rng(2)
    d = 6 if dim == 3 else 3
    res = oracle_results(topo, data, max_iterations=K, implicit=True)
    if kind == D.GRAD_TANGENT:
        v = rng.standard_normal((B, N, d))
        gpose = torch.from_numpy(v).to(DEV)
    else:
        gm = rng.standard_normal(poses.shape)
        gpose = torch.from_numpy(gm).to(DEV)
        v = np.stack([oimp.tangent_from_matrix_grad(solver_group(dim), r.x, gm[b]) for b, r in enumerate(res)])
    ge, gp = solver.backward(poses, t["meas"], t["prior_meas"], t["w_edge"], t["w_prior"], gpose, kind)
    gep, gpp = solver.backward(poses, t["meas"], t["prior_meas"], t["w_edge"], t["w_prior"], gpose, kind,
                               per_element=True)
    torch.cuda.synchronize()
    ge_ref = np.zeros(topo.num_edges)
    gp_ref = np.zeros(1)
    for b, r in enumerate(res):
        a, c, _ = oimp.implicit_weight_grads(oracle_problem(topo, data, b), r.x, v[b].reshape(-1), L_K=r.L_final)
        assert rel_vec_err(np.concatenate([gep[b].cpu().numpy(), gpp[b].cpu().numpy()]),
                           np.concatenate([a, c])) <= TOL_GRAD
        ge_ref += a
        gp_ref += c
    assert rel_vec_err(np.concatenate([ge.cpu().numpy(), gp.cpu().numpy()]),
                       np.concatenate([ge_ref, gp_ref])) <= TOL_GRAD


def solver_group(dim):
    return olie.SE3 if dim == 3 else olie.SE2


def test_backward_state_errors_and_layer():
    topo, data = make_case(20, dim=3, p=0.3, seed=12, B=2)
    g = graph_for(topo)
    t = to_dev(data)
    ws = D.alloc_workspace(g, 2)
    pr = D.make_problem(t["poses0"].clone(), t["meas"], t["prior_meas"], t["w_edge"], t["w_prior"])
    D.dnls_forward(g, 2, D.dnls_options_default(max_iterations=2), pr, ws)   # not implicit
    v = torch.zeros(2, 20, 6, dtype=torch.float64, device=DEV)
    ge = torch.zeros(topo.num_edges, dtype=torch.float64, device=DEV)
    with pytest.raises(Exception) as ei:
        D.dnls_backward_implicit(g, 2, pr, v, D.GRAD_TANGENT, ge, None, 0, ws)
    assert ei.value.status == 5
    # autograd layer: gradient flows to w_edge only; zero upstream -> zero gradient
    solver = PoseGraphSolver(D.SE3, 20, topo.edges, topo.prior_vars, device=0, max_iterations=4)
    w = t["w_edge"].clone().requires_grad_(True)
    poses, obj, st, it = pose_graph_layer(solver, t["poses0"], t["meas"], t["prior_meas"], w, t["w_prior"])
    (poses * 0.0).sum().backward()
    assert w.grad is not None and torch.count_nonzero(w.grad).item() == 0
    with pytest.raises(ValueError):
        pose_graph_layer(solver, t["poses0"].clone().requires_grad_(True), t["meas"], t["prior_meas"], w,
                         t["w_prior"])


def test_layer_gradient_matches_finite_difference_of_layer():
    # end-to-end: L = sum(gt_dist(poses*)) through the layer; implicit grad vs the oracle's GN-implicit
    topo, data = make_case(16, dim=2, p=0.4, seed=13, B=2)
    solver = PoseGraphSolver(D.SE2, 16, topo.edges, topo.prior_vars, device=0, max_iterations=10)
    t = to_dev(data)
    w = t["w_edge"].clone().requires_grad_(True)
    poses, *_ = pose_graph_layer(solver, t["poses0"], t["meas"], t["prior_meas"], w, t["w_prior"])
    gt = torch.from_numpy(np.broadcast_to(data["gt"], poses.shape).copy()).to(DEV)
    loss = ((poses - gt) ** 2).sum()
    loss.backward()
    res = oracle_results(topo, data, max_iterations=10, implicit=True)
    ref = np.zeros(topo.num_edges)
    for b, r in enumerate(res):
        gm = 2.0 * (olie.from_homog(r.x) - data["gt"])
        v = oimp.tangent_from_matrix_grad(olie.SE2, r.x, gm)
        a, _, _ = oimp.implicit_weight_grads(oracle_problem(topo, data, b), r.x, v.reshape(-1), L_K=r.L_final)
        ref += a
    assert rel_vec_err(w.grad.cpu().numpy(), ref) <= TOL_GRAD


# ------------------------------------------------------------------ edge cases
def test_batch_zero_and_one_and_chain():
    topo, data = make_case(12, dim=3, p=0.0, seed=3, B=1)       # pure odometry chain
    _, _, poses, obj, st, it = run_forward(topo, data, max_iterations=4)
    r = oracle_results(topo, data, max_iterations=4)[0]
    assert pose_err(poses[0].cpu().numpy(), r.x) <= TOL_POSE
    g = graph_for(topo)
    ws = D.alloc_workspace(g, 0)
    pr = D.make_problem(torch.zeros(0, 12, 3, 4, dtype=torch.float64, device=DEV), None, None, None, None)
    with pytest.raises(Exception):
        D.dnls_forward(g, 0, D.dnls_options_default(), pr, ws)    # meas NULL with E > 0 -> INVALID


def test_workspace_too_small():
    topo, data = make_case(12, dim=3, p=0.2, seed=3, B=2)
    g = graph_for(topo)
    t = to_dev(data)
    ws = D.alloc_workspace(g, 1)
    pr = D.make_problem(t["poses0"], t["meas"], t["prior_meas"], t["w_edge"], t["w_prior"])
    with pytest.raises(Exception) as ei:
        D.dnls_forward(g, 2, D.dnls_options_default(), pr, ws)
    assert ei.value.status == 4


@pytest.mark.parametrize("dim", [3, 2])
def test_forward_with_parallel_edges(dim):
    """Several edges between the same two poses (one reversed): their off-diagonal H block is a
    sum of contributions (the shared-block gather path of the linearisation), GN + implicit."""
    import dataclasses
    topo, data = make_case(40, dim=dim, p=0.3, mode="local", seed=7, B=3)
    pick = np.array([0, 3, 5, 10])
    extra = topo.edges[pick].copy()
    extra[1] = extra[1][::-1]            # reversed orientation: (j, i)
    topo2 = dataclasses.replace(topo, edges=np.concatenate([topo.edges, extra]).astype(np.int32),
                                outlier=np.concatenate([topo.outlier, np.zeros(len(pick), bool)]))
    data2 = dict(data)
    data2["meas"] = np.concatenate([data["meas"], data["meas"][:, pick]], axis=1)
    data2["w_edge"] = np.concatenate([data["w_edge"], 0.5 + 0.1 * np.arange(len(pick))])
    _, _, poses, obj, st, it = run_forward(topo2, data2, max_iterations=6)
    res = oracle_results(topo2, data2, max_iterations=6)
    P = poses.cpu().numpy()
    for b, r in enumerate(res):
        assert pose_err(P[b], r.x) <= TOL_POSE
        assert abs(obj[b].item() - r.objective) <= TOL_OBJ * r.objective + 1e-20


# ------------------------------------------------------------------ DLM backward
@pytest.mark.parametrize("dim,kind,eps", [(3, D.GRAD_TANGENT, 1e-3), (3, D.GRAD_MATRIX, 1e-2),
                                          (2, D.GRAD_TANGENT, 1e-4)])
def test_dlm_backward_matches_oracle(dim, kind, eps):
    """dnls_backward_dlm (one augmented GN step) vs oracle.dlm on the
    oracle's own theta_K, per element and batch-summed, 1e-6 relative."""
    from oracle import dlm as odlm
    N, B, K = 36, 4, 8
    topo, data = make_case(N, dim=dim, p=0.3, seed=11, B=B)
    solver, t, poses, obj, st, it = run_forward(topo, data, max_iterations=K)
    rng = np.random.default_rng(5)
    d = 6 if dim == 3 else 3
    res = oracle_results(topo, data, max_iterations=K)
    if kind == D.GRAD_TANGENT:
        v = rng.standard_normal((B, N, d))
        gpose = torch.from_numpy(v).to(DEV)
    else:
        gm = rng.standard_normal(poses.shape)
        gpose = torch.from_numpy(gm).to(DEV)
        v = np.stack([oimp.tangent_from_matrix_grad(solver_group(dim), r.x, gm[b]) for b, r in enumerate(res)])
    gep, gpp = solver.backward(poses, t["meas"], t["prior_meas"], t["w_edge"], t["w_prior"], gpose, kind,
                               per_element=True, mode="dlm", epsilon=eps)
    ge, gp = solver.backward(poses, t["meas"], t["prior_meas"], t["w_edge"], t["w_prior"], gpose, kind,
                             mode="dlm", epsilon=eps)
    torch.cuda.synchronize()
    ref = np.zeros(topo.num_edges + 1)
    for b, r in enumerate(res):
        a, c, _ = odlm.dlm_weight_grads(oracle_problem(topo, data, b), r.x, v[b].reshape(-1), eps)
        assert rel_vec_err(np.concatenate([gep[b].cpu().numpy(), gpp[b].cpu().numpy()]),
                           np.concatenate([a, c])) <= TOL_GRAD
        ref += np.concatenate([a, c])
    assert rel_vec_err(np.concatenate([ge.cpu().numpy(), gp.cpu().numpy()]), ref) <= TOL_GRAD


def test_dlm_invalidates_implicit_cache_and_layer_mode():
    topo, data = make_case(30, dim=3, p=0.3, seed=3, B=2)
    solver, t, poses, obj, st, it = run_forward(topo, data, implicit=True, max_iterations=6)
    v = torch.zeros(2, 30, 6, dtype=torch.float64, device=DEV)
    solver.backward(poses, t["meas"], t["prior_meas"], t["w_edge"], t["w_prior"], v, D.GRAD_TANGENT, mode="dlm")
    with pytest.raises(DnlsError):
        solver.backward(poses, t["meas"], t["prior_meas"], t["w_edge"], t["w_prior"], v, D.GRAD_TANGENT)
    with pytest.raises(Exception):
        solver.backward(poses, t["meas"], t["prior_meas"], t["w_edge"], t["w_prior"], v, D.GRAD_TANGENT,
                        mode="dlm", epsilon=0.0)
    # autograd layer in DLM mode: a gradient flows to the weights and matches the direct call
    w = t["w_edge"].clone().requires_grad_(True)
    from paper_2207_09442_b200.layer import pose_graph_layer
    out, *_ = pose_graph_layer(solver, t["poses0"], t["meas"], t["prior_meas"], w, t["w_prior"],
                               backward_mode="dlm", epsilon=1e-3)
    gm = torch.from_numpy(np.random.default_rng(0).standard_normal(out.shape)).to(DEV)
    (out * gm).sum().backward()
    ge, _ = solver.backward(out.detach(), t["meas"], t["prior_meas"], t["w_edge"], t["w_prior"], gm,
                            D.GRAD_MATRIX, mode="dlm", epsilon=1e-3)
    assert torch.allclose(w.grad, ge, rtol=0, atol=0)


# ------------------------------------------------------------------ Welsch robust kernel
def robust_case(dim, N=40, B=3, seed=21, radius=None):
    topo, data = make_case(N, dim=dim, p=0.4, seed=seed, B=B)
    topo = synth.cube_topology(N, dim=dim, p=0.4, seed=seed, outlier_ratio=0.3)
    data = synth.cube_batch(topo, B, seed=seed)
    data["radius"] = np.array([0.4]) if radius is None else np.asarray(radius, dtype=np.float64)
    return topo, data


@pytest.mark.parametrize("dim,opt,radius", [(3, "gn", None), (2, "gn", [0.3, 0.5, 0.8]), (3, "lm", None)])
def test_welsch_forward_matches_oracle(dim, opt, radius):
    topo, data = robust_case(dim, radius=radius)
    group = D.SE3 if dim == 3 else D.SE2
    solver = PoseGraphSolver(group, topo.num_poses, topo.edges, topo.prior_vars, device=0, max_iterations=8,
                             optimizer=(D.LM if opt == "lm" else D.GN))
    t = to_dev({k: v for k, v in data.items() if k != "gt"})
    poses, obj, st, it = solver.forward(t["poses0"], t["meas"], t["prior_meas"], t["w_edge"], t["w_prior"],
                                        radius=t["radius"])
    torch.cuda.synchronize()
    res = oracle_results(topo, data, max_iterations=8, optimizer=opt)
    P = poses.cpu().numpy()
    for b, r in enumerate(res):
        assert abs(obj[b].item() - r.objective) <= TOL_OBJ * r.objective + 1e-20
        if opt == "lm" and lm_has_tie(r):   # reading A13: compared on the converged iterate
            assert pose_err(P[b], r.x) <= 1e-7
        else:
            assert pose_err(P[b], r.x) <= TOL_POSE


@pytest.mark.parametrize("mode,per_el_radius", [("implicit", False), ("implicit", True), ("dlm", False)])
def test_welsch_backward_matches_oracle(mode, per_el_radius):
    """Weight and radius gradients (implicit: Prop. 1 with the IRLS Hessian; dlm) vs the oracle."""
    from oracle import dlm as odlm
    B, N, dim = 3, 36, 3
    topo, data = robust_case(dim, N=N, B=B, radius=[0.35, 0.5, 0.7] if per_el_radius else None)
    group = D.SE3
    solver = PoseGraphSolver(group, topo.num_poses, topo.edges, topo.prior_vars, device=0, max_iterations=8)
    t = to_dev({k: v for k, v in data.items() if k != "gt"})
    poses, obj, st, it = solver.forward(t["poses0"], t["meas"], t["prior_meas"], t["w_edge"], t["w_prior"],
                                        implicit=(mode == "implicit"), radius=t["radius"])
    v = np.random.default_rng(9).standard_normal((B, N, 6))
    ge, gp, gr = solver.backward(poses, t["meas"], t["prior_meas"], t["w_edge"], t["w_prior"],
                                 torch.from_numpy(v).to(DEV), D.GRAD_TANGENT, mode=mode, epsilon=1e-3,
                                 radius=t["radius"])
    torch.cuda.synchronize()
    res = oracle_results(topo, data, max_iterations=8, implicit=(mode == "implicit"))
    ref_w = np.zeros(topo.num_edges + 1)
    ref_r = np.zeros(B)
    for b, r in enumerate(res):
        prob = oracle_problem(topo, data, b)
        if mode == "implicit":
            a, c, lam = oimp.implicit_weight_grads(prob, r.x, v[b].reshape(-1), L_K=r.L_final)
            ref_r[b] = oimp.radius_vjp(prob, r.x, lam)
        else:
            a, c, Td = odlm.dlm_weight_grads(prob, r.x, v[b].reshape(-1), 1e-3)
            ref_r[b] = odlm.dlm_radius_grad(prob, r.x, Td, 1e-3)
        ref_w += np.concatenate([a, c])
    assert rel_vec_err(np.concatenate([ge.cpu().numpy(), gp.cpu().numpy()]), ref_w) <= TOL_GRAD
    g_r = gr.cpu().numpy().reshape(-1)
    if per_el_radius:
        assert rel_vec_err(g_r, ref_r) <= TOL_GRAD
    else:
        assert rel_vec_err(g_r, [ref_r.sum()]) <= TOL_GRAD


def test_welsch_layer_learnable_radius():
    topo, data = robust_case(3, N=30, B=2)
    solver = PoseGraphSolver(D.SE3, topo.num_poses, topo.edges, topo.prior_vars, device=0, max_iterations=6)
    t = to_dev({k: v for k, v in data.items() if k != "gt"})
    rad = t["radius"].clone().requires_grad_(True)
    out, *_ = pose_graph_layer(solver, t["poses0"], t["meas"], t["prior_meas"], t["w_edge"], t["w_prior"],
                               radius=rad)
    gt = torch.from_numpy(np.broadcast_to(data["gt"], out.shape).copy()).to(DEV)
    ((out - gt) ** 2).sum().backward()
    assert rad.grad is not None and rad.grad.shape == rad.shape and torch.isfinite(rad.grad).all()


# ------------------------------------------------------------------ cluster path (few large problems)
@pytest.mark.parametrize("cl", [2, 8])
@pytest.mark.parametrize("N,dim,opt,B", [(64, 3, "gn", 3), (40, 2, "lm", 3), (150, 3, "gn", 2), (30, 3, "gn", 1)])
def test_forward_cluster_matches_oracle(cl, N, dim, opt, B):
    """dnls_forward with a cluster of cl CTAs per element (global-memory factor, cluster barriers)
    vs the oracle; then the implicit backward on the factor the cluster left in the workspace."""
    topo, data = make_case(N, dim=dim, p=0.3, seed=N + cl, B=B)
    K = 8
    solver, t, poses, obj, st, it = run_forward(topo, data, implicit=True, max_iterations=K, cluster_ctas=cl,
                                                optimizer=(D.LM if opt == "lm" else D.GN))
    res = oracle_results(topo, data, max_iterations=K, optimizer=opt, implicit=True)
    P = poses.cpu().numpy()
    d = 6 if dim == 3 else 3
    v = np.random.default_rng(4).standard_normal((B, N, d))
    ge, gp = solver.backward(poses, t["meas"], t["prior_meas"], t["w_edge"], t["w_prior"],
                             torch.from_numpy(v).to(DEV), D.GRAD_TANGENT, per_element=True)
    torch.cuda.synchronize()
    for b, r in enumerate(res):
        assert abs(obj[b].item() - r.objective) <= TOL_OBJ * r.objective + 1e-20
        if opt == "lm" and lm_has_tie(r):   # reading A13: compared on the converged iterate
            assert pose_err(P[b], r.x) <= 1e-7
        else:
            assert pose_err(P[b], r.x) <= TOL_POSE
        assert (st[b].item() & 0xff) == r.status and it[b].item() == r.iterations
        a, c, _ = oimp.implicit_weight_grads(oracle_problem(topo, data, b), r.x, v[b].reshape(-1), L_K=r.L_final)
        assert rel_vec_err(np.concatenate([ge[b].cpu().numpy(), gp[b].cpu().numpy()]),
                           np.concatenate([a, c])) <= TOL_GRAD


def test_cluster_option_validation():
    topo, data = make_case(20, dim=3, B=1)
    with pytest.raises(DnlsError):
        run_forward(topo, data, max_iterations=2, cluster_ctas=3)


# ------------------------------------------------------------------ Dogleg
def dogleg_tie(r):
    """Decisions that can flip between two correct implementations (rounding, reading DL1 / the
    LM caveat A13): a gain ratio at a threshold, a GN point on the radius, or an actual decrease at
    rounding level (converged element: rho is then noise).  Such elements are compared on the
    converged iterate (1e-7) instead of the exact iterate."""
    for (S, S_try, acc, rho, Delta, kind, ngn) in r.trials:
        if min(abs(rho), abs(rho - 0.25), abs(rho - 0.75)) < 1e-7 or abs(ngn - Delta) <= 1e-9 * Delta:
            return True
        if S_try is not None and abs(S - S_try) <= 1e-10 * S:
            return True
    return False


@pytest.mark.parametrize("N,dim,B,delta0", [(40, 3, 4, 0.3), (30, 2, 4, 0.1), (64, 3, 3, 5.0)])
def test_forward_dogleg_matches_oracle(N, dim, B, delta0):
    noise = dict(init_sigma_t=0.4, init_sigma_r=0.2) if delta0 < 1.0 else {}   # far init: the radius binds
    topo, data = make_case(N, dim=dim, p=0.3, seed=N, B=B, **noise)
    K = 10 if delta0 < 1.0 else 3   # (GN-like steps converge to rounding level after ~4 iterations)
    solver, t, poses, obj, st, it = run_forward(topo, data, implicit=True, max_iterations=K, optimizer=D.DOGLEG,
                                                trust_radius0=delta0)
    res = oracle_results(topo, data, max_iterations=K, optimizer="dogleg", delta0=delta0, implicit=True)
    P = poses.cpu().numpy()
    d = 6 if dim == 3 else 3
    v = np.random.default_rng(8).standard_normal((B, N, d))
    ge, gp = solver.backward(poses, t["meas"], t["prior_meas"], t["w_edge"], t["w_prior"],
                             torch.from_numpy(v).to(DEV), D.GRAD_TANGENT, per_element=True)
    torch.cuda.synchronize()
    kinds = set()
    compared = 0
    for b, r in enumerate(res):
        kinds |= {tr[5] for tr in r.trials}
        if dogleg_tie(r):
            assert pose_err(P[b], r.x) <= 1e-7
            continue
        compared += 1
        assert pose_err(P[b], r.x) <= TOL_POSE
        assert abs(obj[b].item() - r.objective) <= TOL_OBJ * r.objective + 1e-20
        assert (st[b].item() & 0xff) == r.status and it[b].item() == r.iterations
        a, c, _ = oimp.implicit_weight_grads(oracle_problem(topo, data, b), r.x, v[b].reshape(-1), L_K=r.L_final)
        assert rel_vec_err(np.concatenate([ge[b].cpu().numpy(), gp[b].cpu().numpy()]),
                           np.concatenate([a, c])) <= TOL_GRAD
    assert compared >= 1
    if delta0 < 1.0:
        assert kinds & {"sd", "dogleg"}   # the trust region was active
