"""-m gpu tests of the C-ABI contract (include/dnls.h) and of the device Lie coefficient
functions (SURVEY.md §8(c) reading A7):
 * A7: dnls_linearize on 2-pose graphs whose edge residual sweeps the rotation angle over [1e-9, 3],
   including both sides of the series/closed-form switch points 0.5 and 1.0, against the oracle
   (c through S, H and b at 1e-12; the oracle's coefficients are pinned to mpmath in test_oracle_lie);
 * dnls_block_offsets: the oracle's per-cost H blocks read back at the exported offsets;
 * dnls_status_summary / DNLS_E_ALL_FAILED, the not-converged warning bit and the precedence of a failed
   final (implicit) factor;
 * the factor-cache registry: stage-level calls that overwrite a workspace's factor invalidate its
   implicit cache (DNLS_E_STATE), two workspaces of one graph keep their own cached factors."""
import numpy as np
import pytest
import torch

from gpu_helpers import DEV, TOL_GRAD, D, graph_for, make_case, oimp, olie, onls, oracle_problem, to_dev
from paper_2207_09442_b200._lib import DnlsError
from paper_2207_09442_b200.layer import PoseGraphSolver

pytestmark = pytest.mark.gpu

ANGLES = [1e-9, 1e-6, 1e-4, 1e-2, 0.1, 0.3, 0.5 - 1e-9, 0.5, 0.5 + 1e-9, 0.7, 1.0 - 1e-9, 1.0, 1.0 + 1e-9,
          1.5, 2.0, 2.5, 3.0]


def two_pose_problem(G, theta, rng):
    """T_0 = Z_prior (prior at its target), T_1 = Exp(xi) with |omega| = theta, Z_e = I: c_e = xi."""
    d = G.d
    if d == 6:
        axis = rng.standard_normal(3)
        axis /= np.linalg.norm(axis)
        xi = np.concatenate([rng.standard_normal(3), theta * axis])
    else:
        xi = np.array([rng.standard_normal(), rng.standard_normal(), theta])
    T0 = np.eye(G.m)
    T1 = G.exp(xi[None])[0]
    Z = np.eye(G.m)
    return xi, np.stack([T0, T1]), Z


@pytest.mark.parametrize("dim", [3, 2])
def test_a7_coefficient_sweep_linearize(dim):
    G = olie.SE3 if dim == 3 else olie.SE2
    rng = np.random.default_rng(11)
    edges = np.array([[0, 1]], dtype=np.int32)
    priors = np.array([0], dtype=np.int32)
    group = D.SE3 if dim == 3 else D.SE2
    g = D.dnls_graph_create(group, 2, edges, priors, 0)
    B = len(ANGLES)
    poses, meas, pmeas = [], [], []
    xis = []
    for th in ANGLES:
        xi, T, Z = two_pose_problem(G, th, rng)
        xis.append(xi)
        poses.append(olie.from_homog(T))
        meas.append(olie.from_homog(Z[None]))
        pmeas.append(olie.from_homog(T[:1]))
    data = {"poses0": np.stack(poses), "meas": np.stack(meas), "prior_meas": np.stack(pmeas),
            "w_edge": np.array([1.3]), "w_prior": np.array([0.7])}
    t = to_dev(data)
    ws = D.alloc_workspace(g, B)
    obj = torch.zeros(B, dtype=torch.float64, device=DEV)
    pr = D.make_problem(t["poses0"], t["meas"], t["prior_meas"], t["w_edge"], t["w_prior"], obj)
    D.dnls_linearize(g, B, pr, None, D.DAMP_MARQUARDT, ws)
    n = 2 * G.d
    Hd = torch.zeros(B, n, n, dtype=torch.float64, device=DEV)
    bd = torch.zeros(B, n, dtype=torch.float64, device=DEV)
    D.dnls_export_factor(g, B, ws, Hd)
    D.dnls_export_rhs(g, B, ws, bd)
    torch.cuda.synchronize()
    perm = D.dnls_graph_perm(g)
    idx = (perm[:, None] * G.d + np.arange(G.d)[None, :]).reshape(-1)
    for b, th in enumerate(ANGLES):
        prob = onls.PGOProblem(G, 2, edges, priors, data["meas"][b], data["prior_meas"][b], data["w_edge"],
                               data["w_prior"])
        S, H, bb = prob.linearize(olie.to_homog(data["poses0"][b]))
        c, _, _ = prob.edge_terms(olie.to_homog(data["poses0"][b]))
        # the oracle's residual is the generated xi (Log(Exp(xi)) roundtrip, pinned in test_oracle_lie)
        assert np.max(np.abs(c[0] - xis[b])) <= 1e-12 * max(1.0, np.max(np.abs(xis[b])))
        assert abs(obj[b].item() - S) <= 1e-12 * S, (th, obj[b].item(), S)
        Hp = np.tril(H[np.ix_(idx, idx)])
        Hg = Hd[b].cpu().numpy()
        assert np.max(np.abs(Hg - Hp)) <= 1e-12 * np.max(np.abs(Hp)), th
        assert np.max(np.abs(bd[b].cpu().numpy() - bb)) <= 1e-12 * np.max(np.abs(bb)), th


@pytest.mark.parametrize("dim", [3, 2])
def test_block_offsets_address_the_oracle_blocks(dim):
    topo, data = make_case(30, dim=dim, p=0.4, seed=21, B=2)
    g = graph_for(topo)
    ed, pd = D.dnls_block_offsets(g)
    assert ed.shape == (topo.num_edges, 7) and pd.shape == (1, 2)
    t = to_dev(data)
    ws = D.alloc_workspace(g, 2)
    pr = D.make_problem(t["poses0"], t["meas"], t["prior_meas"], t["w_edge"], t["w_prior"])
    D.dnls_linearize(g, 2, pr, None, D.DAMP_MARQUARDT, ws)
    torch.cuda.synchronize()
    storage = D.dnls_graph_stats(g)["storage_doubles"]
    raw = ws[: 2 * storage * 8].view(torch.float64).reshape(2, storage).cpu().numpy()
    d = g.d

    def block(b, off, ld):
        return np.stack([raw[b, off + q * ld: off + q * ld + d] for q in range(d)], axis=1)   # [row][col]

    for b in range(2):
        prob = oracle_problem(topo, data, b)
        _, H, _ = prob.linearize(olie.to_homog(data["poses0"][b]))
        scale = np.max(np.abs(H))
        for e, (i, j) in enumerate(topo.edges):
            o = ed[e]
            Hii, Hjj = H[i * d:(i + 1) * d, i * d:(i + 1) * d], H[j * d:(j + 1) * d, j * d:(j + 1) * d]
            assert np.max(np.abs(np.tril(block(b, o[0], o[1]) - Hii))) <= 1e-12 * scale
            assert np.max(np.abs(np.tril(block(b, o[2], o[3]) - Hjj))) <= 1e-12 * scale
            Hoff = H[j * d:(j + 1) * d, i * d:(i + 1) * d] if o[6] else H[i * d:(i + 1) * d, j * d:(j + 1) * d]
            assert np.max(np.abs(block(b, o[4], o[5]) - Hoff)) <= 1e-12 * scale
        p0 = topo.prior_vars[0]
        Hpp = H[p0 * d:(p0 + 1) * d, p0 * d:(p0 + 1) * d]
        assert np.max(np.abs(np.tril(block(b, pd[0, 0], pd[0, 1]) - Hpp))) <= 1e-12 * scale


def test_status_summary_all_failed_and_warning_bit():
    # no prior: H is gauge-singular, every element fails (GN freezes at iteration 0)
    topo, data = make_case(12, dim=3, p=0.3, seed=4, B=3)
    solver = PoseGraphSolver(D.SE3, topo.num_poses, topo.edges, np.zeros(0, np.int32), device=0, max_iterations=3)
    t = to_dev(data)
    wp = torch.zeros(0, dtype=torch.float64, device=DEV)
    pm = torch.zeros(0, 3, 4, dtype=torch.float64, device=DEV)
    _, _, st, _ = solver.forward(t["poses0"], t["meas"], pm, t["w_edge"], wp, implicit=True)
    with pytest.raises(DnlsError) as ei:
        D.dnls_status_summary(st)
    assert ei.value.status == 6
    assert all((v & D.ST_CODE_MASK) == D.ST_NOT_SPD for v in st.tolist())
    # K = 1 from a noisy start: the last step still changes S a lot -> warning bit, code OK;
    # K = 12: converged to rounding, no warning
    topo, data = make_case(20, dim=3, p=0.3, seed=6, B=2)
    t = to_dev(data)
    for K, warn in [(1, True), (12, False)]:
        solver = PoseGraphSolver(D.SE3, topo.num_poses, topo.edges, topo.prior_vars, device=0, max_iterations=K)
        _, _, st, _ = solver.forward(t["poses0"], t["meas"], t["prior_meas"], t["w_edge"], t["w_prior"],
                                     implicit=True)
        nf, nw = D.dnls_status_summary(st)
        assert nf == 0 and nw == (2 if warn else 0), (K, st.tolist())
        assert all((v & D.ST_CODE_MASK) == D.ST_OK for v in st.tolist())


def test_failed_final_factor_takes_precedence_and_zeroes_gradient():
    """An element that early-stops (CONVERGED) on a gauge-singular H must report NOT_SPD (its implicit
    factor is unusable) and contribute zero gradient."""
    topo, data = make_case(10, dim=3, p=0.3, seed=8, B=2)
    solver = PoseGraphSolver(D.SE3, topo.num_poses, topo.edges, topo.prior_vars, device=0, max_iterations=8,
                             optimizer=D.LM, early_stop=1)
    t = to_dev(data)
    wp = torch.tensor([1.0], dtype=torch.float64, device=DEV)
    P, _, st, _ = solver.forward(t["poses0"], t["meas"], t["prior_meas"], t["w_edge"], wp, implicit=True)
    v = torch.randn(2, topo.num_poses, 6, dtype=torch.float64, device=DEV)
    ge, gp = solver.backward(P, t["meas"], t["prior_meas"], t["w_edge"], wp, v, D.GRAD_TANGENT, per_element=True)
    torch.cuda.synchronize()
    assert all((s & D.ST_CODE_MASK) in (D.ST_OK, D.ST_CONVERGED) for s in st.tolist())
    # now a prior weight of 0 makes H singular at theta_K: the final factor fails for both elements
    wp0 = torch.zeros(1, dtype=torch.float64, device=DEV)
    P, _, st, _ = solver.forward(t["poses0"], t["meas"], t["prior_meas"], t["w_edge"], wp0, implicit=True)
    ge, gp = solver.backward(P, t["meas"], t["prior_meas"], t["w_edge"], wp0, v, D.GRAD_TANGENT, per_element=True)
    torch.cuda.synchronize()
    assert all((s & D.ST_CODE_MASK) == D.ST_NOT_SPD for s in st.tolist())
    assert torch.all(ge == 0) and torch.all(gp == 0)


def test_factor_cache_registry():
    topo, data = make_case(24, dim=3, p=0.3, seed=9, B=2)
    g = graph_for(topo)
    t = to_dev(data)
    opt = D.dnls_options_default(max_iterations=4, backward_mode=D.BWD_IMPLICIT)
    wsA, wsB = D.alloc_workspace(g, 2), D.alloc_workspace(g, 2)
    PA, PB = t["poses0"].clone(), t["poses0"].clone()
    prA = D.make_problem(PA, t["meas"], t["prior_meas"], t["w_edge"], t["w_prior"])
    prB = D.make_problem(PB, t["meas"], t["prior_meas"], t["w_edge"], t["w_prior"])
    D.dnls_forward(g, 2, opt, prA, wsA)
    D.dnls_forward(g, 2, opt, prB, wsB)
    v = torch.randn(2, topo.num_poses, 6, dtype=torch.float64, device=DEV)
    gA = torch.zeros(topo.num_edges, dtype=torch.float64, device=DEV)
    gB = torch.zeros_like(gA)
    gpA = torch.zeros(1, dtype=torch.float64, device=DEV)
    # both workspaces hold their own cached factor (the forward on B did not invalidate A)
    D.dnls_backward_implicit(g, 2, prA, v, D.GRAD_TANGENT, gA, gpA, 0, wsA)
    D.dnls_backward_implicit(g, 2, prB, v, D.GRAD_TANGENT, gB, gpA, 0, wsB)
    torch.cuda.synchronize()
    assert torch.equal(gA, gB)
    # a stage-level call that writes the factor storage invalidates that workspace only
    for stage in ("linearize", "factorize", "import"):
        D.dnls_forward(g, 2, opt, prA, wsA)
        if stage == "linearize":
            D.dnls_linearize(g, 2, prA, None, D.DAMP_MARQUARDT, wsA)
        elif stage == "factorize":
            D.dnls_factorize(g, 2, wsA)
        else:
            n = topo.num_poses * 6
            D.dnls_import_matrix(g, 2, torch.eye(n, dtype=torch.float64, device=DEV).expand(2, n, n).contiguous(), wsA)
        with pytest.raises(DnlsError) as ei:
            D.dnls_backward_implicit(g, 2, prA, v, D.GRAD_TANGENT, gA, gpA, 0, wsA)
        assert ei.value.status == 5, stage
        D.dnls_backward_implicit(g, 2, prB, v, D.GRAD_TANGENT, gB, gpA, 0, wsB)
    # batch mismatch
    D.dnls_forward(g, 2, opt, prA, wsA)
    with pytest.raises(DnlsError) as ei:
        D.dnls_backward_implicit(g, 1, prA, v, D.GRAD_TANGENT, gA, gpA, 0, wsA)
    assert ei.value.status == 5
