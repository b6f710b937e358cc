"""Pin P8 for the oracle implicit backward (Eq. 3 :243-246,
Prop. 1 :250-257 / :870-894):
 (ii) Eq. 3 with the exact Hessian vs central finite differences over the weights of
      the converged solve (h = 1e-5), <= 1e-7 relative;
 (iii) GN-implicit (the factor the forward holds, reading A12) vs exact-IFT: the gap
      shrinks proportionally to the measurement noise;
 zero upstream gradient -> zero weight gradients; the Euclidean-gradient
 -> tangent projection (App. D) vs finite differences."""
import numpy as np
import pytest

import synth
from oracle import implicit, lie, nls

rng = np.random.default_rng(2024)


def make_problem(dim, N, p, seed, sigma):
    topo = synth.cube_topology(N, dim=dim, p=p, seed=seed)
    data = synth.cube_batch(topo, 1, seed=seed, sigma_t=sigma, sigma_r=sigma / 2,
                            init_sigma_t=0.05, init_sigma_r=0.02)
    G = lie.SE3 if dim == 3 else lie.SE2
    w = 0.8 + 0.4 * rng.random(topo.num_edges)
    prob = nls.PGOProblem(G, N, topo.edges, topo.prior_vars, data["meas"][0], data["prior_meas"][0],
                          w, np.array([1.1]))
    return prob, lie.to_homog(data["poses0"][0])


def converged(prob, T0, K=40):
    return nls.gauss_newton(prob, T0, nls.Options(max_iterations=K)).x


def fd_weight_grads(prob, T0, Tstar, v, h=1e-5):
    """v^T d theta*/d w by central differences of the converged solve, in the chart at theta*."""
    G = prob.G

    def chart(T):
        return G.log(G.inv(Tstar) @ T).reshape(-1)
    ge = np.zeros(len(prob.w))
    for e in range(len(prob.w)):
        out = []
        for s in (+1, -1):
            w2 = prob.w.copy()
            w2[e] += s * h
            p2 = nls.PGOProblem(G, prob.n_vars, prob.edges, prob.prior_vars, prob.Z, prob.Zp, w2, prob.wp)
            out.append(chart(converged(p2, T0)))
        ge[e] = v @ (out[0] - out[1]) / (2 * h)
    gp = np.zeros(len(prob.wp))
    for k in range(len(prob.wp)):
        out = []
        for s in (+1, -1):
            wp2 = prob.wp.copy()
            wp2[k] += s * h
            p2 = nls.PGOProblem(G, prob.n_vars, prob.edges, prob.prior_vars, prob.Z, prob.Zp, prob.w, wp2)
            out.append(chart(converged(p2, T0)))
        gp[k] = v @ (out[0] - out[1]) / (2 * h)
    return ge, gp


@pytest.mark.parametrize("dim,N", [(2, 8), (3, 6)])
def test_exact_ift_matches_fd_of_converged_solve(dim, N):
    prob, T0 = make_problem(dim, N, 0.5, seed=11 + dim, sigma=0.1)
    Ts = converged(prob, T0)
    v = rng.standard_normal(N * prob.d)
    ge, gp, _ = implicit.exact_ift_weight_grads(prob, Ts, v)
    fe, fp = fd_weight_grads(prob, T0, Ts, v)
    g = np.concatenate([ge, gp])
    f = np.concatenate([fe, fp])
    assert np.max(np.abs(g - f)) <= 1e-7 * np.max(np.abs(f))


@pytest.mark.parametrize("dim,N", [(2, 8), (3, 6)])
def test_gn_implicit_gap_shrinks_with_noise(dim, N):
    gaps = []
    for sigma in (0.1, 0.01):
        prob, T0 = make_problem(dim, N, 0.5, seed=21 + dim, sigma=sigma)
        Ts = converged(prob, T0)
        v = np.random.default_rng(5).standard_normal(N * prob.d)
        ge, gp, _ = implicit.implicit_weight_grads(prob, Ts, v)
        xe, xp, _ = implicit.exact_ift_weight_grads(prob, Ts, v)
        g, x = np.concatenate([ge, gp]), np.concatenate([xe, xp])
        gaps.append(np.max(np.abs(g - x)) / np.max(np.abs(x)))
    assert gaps[1] < gaps[0] / 4.0, gaps
    assert gaps[0] < 0.1


def test_zero_upstream_gradient_gives_zero():
    prob, T0 = make_problem(3, 6, 0.5, seed=3, sigma=0.1)
    Ts = converged(prob, T0, K=5)
    ge, gp, lam = implicit.implicit_weight_grads(prob, Ts, np.zeros(6 * 6))
    assert not ge.any() and not gp.any() and not lam.any()


def test_gn_implicit_uses_cached_factor_identically():
    prob, T0 = make_problem(3, 6, 0.5, seed=4, sigma=0.1)
    res = nls.gauss_newton(prob, T0, nls.Options(max_iterations=5, implicit=True))
    v = rng.standard_normal(36)
    a = implicit.implicit_weight_grads(prob, res.x, v, L_K=res.L_final)
    b = implicit.implicit_weight_grads(prob, res.x, v)
    for x, y in zip(a, b):
        np.testing.assert_array_equal(x, y)


@pytest.mark.parametrize("G", [lie.SE3, lie.SE2])
def test_tangent_projection_matches_fd(G):
    # L(T) = sum(M * T_top) for a random M; v_k = dL(T Exp(h e_k))/dh
    T = G.exp(rng.standard_normal((4, G.d)))
    M = rng.standard_normal(T[..., :-1, :].shape)
    v = implicit.tangent_from_matrix_grad(G, T, M)
    h = 1e-6
    for k in range(G.d):
        e = np.zeros(G.d)
        e[k] = h
        Lp = np.einsum("nij,nij->n", M, (T @ G.exp(e))[..., :-1, :])
        Lm = np.einsum("nij,nij->n", M, (T @ G.exp(-e))[..., :-1, :])
        np.testing.assert_allclose(v[:, k], (Lp - Lm) / (2 * h), atol=1e-8)
