"""Pins for the oracle Welsch robust kernel (oracle/robust.py; SPEC.md:257-265;
DESIGN.md readings W1-W3), -m "not gpu":
 * SPEC.md:264 hand values (k = 1, s = 1: rho = (1 - e^-1)/2, kappa = sqrt(1 - e^-1)), the s -> 0
   limits, psi = 2 rho' and d rho/dk against central differences;
 * IRLS consistency: the assembled b equals the gradient of the robust objective in the chart
   (central differences), and the IRLS fixed point is a stationary point of S;
 * k -> inf recovers the plain quadratic solve;
 * the implicit VJP's D_phi g for the radius and the weights: Eq. 3 with the exact Hessian vs
   central differences of the converged solve over k and over w."""
import numpy as np
import pytest

import synth
from oracle import implicit, lie, nls, robust


def test_welsch_spec_values_and_limits():
    assert abs(robust.rho(1.0, 1.0) - 0.31606027941427883) < 1e-15
    # SPEC.md:264 prints kappa ~ 0.79520; the formula it states, sqrt(1 - e^-1), is 0.7950601 (the
    # printed digits are off by 1.4e-4) -- we pin the formula
    assert abs(robust.kappa(1.0, 1.0) - np.sqrt(1.0 - np.exp(-1.0))) < 1e-15
    assert abs(robust.kappa(1.0, 1.0) - 0.79520) < 2e-4
    assert robust.kappa(0.0, 2.0) == 1.0
    s0 = 1e-6   # Taylor s/2 - s^2/(4 k^2) + s^3/(12 k^4): expm1 keeps full relative precision
    assert abs(robust.rho(s0, 1.0) - (s0 / 2 - s0 * s0 / 4 + s0 ** 3 / 12)) <= 1e-16 * s0
    for s, k in [(0.3, 0.7), (2.0, 1.3), (1e-3, 0.1)]:
        h = 1e-6 * max(s, 1e-3)
        fd = (robust.rho(s + h, k) - robust.rho(s - h, k)) / (2 * h)
        assert abs(robust.psi(s, k) - 2 * fd) <= 1e-8 * max(1.0, robust.psi(s, k))
        hk = 1e-6 * k
        fdk = (robust.rho(s, k + hk) - robust.rho(s, k - hk)) / (2 * hk)
        assert abs(robust.drho_dk(s, k) - fdk) <= 1e-7 * max(1.0, abs(fdk))


def robust_problem(dim, N, seed, k, outliers=0.3, noise=0.1):
    topo = synth.cube_topology(N, dim=dim, p=0.6, seed=seed, outlier_ratio=outliers)
    data = synth.cube_batch(topo, 1, seed=seed, sigma_t=noise, sigma_r=noise / 2)
    G = lie.SE3 if dim == 3 else lie.SE2
    w = 0.8 + 0.4 * np.random.default_rng(seed).random(topo.num_edges)
    prob = nls.PGOProblem(G, N, topo.edges, topo.prior_vars, data["meas"][0], data["prior_meas"][0], w,
                          np.array([1.1]), radius=k)
    return prob, lie.to_homog(data["poses0"][0])


@pytest.mark.parametrize("dim", [2, 3])
def test_irls_b_is_robust_gradient(dim):
    prob, T = robust_problem(dim, 10, seed=4, k=0.3)
    _, _, b = prob.linearize(T)
    n = prob.n_vars * prob.d
    fd = np.zeros(n)
    h = 1e-6
    for i in range(n):
        e = np.zeros(n)
        e[i] = h
        fd[i] = (prob.objective(prob.retract(T, e)) - prob.objective(prob.retract(T, -e))) / (2 * h)
    # chart gradient at delta = 0 equals J^T r-style b (Jr(0) = I)
    assert np.max(np.abs(fd - b)) <= 1e-7 * max(1.0, np.max(np.abs(b)))


def test_irls_fixed_point_is_stationary_and_large_radius_is_quadratic():
    prob, T0 = robust_problem(3, 10, seed=9, k=0.5)
    res = nls.gauss_newton(prob, T0, nls.Options(max_iterations=60))
    _, _, b = prob.linearize(res.x)
    assert np.max(np.abs(b)) < 1e-10
    assert res.objective <= prob.objective(T0)
    plain = nls.PGOProblem(prob.G, prob.n_vars, prob.edges, prob.prior_vars, prob.Z, prob.Zp, prob.w, prob.wp)
    big = nls.PGOProblem(prob.G, prob.n_vars, prob.edges, prob.prior_vars, prob.Z, prob.Zp, prob.w, prob.wp,
                         radius=1e5)
    a = nls.gauss_newton(plain, T0, nls.Options(max_iterations=8)).x
    c = nls.gauss_newton(big, T0, nls.Options(max_iterations=8)).x
    assert np.max(np.abs(a - c)) < 1e-8


def test_radius_and_weight_vjp_vs_fd_of_converged_solve():
    k0 = 0.6
    prob, T0 = robust_problem(2, 8, seed=2, k=k0, noise=0.05)
    K = 80
    Ts = nls.gauss_newton(prob, T0, nls.Options(max_iterations=K)).x
    G = prob.G
    v = np.random.default_rng(1).standard_normal(prob.n_vars * prob.d)

    def chart(T):
        return G.log(G.inv(Ts) @ T).reshape(-1)

    def solve(radius=k0, w=None):
        p2 = nls.PGOProblem(G, prob.n_vars, prob.edges, prob.prior_vars, prob.Z, prob.Zp,
                            prob.w if w is None else w, prob.wp, radius=radius)
        return chart(nls.gauss_newton(p2, T0, nls.Options(max_iterations=K)).x)
    h = 1e-5
    fd_k = v @ (solve(k0 + h) - solve(k0 - h)) / (2 * h)
    ge, gp, lam = implicit.exact_ift_weight_grads(prob, Ts, v)
    gk = implicit.radius_vjp(prob, Ts, lam)
    assert abs(gk - fd_k) <= 1e-6 * max(1.0, abs(fd_k)), (gk, fd_k)
    for e in (0, 3):
        w2p, w2m = prob.w.copy(), prob.w.copy()
        w2p[e] += h
        w2m[e] -= h
        fd_w = v @ (solve(w=w2p) - solve(w=w2m)) / (2 * h)
        assert abs(ge[e] - fd_w) <= 1e-6 * max(1.0, abs(fd_w)), (e, ge[e], fd_w)
