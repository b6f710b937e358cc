"""Pins P4/P7/P9/P10/P11 for the oracle GN/LM loop:
App. B curve fit, one-step exactness
on affine residuals, brute force vs scipy.optimize.least_squares with
residuals from scipy expm/logm (independent of oracle.lie), zero-noise invariants
(SPEC.md:639/655), SE2-embedded-in-SE3 equivalence, gauge (left-multiplication)
invariance."""
import math

import numpy as np
import pytest
from scipy.linalg import expm, logm
from scipy.optimize import least_squares

import synth
from oracle import lie, nls

rng = np.random.default_rng(99)


# ---------------------------------------------------------------- App. B curve fit
def appb_problem(x, y):
    x = np.asarray(x, dtype=float)
    y = np.asarray(y, dtype=float)
    return nls.EuclidProblem(1, 1, lambda v: y - v[0, 0] * np.exp(x), lambda v: -np.exp(x)[:, None])


def test_appb_first_gn_step_is_exact():
    prob = appb_problem([0.0, math.log(2.0)], [3.0, 6.0])
    S, H, b = prob.linearize(np.ones((1, 1)))
    assert S == 10.0 and H[0, 0] == 5.0 and b[0] == -10.0
    res = nls.gauss_newton(prob, np.ones((1, 1)), nls.Options(max_iterations=1))
    assert abs(res.x[0, 0] - 3.0) < 1e-15                            # SPEC.md:435 v0=1 -> v1=3
    assert res.objective < 1e-28
    res = nls.gauss_newton(prob, np.ones((1, 1)), nls.Options(max_iterations=1, step_size=0.5))
    assert abs(res.x[0, 0] - 2.0) < 1e-15                            # alpha = 0.5 -> v1 = 2


def test_appb_closed_form_and_lm_hand_step():
    xs = rng.standard_normal(20) * 0.5
    ys = 1.7 * np.exp(xs) + 0.01 * rng.standard_normal(20)
    res = nls.gauss_newton(appb_problem(xs, ys), np.ones((1, 1)), nls.Options(max_iterations=10))
    vstar = np.sum(ys * np.exp(xs)) / np.sum(np.exp(2 * xs))        # SPEC.md:461 closed form
    assert abs(res.x[0, 0] - vstar) < 1e-12
    # LM at v=1 with lambda=1: (5+5) delta = -10 -> v' = 2, S 10 -> 2.5, accept
    prob = appb_problem([0.0, math.log(2.0)], [3.0, 6.0])
    res = nls.levenberg_marquardt(prob, np.ones((1, 1)), nls.Options(optimizer="lm", max_iterations=1, lambda0=1.0))
    assert abs(res.x[0, 0] - 2.0) < 1e-15 and abs(res.objective - 2.5) < 1e-14
    assert abs(res.lam - 1.0 / 3.0) < 1e-16


def test_gn_one_step_exact_on_affine_residuals():
    for trial in range(100):
        m, n = 12, 5
        A = rng.standard_normal((m, n))
        bb = rng.standard_normal(m)
        prob = nls.EuclidProblem(n, 1, lambda x: A @ x[:, 0] - bb, lambda x: A)
        res = nls.gauss_newton(prob, rng.standard_normal((n, 1)), nls.Options(max_iterations=1))
        ref = np.linalg.lstsq(A, bb, rcond=None)[0]
        assert np.max(np.abs(res.x[:, 0] - ref)) <= 1e-12 * max(1.0, np.max(np.abs(ref)))


def test_lm_rejects_and_accepts_monotone():
    topo = synth.cube_topology(12, dim=3, p=0.4, seed=3)
    data = synth.cube_batch(topo, 1, seed=3, init_sigma_t=0.5, init_sigma_r=0.3)
    opt = nls.Options(optimizer="lm", max_iterations=15, lambda0=1e-4)
    res = nls.solve_batch("SE3", 12, topo.edges, topo.prior_vars, data["poses0"], data["meas"],
                          data["prior_meas"], data["w_edge"], data["w_prior"], opt)[0]
    h = res.history
    assert all(h[k + 1] <= h[k] * (1 + 1e-14) for k in range(len(h) - 1))   # accepted-S monotone (1 ulp: summation order)
    assert res.objective < h[0]


# ---------------------------------------------------------------- brute force on tiny graphs
def _vee_log(T, d):
    X = np.real(logm(T))
    if d == 6:
        return np.array([X[0, 3], X[1, 3], X[2, 3], X[2, 1], X[0, 2], X[1, 0]])
    return np.array([X[0, 2], X[1, 2], X[1, 0]])


def _hat(x, d):
    if d == 6:
        X = np.zeros((4, 4))
        X[:3, 3] = x[:3]
        X[:3, :3] = [[0, -x[5], x[4]], [x[5], 0, -x[3]], [-x[4], x[3], 0]]
        return X
    X = np.zeros((3, 3))
    X[:2, 2] = x[:2]
    X[0, 1], X[1, 0] = -x[2], x[2]
    return X


def brute_force(d, N, edges, prior_vars, Z, Zp, w, wp, Tref):
    """Independent solve: residuals from scipy logm/expm, scipy trust-region solver."""
    def fun(x):
        x = x.reshape(N, d)
        T = [Tref[k] @ expm(_hat(x[k], d)) for k in range(N)]
        out = []
        for e, (i, j) in enumerate(edges):
            out.append(w[e] * _vee_log(np.linalg.inv(Z[e]) @ np.linalg.inv(T[i]) @ T[j], d))
        for p, k in enumerate(prior_vars):
            out.append(wp[p] * _vee_log(np.linalg.inv(Zp[p]) @ T[k], d))
        return np.concatenate(out)
    sol = least_squares(fun, np.zeros(N * d), method="trf", xtol=1e-15, ftol=1e-15, gtol=1e-15, max_nfev=2000)
    sol = least_squares(fun, sol.x, method="lm", xtol=1e-15, ftol=1e-15, gtol=1e-15, max_nfev=4000)  # polish
    x = sol.x.reshape(N, d)
    return np.stack([Tref[k] @ expm(_hat(x[k], d)) for k in range(N)])


@pytest.mark.parametrize("G,edges", [
    (lie.SE3, [(0, 1)]),                       # 2 poses + prior
    (lie.SE3, [(0, 1), (1, 2), (0, 2)]),       # 3-cycle
    (lie.SE2, [(0, 1), (1, 2), (0, 2)]),
    (lie.SE2, [(0, 1), (1, 2), (2, 3), (0, 3), (1, 3)]),
])
def test_converged_gn_matches_brute_force(G, edges):
    rng = np.random.default_rng(len(edges) * 10 + G.d)
    d = G.d
    N = 1 + max(max(e) for e in edges)
    edges = np.array(edges)
    Tgt = G.exp(rng.standard_normal((N, d)))
    Z = G.inv(Tgt[edges[:, 0]]) @ Tgt[edges[:, 1]] @ G.exp(rng.standard_normal((len(edges), d)) * 0.1)
    Zp = Tgt[:1] @ G.exp(rng.standard_normal((1, d)) * 0.05)
    w = 0.5 + rng.random(len(edges))
    wp = np.array([1.3])
    T0 = Tgt @ G.exp(rng.standard_normal((N, d)) * 0.1)
    prob = nls.PGOProblem(G, N, edges, [0], Z, Zp, w, wp)
    res = nls.gauss_newton(prob, T0, nls.Options(max_iterations=30))
    Tb = brute_force(d, N, edges, [0], Z, Zp, w, wp, T0)
    # the independent solver stops on its own tolerances, so poses agree to ~1e-8; the objective
    # at both optima agrees to rounding, and GN's iterate is stationary for the independent
    # (logm/expm) residuals: central-difference gradient ~ 0
    np.testing.assert_allclose(res.x, Tb, atol=1e-8)
    assert abs(res.objective - prob.objective(Tb)) <= 1e-12 * max(1e-12, res.objective) + 1e-20

    def S_ind(x):
        x = x.reshape(N, d)
        T = [res.x[k] @ expm(_hat(x[k], d)) for k in range(N)]
        r = [w[e] * _vee_log(np.linalg.inv(Z[e]) @ np.linalg.inv(T[i]) @ T[j], d) for e, (i, j) in enumerate(edges)]
        r.append(wp[0] * _vee_log(np.linalg.inv(Zp[0]) @ T[0], d))
        r = np.concatenate(r)
        return 0.5 * float(r @ r)
    h = 1e-6
    grad = np.array([(S_ind(h * e) - S_ind(-h * e)) / (2 * h) for e in np.eye(N * d)])
    assert np.max(np.abs(grad)) <= 1e-8 * max(1.0, np.sqrt(res.objective))


# ---------------------------------------------------------------- invariants
@pytest.mark.parametrize("dim", [2, 3])
def test_zero_noise_cube(dim):
    topo = synth.cube_topology(27, dim=dim, p=0.3, seed=1)
    data = synth.cube_batch(topo, 1, seed=1, zero_noise=True)
    G = "SE3" if dim == 3 else "SE2"
    res = nls.solve_batch(G, 27, topo.edges, topo.prior_vars, data["poses0"], data["meas"],
                          data["prior_meas"], data["w_edge"], data["w_prior"], nls.Options(max_iterations=3))[0]
    assert res.history[0] < 1e-25 and res.objective < 1e-25
    np.testing.assert_allclose(lie.from_homog(res.x), data["poses0"][0], atol=1e-13)


def test_se2_embedded_in_se3_identical_iterates():
    topo = synth.cube_topology(16, dim=2, p=0.4, seed=5)
    data = synth.cube_batch(topo, 1, seed=5)

    def embed(P):   # [.., 2, 3] -> [.., 3, 4] rotation about z, z = 0
        out = np.zeros(P.shape[:-2] + (3, 4))
        out[..., :2, :2] = P[..., :2, :2]
        out[..., 2, 2] = 1.0
        out[..., :2, 3] = P[..., :2, 2]
        return out
    opt = nls.Options(max_iterations=6)
    r2 = nls.solve_batch("SE2", 16, topo.edges, topo.prior_vars, data["poses0"], data["meas"],
                         data["prior_meas"], data["w_edge"], data["w_prior"], opt)[0]
    r3 = nls.solve_batch("SE3", 16, topo.edges, topo.prior_vars, embed(data["poses0"]), embed(data["meas"]),
                         embed(data["prior_meas"]), data["w_edge"], data["w_prior"], opt)[0]
    np.testing.assert_allclose(np.array(r3.history), np.array(r2.history), rtol=1e-12, atol=1e-18)
    np.testing.assert_allclose(lie.from_homog(r3.x), embed(lie.from_homog(r2.x)), atol=1e-12)


def test_gauge_left_multiplication():
    topo = synth.cube_topology(20, dim=3, p=0.3, seed=2)
    data = synth.cube_batch(topo, 1, seed=2)
    Gt = lie.se3_exp(np.array([0.3, -1.0, 2.0, 0.4, -0.2, 0.9]))
    opt = nls.Options(max_iterations=5)
    r1 = nls.solve_batch("SE3", 20, topo.edges, topo.prior_vars, data["poses0"], data["meas"],
                         data["prior_meas"], data["w_edge"], data["w_prior"], opt)[0]
    P0 = lie.from_homog(Gt @ lie.to_homog(data["poses0"]))
    Pp = lie.from_homog(Gt @ lie.to_homog(data["prior_meas"]))
    r2 = nls.solve_batch("SE3", 20, topo.edges, topo.prior_vars, P0, data["meas"], Pp,
                         data["w_edge"], data["w_prior"], opt)[0]
    np.testing.assert_allclose(r2.history, r1.history, rtol=1e-10, atol=1e-16)
    np.testing.assert_allclose(r2.x, Gt @ r1.x, atol=1e-10)


def test_not_spd_flag_without_prior():
    # no prior -> gauge freedom -> H singular -> status 2 (not SPD) and the element is frozen
    topo = synth.cube_topology(8, dim=2, p=0.0, seed=0)
    data = synth.cube_batch(topo, 1)
    prob = nls.PGOProblem("SE2", 8, topo.edges, [], data["meas"][0], data["prior_meas"][0][:0],
                          data["w_edge"], [])
    res = nls.gauss_newton(prob, lie.to_homog(data["poses0"][0]), nls.Options(max_iterations=3))
    assert res.status == nls.ST_NOT_SPD and res.iterations == 0
