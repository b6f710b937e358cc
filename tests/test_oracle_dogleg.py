"""Pins for the oracle Dogleg (oracle/nls.py:dogleg; SPEC.md:446-454,
:468; reading DL1), -m "not gpu":
 * SPEC.md:452 hand geometry: H = I, gradient (3, 4), Delta = 1 -> step (0.6, 0.8) subtracted,
   gain ratio 1 -> Delta doubles;
 * generous Delta on a quadratic: one step equals the GN step (converges like GN);
 * the interpolated dogleg step has norm Delta and lies on the segment Cauchy -> GN point;
 * step norm <= Delta + 1e-12 and accepted objectives non-increasing on noisy pose graphs
   (SPEC.md:468)."""
import numpy as np
import pytest

import synth
from oracle import lie, nls


def affine(A, c):
    A = np.asarray(A, dtype=np.float64)
    return nls.EuclidProblem(1, A.shape[1], lambda x: A @ x.reshape(-1) - c, lambda x: A)


def test_spec_hand_example_scaled_steepest_descent():
    c = np.zeros(2)
    prob = affine(np.eye(2), c)
    x0 = np.array([[3.0, 4.0]])
    res = nls.dogleg(prob, x0, nls.Options(optimizer="dogleg", max_iterations=1, delta0=1.0))
    assert np.allclose(res.x.reshape(-1), [3.0 - 0.6, 4.0 - 0.8], atol=1e-15)
    S, S_try, accept, rho, Delta, kind, ngn = res.trials[0]
    assert kind == "sd" and accept and abs(rho - 1.0) < 1e-14 and abs(ngn - 5.0) < 1e-14
    assert res.lam == 2.0   # Delta doubled (rho > 0.75)


def test_generous_radius_is_gauss_newton():
    rng = np.random.default_rng(0)
    A = rng.standard_normal((7, 4))
    c = rng.standard_normal(7)
    prob = affine(A, c)
    x0 = rng.standard_normal((1, 4))
    dl = nls.dogleg(prob, x0, nls.Options(optimizer="dogleg", max_iterations=1, delta0=1e6))
    gn = nls.gauss_newton(prob, x0, nls.Options(max_iterations=1))
    assert np.allclose(dl.x, gn.x, rtol=1e-12, atol=1e-12)
    xs = np.linalg.lstsq(A, c, rcond=None)[0]
    assert np.allclose(dl.x.reshape(-1), xs, atol=1e-10)


def test_dogleg_interpolation_hits_the_radius():
    A = np.array([[3.0, 0.0], [0.0, 0.3]])
    prob = affine(A, np.zeros(2))
    x0 = np.array([[1.0, 1.0]])
    S, H, b = prob.linearize(x0)
    d_gn = np.linalg.solve(H, b)
    d_c = (b @ b) / (b @ H @ b) * b
    Delta = 0.5 * (np.linalg.norm(d_c) + np.linalg.norm(d_gn))
    res = nls.dogleg(prob, x0, nls.Options(optimizer="dogleg", max_iterations=1, delta0=Delta))
    d = (x0 - res.x).reshape(-1)
    assert res.trials[0][5] == "dogleg"
    assert abs(np.linalg.norm(d) - Delta) < 1e-12
    # on the segment: d - d_c parallel to d_gn - d_c with parameter in [0, 1]
    u = d_gn - d_c
    tau = (d - d_c) @ u / (u @ u)
    assert 0.0 <= tau <= 1.0 and np.allclose(d_c + tau * u, d, atol=1e-14)


@pytest.mark.parametrize("dim,N,seed", [(2, 20, 1), (3, 16, 2)])
def test_step_norm_and_monotone_objective_on_pose_graphs(dim, N, seed):
    topo = synth.cube_topology(N, dim=dim, p=0.4, seed=seed)
    data = synth.cube_batch(topo, 1, seed=seed, init_sigma_t=0.5, init_sigma_r=0.3)
    G = lie.SE3 if dim == 3 else lie.SE2
    prob = nls.PGOProblem(G, N, topo.edges, topo.prior_vars, data["meas"][0], data["prior_meas"][0],
                          data["w_edge"], data["w_prior"])
    res = nls.dogleg(prob, lie.to_homog(data["poses0"][0]),
                     nls.Options(optimizer="dogleg", max_iterations=15, delta0=0.3))
    S_acc = [t[0] for t in res.trials if t[2]]
    assert all(a >= b for a, b in zip(S_acc, S_acc[1:]))
    assert res.objective <= res.trials[0][0]
    for (S, S_try, acc, rho, Delta, kind, ngn) in res.trials:
        assert kind in ("gn", "sd", "dogleg")
        if kind == "gn":
            assert ngn <= Delta + 1e-12
