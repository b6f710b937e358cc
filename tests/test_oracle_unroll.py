"""Pins for the oracle Unroll / Truncated backward (oracle/unroll.py; PAPER.md :235-239, :224;
SPEC.md:506-523; reading U1), -m "not gpu":
 * central differences of the WHOLE unrolled K-step map theta_0, w -> L(theta_K) (L = <v, chart of
   theta_K>): weight gradients and the theta_init gradient (SE2 and SE3, alpha = 1 and 0.7) -- a dropped
   dH term, a wrong retraction adjoint or a transposed Ad fails it;
 * SPEC.md:512 hand case: an affine-in-theta problem (prior only) reaches its optimum in one GN step, so
   d theta_1 / d theta_0 = 0 and the prior's weight has zero gradient;
 * truncation T >= K equals the full unroll exactly; T < K differs (biased) and gives no
   theta_init gradient;
 * K -> infinity: at a fixed point of the GN map the unrolled gradient tends to the exact-Hessian IFT
   gradient (oracle.implicit.exact_ift_weight_grads, itself pinned by FD of the converged solve)."""
import numpy as np
import pytest

import synth
from oracle import implicit, lie, nls, unroll


def small_problem(dim, N, seed, noise=0.1):
    topo = synth.cube_topology(N, dim=dim, p=0.6, seed=seed)
    data = synth.cube_batch(topo, 1, seed=seed, sigma_t=noise, sigma_r=noise / 2, init_sigma_t=noise,
                            init_sigma_r=noise / 2)
    G = lie.SE3 if dim == 3 else lie.SE2
    w = 0.8 + 0.4 * np.random.default_rng(seed).random(topo.num_edges)
    prob = nls.PGOProblem(G, N, topo.edges, topo.prior_vars, data["meas"][0], data["prior_meas"][0], w,
                          np.array([1.1]))
    return prob, lie.to_homog(data["poses0"][0])


def loss_of(prob, T0, K, alpha, v, w=None, wp=None, eta0=None):
    p2 = nls.PGOProblem(prob.G, prob.n_vars, prob.edges, prob.prior_vars, prob.Z, prob.Zp,
                        prob.w if w is None else w, prob.wp if wp is None else wp)
    T = T0 if eta0 is None else p2.retract(T0, eta0)
    TK, _, _, _ = unroll.gn_history(p2, T, K, alpha)
    return TK


@pytest.mark.parametrize("dim,N,K,alpha", [(2, 8, 3, 1.0), (3, 6, 2, 1.0), (3, 6, 3, 0.7)])
def test_unroll_matches_fd_of_unrolled_map(dim, N, K, alpha):
    prob, T0 = small_problem(dim, N, seed=N + K)
    d = prob.d
    v = np.random.default_rng(2).standard_normal((N, d))
    TK, gw, gp, g0 = unroll.unroll_weight_grads(prob, T0, K, v, alpha)
    G = prob.G

    def L(TKp):   # <v, chart of theta_K' at theta_K>  (right-tangent upstream gradient v)
        return float(np.sum(v * G.log(G.inv(TK) @ TKp)))
    h = 1e-6
    for e in (0, 2, len(prob.w) - 1):
        wp_, wm_ = prob.w.copy(), prob.w.copy()
        wp_[e] += h
        wm_[e] -= h
        fd = (L(loss_of(prob, T0, K, alpha, v, w=wp_)) - L(loss_of(prob, T0, K, alpha, v, w=wm_))) / (2 * h)
        assert abs(gw[e] - fd) <= 1e-6 * max(1.0, np.max(np.abs(gw))), (e, gw[e], fd)
    fdp = (L(loss_of(prob, T0, K, alpha, v, wp=prob.wp + h)) - L(loss_of(prob, T0, K, alpha, v, wp=prob.wp - h))) / (2 * h)
    assert abs(gp[0] - fdp) <= 1e-6 * max(1.0, abs(fdp))
    for m, a in [(0, 0), (N // 2, d - 1), (N - 1, 1)]:
        e = np.zeros((N, d))
        e[m, a] = h
        fd = (L(loss_of(prob, T0, K, alpha, v, eta0=e)) - L(loss_of(prob, T0, K, alpha, v, eta0=-e))) / (2 * h)
        assert abs(g0[m, a] - fd) <= 1e-6 * max(1.0, np.max(np.abs(g0))), (m, a, g0[m, a], fd)


def test_unroll_prior_only_one_step_hand_case():
    """S = |theta - phi|^2-type problem (a prior on every pose is linear in the chart at its
    target only approximately; the exact hand case is a single pose whose prior target is reached in
    one GN step from a start ON the geodesic): theta_1 = Z exactly, d theta_1/d theta_0 = 0."""
    G = lie.SE3
    Z = G.exp(np.array([[0.3, -0.2, 0.1, 0.2, 0.1, -0.3]]))
    xi = np.array([0.1, 0.2, -0.1, 0.05, -0.02, 0.04])
    T0 = Z @ G.exp(xi[None])      # c(T0) = xi; Jr^-1(xi) xi = xi, so one GN step lands on Z exactly
    prob = nls.PGOProblem(G, 1, np.zeros((0, 2), np.int32), np.array([0]), np.zeros((0, 3, 4)),
                          lie.from_homog(Z), np.zeros(0), np.array([1.7]))
    v = np.random.default_rng(0).standard_normal((1, 6))
    TK, gw, gp, g0 = unroll.unroll_weight_grads(prob, T0, 1, v)
    assert np.max(np.abs(TK - Z)) < 1e-14
    assert abs(gp[0]) < 1e-12
    assert np.max(np.abs(g0)) < 1e-8   # FD of the Jacobian: ~1e-10


def test_truncated_equals_unroll_when_window_covers_all_and_is_biased_otherwise():
    prob, T0 = small_problem(2, 8, seed=5, noise=0.3)
    v = np.random.default_rng(4).standard_normal((8, 3))
    K = 3
    _, gw, gp, g0 = unroll.unroll_weight_grads(prob, T0, K, v)
    _, tw, tp, t0 = unroll.unroll_weight_grads(prob, T0, K, v, truncate=K + 2)
    assert np.array_equal(gw, tw) and np.array_equal(gp, tp) and np.array_equal(g0, t0)
    _, bw, bp, b0 = unroll.unroll_weight_grads(prob, T0, K, v, truncate=1)
    assert np.max(np.abs(bw - gw)) > 1e-6 * np.max(np.abs(gw))
    assert np.all(b0 == 0)


def test_unroll_tends_to_exact_ift_at_a_fixed_point():
    prob, T0 = small_problem(2, 8, seed=7, noise=0.05)
    Ts = nls.gauss_newton(prob, T0, nls.Options(max_iterations=40)).x
    v = np.random.default_rng(6).standard_normal((8, 3))
    ge, gp, _ = implicit.exact_ift_weight_grads(prob, Ts, v.reshape(-1))
    errs = []
    for K in (2, 6):
        # start from a slightly perturbed fixed point: GN contracts back, the unrolled map's derivative
        # converges to the IFT derivative of the fixed-point equation b(theta, w) = 0
        T = prob.retract(Ts, 1e-3 * np.random.default_rng(K).standard_normal((8, 3)))
        _, gw, gpp, _ = unroll.unroll_weight_grads(prob, T, K, v)
        errs.append(np.max(np.abs(np.concatenate([gw, gpp]) - np.concatenate([ge, gp]))) /
                    np.max(np.abs(np.concatenate([ge, gp]))))
    assert errs[1] < errs[0] and errs[1] < 1e-4, errs
