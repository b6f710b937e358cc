"""Oracle implicit backward (Eq. 3 :243-246, Prop. 1 :250-257, proof :870-894).

Prop. 1 differentiates one Newton step h(theta; w) = theta - [H]^-1_stop g(theta; w) at
theta*, with g = grad_theta S = sum_e w_e^2 C_e^T c_e.  Hence, for an upstream gradient
v = dL/dtheta* (right-perturbation tangent coordinates),
    lambda = H^-1 v,         dL/dw_e = v^T D_{w_e} h = -2 w_e (C_e lambda_e) . c_e
(and the same for the prior weight), with H the Gauss-Newton Hessian J^T J at theta_K
(readings A11/A12: the factor the forward already holds).

``exact_ift_weight_grads`` is a PIN ONLY (tests): the same Eq. 3 with the exact Hessian
D_theta g obtained by central differences of the analytic chart gradient.
"""
from __future__ import annotations

import numpy as np

from . import linalg
from .nls import PGOProblem


def _weight_vjp(prob: PGOProblem, T, lam):
    """dL/dphi = -lambda^T D_phi g with g = grad S = sum_e psi_e w_e^2 C_e^T c_e + priors:
    dL/dw_e = -2 w_e psi_e (1 - s_e/k^2) (C_e lambda_e) . c_e   (psi = 1, k = inf without kernel),
    priors: -2 w_p (C_p lambda_p) . c_p (readings W1-W3; the radius: ``radius_vjp``)."""
    d = prob.d
    lam = np.asarray(lam).reshape(prob.n_vars, d)
    c, Ci, Cj = prob.edge_terms(T)
    e = prob.edges
    Cl = np.einsum("eab,eb->ea", Ci, lam[e[:, 0]]) + np.einsum("eab,eb->ea", Cj, lam[e[:, 1]])
    dot = np.einsum("ea,ea->e", Cl, c)
    if prob.radius is None:
        g_edge = -2.0 * prob.w * dot
    else:
        k = prob.radius
        s = np.sum((prob.w[:, None] * c) ** 2, axis=1)
        p = np.exp(-s / (k * k))
        g_edge = -2.0 * prob.w * p * (1.0 - s / (k * k)) * dot
    g_prior = np.zeros(len(prob.prior_vars))
    if len(prob.prior_vars):
        cp, Cp = prob.prior_terms(T)
        Clp = np.einsum("pab,pb->pa", Cp, lam[prob.prior_vars])
        g_prior = -2.0 * prob.wp * np.einsum("pa,pa->p", Clp, cp)
    return g_edge, g_prior


def radius_vjp(prob: PGOProblem, T, lam):
    """dL/dk = -lambda^T D_k g = -sum_e (2 s_e / k^3) psi_e w_e^2 (C_e lambda_e) . c_e  (W1-W3)."""
    if prob.radius is None:
        return 0.0
    lam = np.asarray(lam).reshape(prob.n_vars, prob.d)
    c, Ci, Cj = prob.edge_terms(T)
    e = prob.edges
    Cl = np.einsum("eab,eb->ea", Ci, lam[e[:, 0]]) + np.einsum("eab,eb->ea", Cj, lam[e[:, 1]])
    k = prob.radius
    s = np.sum((prob.w[:, None] * c) ** 2, axis=1)
    p = np.exp(-s / (k * k))
    return float(-np.sum(2.0 * s / k ** 3 * p * prob.w ** 2 * np.einsum("ea,ea->e", Cl, c)))


def implicit_weight_grads(prob: PGOProblem, T_K, v, L_K=None):
    """GN-implicit VJP at theta_K.  Returns (grad_w_edge [E], grad_w_prior [P], lambda [n]).

    L_K: optional cached Cholesky factor of H(theta_K) (factor reuse)."""
    if L_K is None:
        _, H, _ = prob.linearize(T_K)
        L_K, ok = linalg.cholesky(H)
        if not ok:
            raise np.linalg.LinAlgError("H(theta_K) not SPD")
    lam = linalg.chol_solve(L_K, np.asarray(v, dtype=np.float64).reshape(-1))
    ge, gp = _weight_vjp(prob, T_K, lam)
    return ge, gp, lam


def chart_gradient(prob: PGOProblem, T_star, x):
    """G(x) = grad_x S(T* [+] x) analytically: sum_m Jr(x_m)^T (J^T r)(T* [+] x)_m."""
    d = prob.d
    x = np.asarray(x).reshape(prob.n_vars, d)
    T = prob.retract(T_star, x)
    _, _, b = prob.linearize(T)
    Jr = prob.G.jr(x)
    return np.einsum("mba,mb->ma", Jr, b.reshape(prob.n_vars, d)).reshape(-1)


def exact_hessian(prob: PGOProblem, T_star, h: float = 1e-5):
    """D_x G at x = 0 by central differences of the analytic chart gradient (pin only)."""
    n = prob.n_vars * prob.d
    Hx = np.zeros((n, n))
    for k in range(n):
        e = np.zeros(n)
        e[k] = h
        Hx[:, k] = (chart_gradient(prob, T_star, e) - chart_gradient(prob, T_star, -e)) / (2 * h)
    return 0.5 * (Hx + Hx.T)


def exact_ift_weight_grads(prob: PGOProblem, T_star, v, h: float = 1e-5):
    """Eq. 3 with the exact Hessian (pin only): lambda = (D_theta g)^-1 v, same D_w g."""
    Hx = exact_hessian(prob, T_star, h)
    lam = np.linalg.solve(Hx, np.asarray(v, dtype=np.float64).reshape(-1))
    ge, gp = _weight_vjp(prob, T_star, lam)
    return ge, gp, lam


def tangent_from_matrix_grad(G, T, gT):
    """Euclidean gradient dL/dT on the top rows [.., r, r+1] -> right-tangent gradient:
    v_k = < dL/dT , T G_k >  with G_k the Lie-algebra generators (App. D projection)."""
    d = G.d
    T = np.asarray(T)
    r = T.shape[-1] - 1
    out = np.zeros(T.shape[:-2] + (d,))
    for k in range(d):
        e = np.zeros(d)
        e[k] = 1.0
        TG = T @ G.hat(e)
        out[..., k] = np.einsum("...ij,...ij->...", np.asarray(gT), TG[..., :r, :])
    return out
