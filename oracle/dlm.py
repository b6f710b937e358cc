"""Oracle DLM backward (direct loss minimisation, PAPER.md :259-271 and App. :897-934) --
TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

The paper's modified DLM (:267 / :928):
    theta_direct = argmin_theta S(theta; phi) + || eps theta - 1/2 v ||^2,
solved "by starting from theta* and using just one iteration of Gauss-Newton" (:934), and
    g_DLM = (1/eps) [ d/dphi S(theta*; phi) - d/dphi S(theta_direct; phi) ]       (:262, :902)
with v = grad_theta L(theta*).

Readings (B1-B3):
  B1  theta lives on SE(2)/SE(3): theta-hat is written in the chart at theta*,
      theta-hat = theta* [+] delta (right perturbation, the same chart as the GN step and as
      the tangent gradient v), so the regulariser is || eps delta - 1/2 v ||^2.
  B2  S carries the 1/2 of Eq. 1 (reading A6), the regulariser does not (as printed):
      S + ||eps delta - v/2||^2 = 1/2 ( sum ||r||^2 + || sqrt2 (eps delta - v/2) ||^2 ),
      i.e. an appended residual sqrt2 (eps delta - v/2) with Jacobian sqrt2 eps I.  One GN
      step from delta = 0 therefore solves
          (J^T J + 2 eps^2 I) delta_a = J^T r - eps v,     theta_direct = theta* [+] (-delta_a)
      (our GN sign convention, reading A5: H delta = J^T r, T <- T Exp(-delta)).
  B3  phi = the learnable weights: S = 1/2 sum ||w_e c_e||^2  =>  dS/dw_e = w_e ||c_e||^2
      (and the same for the prior weight), evaluated at theta* and at theta_direct.
"""
from __future__ import annotations

import numpy as np

from . import linalg, robust
from .nls import PGOProblem


def weight_partials(prob: PGOProblem, T):
    """dS/dw at fixed theta: w_e ||c_e(theta)||^2 per edge (x psi_e with a Welsch kernel, W1-W2),
    w_p ||c_p||^2 per prior (B3)."""
    c, _, _ = prob.edge_terms(T)
    ge = prob.irls_weights(c) * prob.w * np.einsum("ea,ea->e", c, c)
    gp = np.zeros(len(prob.prior_vars))
    if len(prob.prior_vars):
        cp, _ = prob.prior_terms(T)
        gp = prob.wp * np.einsum("pa,pa->p", cp, cp)
    return ge, gp


def dlm_weight_grads(prob: PGOProblem, T_star, v, eps: float):
    """DLM VJP at theta*.  Returns (grad_w_edge [E], grad_w_prior [P], theta_direct)."""
    v = np.asarray(v, dtype=np.float64).reshape(-1)
    _, H, b = prob.linearize(T_star)                      # J^T J and J^T r at theta*
    Ha = H + 2.0 * eps * eps * np.eye(H.shape[0])          # appended residual sqrt2 (eps delta - v/2)
    ga = b - eps * v
    L, ok = linalg.cholesky(Ha)
    if not ok:
        raise np.linalg.LinAlgError("augmented DLM system not SPD")
    delta = linalg.chol_solve(L, ga)
    T_dir = prob.retract(T_star, -delta)                  # one GN step from theta*
    ge0, gp0 = weight_partials(prob, T_star)
    ge1, gp1 = weight_partials(prob, T_dir)
    return (ge0 - ge1) / eps, (gp0 - gp1) / eps, T_dir


def dlm_radius_grad(prob: PGOProblem, T_star, T_dir, eps: float):
    """(1/eps) [dS/dk(theta*) - dS/dk(theta_direct)],  dS/dk = sum_e d rho_k(s_e)/dk  (W1)."""
    if prob.radius is None:
        return 0.0

    def part(T):
        c, _, _ = prob.edge_terms(T)
        return float(np.sum(robust.drho_dk(np.sum((prob.w[:, None] * c) ** 2, axis=1), prob.radius)))
    return (part(T_star) - part(T_dir)) / eps
