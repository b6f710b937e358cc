"""Oracle cost functions: the coordinate-independent relative-pose (Between) error of
App. E.1 and a Gaussian prior on a pose ("Gaussian
measurement"), with analytic Jacobians in the right-perturbation convention, and the
objective of Eq. 1: S = 1/2 sum_i || w_i c_i ||^2.

Between edge e = (i, j) with measurement Z:  E = Z^-1 T_i^-1 T_j,  c = Log(E),
  dc/d(delta_j) = Jr^-1(c),   dc/d(delta_i) = -Jr^-1(c) Ad(T_j^-1 T_i)
Prior on pose p with target Z_p:  c = Log(Z_p^-1 T_p),  dc/d(delta_p) = Jr^-1(c).
All functions are vectorised over the leading (edge) axis; T are homogeneous matrices.
"""
from __future__ import annotations

import numpy as np


def between(G, Ti, Tj, Z):
    """Returns (c [E,d], Ci [E,d,d], Cj [E,d,d]) -- UNWEIGHTED cost and Jacobians."""
    Ti, Tj, Z = np.asarray(Ti), np.asarray(Tj), np.asarray(Z)
    E = G.inv(Z) @ G.inv(Ti) @ Tj
    c = G.log(E)
    A = G.jr_inv(c)
    Cj = A
    Ci = -A @ G.adjoint(G.inv(Tj) @ Ti)
    return c, Ci, Cj


def prior(G, T, Z):
    """Returns (c [P,d], C [P,d,d]) -- UNWEIGHTED prior cost and Jacobian."""
    c = G.log(G.inv(np.asarray(Z)) @ np.asarray(T))
    return c, G.jr_inv(c)


def objective(G, T, edges, Z, w_edge, prior_vars, Zp, w_prior):
    """S(theta) = 1/2 sum_e ||w_e c_e||^2 + 1/2 sum_p ||w_p c_p||^2   (Eq. 1, with the 1/2)."""
    edges = np.asarray(edges)
    c, _, _ = between(G, T[edges[:, 0]], T[edges[:, 1]], Z)
    S = 0.5 * np.sum((np.asarray(w_edge)[:, None] * c) ** 2)
    if len(prior_vars):
        cp, _ = prior(G, T[np.asarray(prior_vars)], Zp)
        S += 0.5 * np.sum((np.asarray(w_prior)[:, None] * cp) ** 2)
    return float(S)
