"""Oracle Unroll / Truncated backward (§4.3 :235-239 "backpropagation through time or
unrolled optimization", "truncated backpropagation through time"; the linear-solve gradients of
:224) -- TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

The forward is K plain Gauss-Newton steps (reading A5):
    H_k = J_k^T J_k,  b_k = J_k^T r_k,  delta_k = H_k^-1 b_k,  theta_{k+1} = theta_k Exp(-alpha delta_k)
with J_k, r_k the weighted Jacobian / residual at theta_k (J_e = w_e C_e, r_e = w_e c_e).  The
backward is the exact reverse-mode chain rule through these steps, in reverse order, for an upstream
gradient v_K = dL/dtheta_K in right-tangent coordinates:

  retraction (per pose m, right perturbations; Exp(eta) X = X Exp(Ad_{X^-1} eta)):
      theta_k [+] eta, delta + d delta  ->  theta_{k+1} [+] ( Ad_{Exp(alpha delta_m)} eta_m - alpha Jr(-alpha delta_m) d delta_m )
      so  u_m = -alpha Jr(-alpha delta_m)^T v_m   (= dL/d delta_m)   and the direct part Ad_{Exp(alpha delta_m)}^T v_m;
  linear solve (df/db = A^-1 df/dy, df/dA = -A^-1 df/dy y^T):
      lambda = H_k^-1 u,   dL = lambda^T db - lambda^T dH delta;
  per cost term (edge or prior) with C, c unweighted at theta_k, p = c - C delta, q = C lambda:
      dL/dw_e   += 2 w_e (q . c - q . C delta)
      dL/deta   += w_e^2 [ C^T q + grad_eta( (C(theta [+] eta) lambda_e) . p - (C(theta [+] eta) delta_e) . q ) ]
  and v_k = Ad^T v_{k+1} + dL/deta.

The only approximation (reading U1): grad_eta of the two contractions of the Jacobian C with
FIXED vectors is taken by central differences of the analytic Jacobian in the chart (step h = 1e-5:
truncation ~h^2 |C'''| and rounding ~eps/h, both ~1e-10 relative), i.e. the second derivative of the
residual is never formed.  Truncated mode (T < K) runs the same reverse loop over the last T steps
only; the iterate entering the window is a constant, so dL/dtheta_0 = 0.  Pinned in
tests/test_oracle_unroll.py against central differences of the whole K-step map.
"""
from __future__ import annotations

import numpy as np

from . import costs, linalg
from .nls import PGOProblem

FD_STEP = 1e-5


def gn_history(prob: PGOProblem, T0, K: int, alpha: float = 1.0):
    """K Gauss-Newton steps; returns (theta_K, [theta_k], [delta_k], [L_k]) -- the per-iteration
    factors are what the unrolled backward solves with ("necessary ... for unrolling")."""
    T = np.array(T0, dtype=np.float64, copy=True)
    Ts, ds, Ls = [], [], []
    for _ in range(K):
        _, H, b = prob.linearize(T)
        L, ok = linalg.cholesky(H)
        if not ok:
            raise np.linalg.LinAlgError("H_k not SPD")
        delta = linalg.chol_solve(L, b)
        Ts.append(T)
        ds.append(delta)
        Ls.append(L)
        T = prob.retract(T, -alpha * delta)
    return T, Ts, ds, Ls


def _jac_at(prob: PGOProblem, kind, k, poses):
    """Unweighted Jacobian blocks of cost term (kind, k) evaluated at the given pose(s)."""
    if kind == "edge":
        _, Ci, Cj = costs.between(prob.G, poses[0][None], poses[1][None], prob.Z[k][None])
        return [Ci[0], Cj[0]]
    _, Cp = costs.prior(prob.G, poses[0][None], prob.Zp[k][None])
    return [Cp[0]]


def unroll_step_vjp(prob: PGOProblem, T, delta, L, v, alpha: float = 1.0, h: float = FD_STEP):
    """Reverse one GN step theta_{k+1} = theta_k Exp(-alpha H^-1 b).  v: dL/dtheta_{k+1} [N, d].
    Returns (dL/dtheta_k [N, d], dL/dw_edge [E], dL/dw_prior [P])."""
    G, d, N = prob.G, prob.d, prob.n_vars
    v = np.asarray(v, dtype=np.float64).reshape(N, d)
    dl = np.asarray(delta).reshape(N, d)
    # retraction adjoint
    u = np.zeros((N, d))
    vk = np.zeros((N, d))
    for m in range(N):
        u[m] = -alpha * G.jr(-alpha * dl[m][None])[0].T @ v[m]
        vk[m] = G.adjoint(G.exp(alpha * dl[m][None]))[0].T @ v[m]
    lam = linalg.chol_solve(L, u.reshape(-1)).reshape(N, d)
    gw = np.zeros(len(prob.w))
    gp = np.zeros(len(prob.wp))
    terms = [("edge", k, (int(i), int(j)), prob.w[k]) for k, (i, j) in enumerate(prob.edges)]
    terms += [("prior", k, (int(p),), prob.wp[k]) for k, p in enumerate(prob.prior_vars)]
    c_e, Ci_e, Cj_e = prob.edge_terms(T)
    if len(prob.prior_vars):
        c_p, C_p = prob.prior_terms(T)
    for kind, k, vars_, w in terms:
        if kind == "edge":
            c, Cb = c_e[k], [Ci_e[k], Cj_e[k]]
        else:
            c, Cb = c_p[k], [C_p[k]]
        lam_e = [lam[a] for a in vars_]
        del_e = [dl[a] for a in vars_]
        q = sum(C @ x for C, x in zip(Cb, lam_e))          # C lambda_e
        Cd = sum(C @ x for C, x in zip(Cb, del_e))         # C delta_e
        p = c - Cd
        g = 2.0 * w * (q @ c - q @ Cd)
        if kind == "edge":
            gw[k] += g
        else:
            gp[k] += g
        # dL/deta of the term: w^2 [C^T q + grad_eta((C(eta) lambda).p - (C(eta) delta).q)]
        for slot, a in enumerate(vars_):
            grad = Cb[slot].T @ q
            for t in range(d):
                e = np.zeros(d)
                e[t] = h
                vals = []
                for sgn in (1.0, -1.0):
                    poses = [T[b] for b in vars_]
                    poses[slot] = poses[slot] @ G.exp((sgn * e)[None])[0]
                    Cn = _jac_at(prob, kind, k, poses)
                    vals.append(sum(C @ x for C, x in zip(Cn, lam_e)) @ p -
                                sum(C @ x for C, x in zip(Cn, del_e)) @ q)
                grad[t] += (vals[0] - vals[1]) / (2.0 * h)
            vk[a] += w * w * grad
    return vk, gw, gp


def unroll_weight_grads(prob: PGOProblem, T0, K: int, v, alpha: float = 1.0, truncate: int | None = None,
                        h: float = FD_STEP):
    """Unroll (truncate None or >= K) / Truncated backward of K GN steps from T0 for the upstream
    gradient v = dL/dtheta_K [N*d].  Returns (theta_K, grad_w_edge [E], grad_w_prior [P],
    grad_theta0 [N, d] (zero when truncated))."""
    TK, Ts, ds, Ls = gn_history(prob, T0, K, alpha)
    Tw = K if truncate is None else min(int(truncate), K)
    vk = np.asarray(v, dtype=np.float64).reshape(prob.n_vars, prob.d)
    gw = np.zeros(len(prob.w))
    gp = np.zeros(len(prob.wp))
    for k in range(K - 1, K - 1 - Tw, -1):
        vk, a, c = unroll_step_vjp(prob, Ts[k], ds[k], Ls[k], vk, alpha, h)
        gw += a
        gp += c
    g0 = vk if Tw == K else np.zeros_like(vk)
    return TK, gw, gp, g0
