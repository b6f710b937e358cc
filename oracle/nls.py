"""Oracle nonlinear least squares: Gauss-Newton and Levenberg-Marquardt executed step by
step in the paper's order: linearise, assemble (sum J^T J) delta =
(sum J^T r) densely, solve by dense Cholesky, update theta <- theta [-] delta by the
retraction (reading A5: T <- T Exp(-alpha delta)).

LM (PAPER.md:64 "damp the linear system", :153 "adaptive damping"; constants are our
reading A13 / SPEC.md:415,440): H_lambda = H + lambda diag(H); trial theta'; accept iff
S(theta') < S(theta) strictly, then lambda <- max(lambda/down, lambda_min); otherwise keep
theta and lambda <- min(lambda*up, lambda_max); a rejected step reuses the
linearisation.  A non-SPD damped system counts as a rejection.  A rejection while
lambda is already lambda_max marks the element "damping saturated" (status 3, frozen).

Status codes (shared meaning with include/dnls.h): 0 ok, 1 converged early (early stop),
2 not SPD (GN: element frozen), 3 LM damping saturated.

Two problem types implement ``linearize / objective / retract``:
  * PGOProblem  -- SE2/SE3 pose graph with Between + Prior costs (oracle.costs);
  * EuclidProblem -- vector variables with user residual/Jacobian callables (used to
    pin GN on App. B's curve fit and on affine residuals).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import costs, linalg, robust
from .lie import group, to_homog

ST_OK, ST_CONVERGED, ST_NOT_SPD, ST_SATURATED = 0, 1, 2, 3


class PGOProblem:
    """One batch element of a pose graph (poses are homogeneous matrices [N, m, m])."""

    def __init__(self, G, num_vars, edges, prior_vars, meas, prior_meas, w_edge, w_prior, radius=None):
        """radius: Welsch radius k of the Between edges (oracle.robust, readings W1-W3) or None."""
        self.radius = None if radius is None else float(radius)
        self.G = group(G) if not hasattr(G, "d") else G
        self.d = self.G.d
        self.n_vars = int(num_vars)
        self.edges = np.asarray(edges, dtype=np.int64).reshape(-1, 2)
        self.prior_vars = np.asarray(prior_vars, dtype=np.int64).reshape(-1)
        m = self.G.m
        self.Z = to_homog(meas) if np.shape(meas)[-2] == m - 1 else np.asarray(meas, dtype=np.float64)
        self.Zp = to_homog(prior_meas) if np.shape(prior_meas)[-2] == m - 1 else np.asarray(prior_meas, dtype=np.float64)
        self.w = np.asarray(w_edge, dtype=np.float64).reshape(-1)
        self.wp = np.asarray(w_prior, dtype=np.float64).reshape(-1)

    # -- per-cost pieces ----------------------------------------------------------
    def edge_terms(self, T):
        e = self.edges
        return costs.between(self.G, T[e[:, 0]], T[e[:, 1]], self.Z)

    def prior_terms(self, T):
        return costs.prior(self.G, T[self.prior_vars], self.Zp)

    def objective(self, T):
        if self.radius is None:
            return costs.objective(self.G, T, self.edges, self.Z, self.w, self.prior_vars, self.Zp, self.wp)
        c, _, _ = self.edge_terms(T)
        s = np.sum((self.w[:, None] * c) ** 2, axis=1)
        S = float(np.sum(robust.rho(s, self.radius)))
        if len(self.prior_vars):
            cp, _ = self.prior_terms(T)
            S += 0.5 * float(np.sum((self.wp[:, None] * cp) ** 2))
        return S

    def irls_weights(self, c):
        """psi_e = exp(-||w_e c_e||^2 / k^2) per edge (ones without a robust kernel)."""
        if self.radius is None:
            return np.ones(len(self.w))
        return robust.psi(np.sum((self.w[:, None] * c) ** 2, axis=1), self.radius)

    def blocks(self, T):
        """Weighted (and, with a robust kernel, IRLS-rescaled by sqrt(psi)) Jacobians / residuals."""
        c, Ci, Cj = self.edge_terms(T)
        sq = np.sqrt(self.irls_weights(c))
        out = []
        for k, (i, j) in enumerate(self.edges):
            w = self.w[k] * sq[k]
            out.append(((int(i), int(j)), [w * Ci[k], w * Cj[k]], w * c[k]))
        if len(self.prior_vars):
            cp, Cp = self.prior_terms(T)
            for k, p in enumerate(self.prior_vars):
                out.append(((int(p),), [self.wp[k] * Cp[k]], self.wp[k] * cp[k]))
        return out

    def linearize(self, T):
        blocks = self.blocks(T)
        S = 0.5 * sum(float(r @ r) for _, _, r in blocks) if self.radius is None else self.objective(T)
        H, b = linalg.assemble(self.n_vars, self.d, blocks)
        return S, H, b

    def retract(self, T, delta):
        """T_m <- T_m Exp(delta_m)."""
        return T @ self.G.exp(np.asarray(delta).reshape(self.n_vars, self.d))


class EuclidProblem:
    """Vector variables x [n_vars, d]; residual(x) -> r (m), jacobian(x) -> J (m x n)."""

    def __init__(self, n_vars, d, residual, jacobian):
        self.n_vars, self.d = int(n_vars), int(d)
        self.residual, self.jacobian = residual, jacobian

    def objective(self, x):
        r = self.residual(x)
        return 0.5 * float(r @ r)

    def linearize(self, x):
        r = self.residual(x)
        J = self.jacobian(x)
        return 0.5 * float(r @ r), J.T @ J, J.T @ r

    def retract(self, x, delta):
        return x + np.asarray(delta).reshape(self.n_vars, self.d)


@dataclass
class Options:
    optimizer: str = "gn"          # "gn" | "lm" | "dogleg"
    max_iterations: int = 10
    step_size: float = 1.0
    lambda0: float = 1e-3
    lambda_min: float = 1e-8
    lambda_max: float = 1e5
    lambda_down: float = 3.0
    lambda_up: float = 2.0
    damping: str = "marquardt"     # "marquardt" | "identity"
    early_stop: bool = False
    abs_tol: float = 1e-10
    rel_tol: float = 1e-8
    implicit: bool = False
    delta0: float = 1.0            # Dogleg trust radius: initial, max, min (reading DL1)
    delta_max: float = 1e4
    delta_min: float = 1e-10


@dataclass
class Result:
    x: np.ndarray
    objective: float               # S(theta_K)
    status: int
    iterations: int
    history: list = field(default_factory=list)   # S(theta_k) for k = 0..K
    lam: float = 0.0
    trials: list = field(default_factory=list)    # LM: (S, S_trial or None, accepted) per iteration
    H_final: np.ndarray | None = None              # undamped H(theta_K) (implicit mode)
    L_final: np.ndarray | None = None              # its Cholesky factor


def gauss_newton(prob, x0, opt: Options) -> Result:
    x = np.array(x0, dtype=np.float64, copy=True)
    status, iters = ST_OK, 0
    hist = []
    S_prev = None
    for k in range(opt.max_iterations):
        S, H, b = prob.linearize(x)
        hist.append(S)
        if opt.early_stop and S_prev is not None and abs(S - S_prev) < opt.abs_tol + opt.rel_tol * S_prev:
            status = ST_CONVERGED
            break
        L, ok = linalg.cholesky(H)
        if not ok:
            status = ST_NOT_SPD
            break
        delta = linalg.chol_solve(L, b)
        x = prob.retract(x, -opt.step_size * delta)
        iters += 1
        S_prev = S
    return _finish(prob, x, status, iters, hist, 0.0, opt)


def levenberg_marquardt(prob, x0, opt: Options) -> Result:
    x = np.array(x0, dtype=np.float64, copy=True)
    status, iters = ST_OK, 0
    lam = opt.lambda0
    hist = []
    trials = []
    S, H, b = prob.linearize(x)
    S_prev = None
    for k in range(opt.max_iterations):
        if opt.early_stop and S_prev is not None and abs(S - S_prev) < opt.abs_tol + opt.rel_tol * S_prev:
            status = ST_CONVERGED
            break
        hist.append(S)
        iters += 1
        L, ok = linalg.cholesky(linalg.damp(H, lam, opt.damping))
        accept = False
        S_try = None
        if ok:
            delta = linalg.chol_solve(L, b)
            x_try = prob.retract(x, -opt.step_size * delta)
            S_try = prob.objective(x_try)
            accept = S_try < S
        trials.append((S, S_try, accept))
        if accept:
            x = x_try
            lam = max(lam / opt.lambda_down, opt.lambda_min)
            S_prev = S
            S, H, b = prob.linearize(x)
        else:
            if lam >= opt.lambda_max:
                status = ST_SATURATED
                break
            lam = min(lam * opt.lambda_up, opt.lambda_max)
    res = _finish(prob, x, status, iters, hist, lam, opt)
    res.trials = trials
    return res


def dogleg(prob, x0, opt: Options) -> Result:
    """Powell's dogleg trust-region step ("Dogleg"; reading DL1).
    With b = J^T r (the gradient of S), H = J^T J and our sign convention theta <- theta [+] (-d):
      d_gn = H^-1 b;  if |d_gn| <= Delta: d = d_gn
      else d_c = (b.b / b.Hb) b;  if |d_c| >= Delta: d = (Delta / |b|) b
      else d = d_c + tau (d_gn - d_c), tau in [0, 1] with |d| = Delta;
    predicted decrease b.d - 1/2 d.Hd, gain ratio rho = (S - S(theta [+] -d)) / predicted;
    accept iff rho > 0; rho > 0.75: Delta <- min(2 Delta, Delta_max); rho < 0.25: Delta <- Delta / 2;
    a rejection with Delta < Delta_min marks the element (status 3, trust region collapsed)."""
    x = np.array(x0, dtype=np.float64, copy=True)
    status, iters = ST_OK, 0
    Delta = opt.delta0
    hist, trials = [], []
    S, H, b = prob.linearize(x)
    S_prev = None
    for k in range(opt.max_iterations):
        if opt.early_stop and S_prev is not None and abs(S - S_prev) < opt.abs_tol + opt.rel_tol * S_prev:
            status = ST_CONVERGED
            break
        hist.append(S)
        iters += 1
        L, ok = linalg.cholesky(H)
        if not ok:
            status = ST_NOT_SPD
            break
        d_gn = linalg.chol_solve(L, b)
        if np.linalg.norm(d_gn) <= Delta:
            d, kind = d_gn, "gn"
        else:
            bb = float(b @ b)
            d_c = (bb / float(b @ H @ b)) * b
            if np.linalg.norm(d_c) >= Delta:
                d, kind = (Delta / np.sqrt(bb)) * b, "sd"
            else:
                u = d_gn - d_c
                qa, qb, qc = float(u @ u), 2.0 * float(d_c @ u), float(d_c @ d_c) - Delta * Delta
                tau = (-qb + np.sqrt(qb * qb - 4.0 * qa * qc)) / (2.0 * qa)
                d, kind = d_c + tau * u, "dogleg"
        pred = float(b @ d) - 0.5 * float(d @ H @ d)
        x_try = prob.retract(x, -d)
        S_try = prob.objective(x_try)
        rho = (S - S_try) / pred if pred > 0 else 0.0
        accept = rho > 0
        trials.append((S, S_try, accept, rho, Delta, kind, float(np.linalg.norm(d_gn))))
        if rho > 0.75:
            Delta = min(2.0 * Delta, opt.delta_max)
        elif rho < 0.25:
            Delta = 0.5 * Delta
        if accept:
            x = x_try
            S_prev = S
            S, H, b = prob.linearize(x)
        elif Delta < opt.delta_min:
            status = ST_SATURATED
            break
    res = _finish(prob, x, status, iters, hist, Delta, opt)
    res.trials = trials
    return res


def _finish(prob, x, status, iters, hist, lam, opt) -> Result:
    res = Result(x=x, objective=prob.objective(x), status=status, iterations=iters,
                 history=hist, lam=lam)
    res.history = hist + [res.objective]
    if opt.implicit:
        _, H, _ = prob.linearize(x)
        L, ok = linalg.cholesky(H)
        res.H_final, res.L_final = H, (L if ok else None)
        if not ok:   # a failed final factor takes precedence: the implicit gradient is unavailable
            res.status = ST_NOT_SPD
    return res


def optimize(prob, x0, opt: Options) -> Result:
    if opt.optimizer == "gn":
        return gauss_newton(prob, x0, opt)
    if opt.optimizer == "lm":
        return levenberg_marquardt(prob, x0, opt)
    if opt.optimizer == "dogleg":
        return dogleg(prob, x0, opt)
    raise ValueError(opt.optimizer)


def solve_batch(G, num_vars, edges, prior_vars, poses0, meas, prior_meas, w_edge, w_prior,
                opt: Options, elements=None, radius=None):
    """Run the oracle on batch elements (all, or the listed indices).

    poses0/meas/prior_meas are [B][..][r][r+1] top-row arrays; w_edge/w_prior are [E]/[P]
    (shared) or [B][E]/[B][P]; radius None, a scalar or [B] (Welsch kernel of the edges).
    Returns a list of Result (poses in homogeneous form).
    """
    Gr = group(G) if not hasattr(G, "d") else G
    B = np.shape(poses0)[0]
    idx = range(B) if elements is None else elements
    out = []
    for b in idx:
        we = np.asarray(w_edge)
        wp = np.asarray(w_prior)
        rk = None if radius is None else float(np.asarray(radius).reshape(-1)[b if np.size(radius) > 1 else 0])
        prob = PGOProblem(Gr, num_vars, edges, prior_vars, meas[b], prior_meas[b],
                          we[b] if we.ndim == 2 else we, wp[b] if wp.ndim == 2 else wp, radius=rk)
        out.append(optimize(prob, to_homog(poses0[b]), opt))
    return out
