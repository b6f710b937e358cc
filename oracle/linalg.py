"""Oracle dense linear algebra: assembly of the Gauss-Newton normal equations
("(sum_i J_i^T J_i) delta = (sum_i J_i^T r_i)"), Marquardt damping
(SPEC.md:330), textbook Cholesky with the per-element pivot rule (DESIGN.md reading
A15: fail if a pivot <= 1e-13 * max diag H), forward/back substitution, and the
linear-solve backward of PAPER.md:224 (dL/db = A^-1 dL/dy, dL/dA = -A^-1 (dL/dy) y^T).
"""
from __future__ import annotations

import numpy as np

PIVOT_REL_TOL = 1e-13


def assemble(n_vars: int, d: int, blocks):
    """Dense H (n x n), b (n) with n = n_vars*d from residual blocks.

    ``blocks`` is an iterable of (var_ids tuple, [J_v (m x d) per var], r (m)) with the
    residual ALREADY weighted.  H = sum J^T J, b = sum J^T r.
    """
    n = n_vars * d
    H = np.zeros((n, n))
    b = np.zeros(n)
    for vids, Js, r in blocks:
        for a, Ja in zip(vids, Js):
            sa = slice(a * d, (a + 1) * d)
            b[sa] += Ja.T @ r
            for c, Jc in zip(vids, Js):
                sc = slice(c * d, (c + 1) * d)
                H[sa, sc] += Ja.T @ Jc
    return H, b


def damp(H, lam: float, mode: str = "marquardt"):
    """H_lambda = H + lambda * diag(H)  (Marquardt) or H + lambda * I."""
    Hd = H.copy()
    idx = np.arange(H.shape[0])
    if mode == "marquardt":
        Hd[idx, idx] += lam * np.diag(H)
    else:
        Hd[idx, idx] += lam
    return Hd


def cholesky(A, rel_tol: float = PIVOT_REL_TOL):
    """Textbook (Cholesky-Crout, column by column) A = L L^T, no pivoting.

    Returns (L, ok).  ok is False if some pivot A_jj - sum_k L_jk^2 <= rel_tol * max diag A.
    For n > 3000 LAPACK (numpy.linalg.cholesky) computes L; the pivot rule is then
    applied to the squared diagonal of L.
    """
    A = np.asarray(A, dtype=np.float64)
    n = A.shape[0]
    tol = rel_tol * float(np.max(np.diag(A))) if n else 0.0
    if n > 3000:
        try:
            L = np.linalg.cholesky(A)
        except np.linalg.LinAlgError:
            return np.zeros_like(A), False
        return L, bool(np.all(np.diag(L) ** 2 > tol))
    L = np.zeros_like(A)
    for j in range(n):
        piv = A[j, j] - L[j, :j] @ L[j, :j]
        if not piv > tol:
            return L, False
        L[j, j] = np.sqrt(piv)
        if j + 1 < n:
            L[j + 1:, j] = (A[j + 1:, j] - L[j + 1:, :j] @ L[j, :j]) / L[j, j]
    return L, True


def forward_sub(L, b):
    """Solve L y = b (L lower triangular), row by row."""
    n = L.shape[0]
    y = np.zeros(n)
    for i in range(n):
        y[i] = (b[i] - L[i, :i] @ y[:i]) / L[i, i]
    return y


def back_sub(L, y):
    """Solve L^T x = y, row by row from the bottom."""
    n = L.shape[0]
    x = np.zeros(n)
    for i in range(n - 1, -1, -1):
        x[i] = (y[i] - L[i + 1:, i] @ x[i + 1:]) / L[i, i]
    return x


def chol_solve(L, b):
    """x = L^-T L^-1 b."""
    return back_sub(L, forward_sub(L, b))


def linear_solve_backward(A, y, gy):
    """dL/db = A^-1 dL/dy ; dL/dA = -A^-1 (dL/dy) y^T."""
    gb = np.linalg.solve(A, gy)
    return gb, -np.outer(gb, y)
