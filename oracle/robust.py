"""Oracle Welsch robust kernel ("we learn the radius of a Welsh robust cost function
for outlier rejection", :154 "robust loss functions") -- TEST INFRASTRUCTURE ONLY.

Reading (W1-W3):
  W1  a Between edge with weighted squared error s = ||w c||^2 costs
          rho_k(s) = (k^2 / 2) (1 - exp(-s / k^2))        (~ s/2 for s << k^2,
      so the non-robust 1/2 ||w c||^2 of reading A6 is the k -> inf limit); priors stay quadratic.
  W2  the Gauss-Newton step is the IRLS step: each edge's J and r are rescaled by sqrt(psi),
          psi(s) = 2 rho_k'(s) = exp(-s / k^2),
      so b = sum psi J^T r is the exact gradient of S and H = sum psi J^T J drops the rho''
      term (the Hessian the forward factors and the implicit backward reuses).
  W3  the radius k is a learnable parameter shared by all edges (and by the batch, like w).
"""
from __future__ import annotations

import numpy as np


def rho(s, k):
    """Welsch loss of the squared norm s (W1); expm1 keeps full precision for s << k^2."""
    s = np.asarray(s, dtype=np.float64)
    return -0.5 * k * k * np.expm1(-s / (k * k))


def psi(s, k):
    """IRLS weight 2 rho'(s) = exp(-s / k^2) (W2)."""
    return np.exp(-np.asarray(s, dtype=np.float64) / (k * k))


def kappa(s, k):
    """Residual rescale with 1/2 ||kappa r||^2 = rho(s); kappa(0) = 1."""
    s = np.asarray(s, dtype=np.float64)
    return np.where(s > 0, np.sqrt(2.0 * rho(s, k) / np.where(s > 0, s, 1.0)), 1.0)


def drho_dk(s, k):
    """d rho_k(s) / dk = k (1 - psi) - (s / k) psi."""
    p = psi(s, k)
    return -k * np.expm1(-np.asarray(s) / (k * k)) - (np.asarray(s) / k) * p
