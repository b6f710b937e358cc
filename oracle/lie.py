"""Oracle Lie-group closed forms ("exponential and logarithm map, inverse,
composition ... in closed form"), fp64 NumPy, vectorised over leading axes.

Conventions (readings A1/A2): right (body-frame) perturbation T <- T Exp(xi);
SE3 tangent xi = (rho, omega) translation first; SE2 xi = (rho_x, rho_y, omega).
Elements are homogeneous matrices [..., 4, 4] (SE3) / [..., 3, 3] (SE2).

Coefficient functions use even Taylor polynomials below pinned switch points
(reading A7: A,B,C,D,f below theta=0.5, c2,c3 below theta=1.0), closed forms
above.  A second, independent route (``jr_series``: sum_k (-ad)^k/(k+1)!) exists only to
pin the closed forms in tests.
"""
from __future__ import annotations

from fractions import Fraction
from math import factorial

import numpy as np

# ----------------------------------------------------------------------------- series


def _bernoulli(nmax: int) -> list[Fraction]:
    """Bernoulli numbers B_0..B_nmax (B_1 = -1/2 convention) by the standard recurrence."""
    B = [Fraction(0)] * (nmax + 1)
    B[0] = Fraction(1)
    for m in range(1, nmax + 1):
        s = Fraction(0)
        for k in range(m):
            s += Fraction(factorial(m + 1), factorial(k) * factorial(m + 1 - k)) * B[k]
        B[m] = -s / (m + 1)
    return B


_BN = _bernoulli(40)
_SW = 0.5    # switch point for A, B, C, D, f
_SW2 = 1.0   # switch point for c2, c3
_NT = 10     # series terms below _SW
_NT2 = 12    # series terms below _SW2

# series coefficients in powers of theta^2
_A_S = [(-1) ** k / factorial(2 * k + 1) for k in range(_NT)]
_B_S = [(-1) ** k / factorial(2 * k + 2) for k in range(_NT)]
_C_S = [(-1) ** k / factorial(2 * k + 3) for k in range(_NT)]
# D = 1/t^2 - (1+cos t)/(2 t sin t) = sum_{n>=1} (-1)^(n+1) B_2n t^(2n-2) / (2n)!
_D_S = [float((-1) ** (n + 1) * _BN[2 * n] / factorial(2 * n)) for n in range(1, _NT + 1)]
# f = t/(2 sin t) = 1/2 * sum_{n>=0} (-1)^(n+1) (2^(2n) - 2) B_2n t^(2n) / (2n)!
_F_S = [float(Fraction(1, 2) * (-1) ** (n + 1) * (2 ** (2 * n) - 2) * _BN[2 * n] / factorial(2 * n))
        for n in range(_NT)]
_C2_S = [(-1) ** k / factorial(2 * k + 4) for k in range(_NT2)]
_C3_S = [(-1) ** k * (k + 1) / factorial(2 * k + 5) for k in range(_NT2)]


def _poly(coeffs, t2):
    out = np.zeros_like(t2)
    for c in reversed(coeffs):
        out = out * t2 + c
    return out


def _branch(t, sw, series, closed):
    t = np.asarray(t, dtype=np.float64)
    small = t < sw
    ts = np.where(small, 1.0, t)          # safe argument for the closed form
    with np.errstate(divide="ignore", invalid="ignore"):
        cf = closed(ts)
    return np.where(small, _poly(series, t * t), cf)


def coef_A(t):   # sin t / t
    return _branch(t, _SW, _A_S, lambda s: np.sin(s) / s)


def coef_B(t):   # (1 - cos t) / t^2
    return _branch(t, _SW, _B_S, lambda s: (1 - np.cos(s)) / s ** 2)


def coef_C(t):   # (t - sin t) / t^3
    return _branch(t, _SW, _C_S, lambda s: (s - np.sin(s)) / s ** 3)


def coef_D(t):   # 1/t^2 - (1 + cos t) / (2 t sin t)
    return _branch(t, _SW, _D_S, lambda s: 1 / s ** 2 - (1 + np.cos(s)) / (2 * s * np.sin(s)))


def coef_f(t):   # t / (2 sin t)
    return _branch(t, _SW, _F_S, lambda s: s / (2 * np.sin(s)))


def coef_c2(t):  # (t^2 + 2 cos t - 2) / (2 t^4)
    return _branch(t, _SW2, _C2_S, lambda s: (s ** 2 + 2 * np.cos(s) - 2) / (2 * s ** 4))


def coef_c3(t):  # (2 t - 3 sin t + t cos t) / (2 t^5)
    return _branch(t, _SW2, _C3_S, lambda s: (2 * s - 3 * np.sin(s) + s * np.cos(s)) / (2 * s ** 5))


# ----------------------------------------------------------------------------- SO(3)


def hat3(w):
    w = np.asarray(w, dtype=np.float64)
    W = np.zeros(w.shape[:-1] + (3, 3))
    W[..., 0, 1] = -w[..., 2]
    W[..., 0, 2] = w[..., 1]
    W[..., 1, 0] = w[..., 2]
    W[..., 1, 2] = -w[..., 0]
    W[..., 2, 0] = -w[..., 1]
    W[..., 2, 1] = w[..., 0]
    return W


def vee3(W):
    return np.stack([W[..., 2, 1], W[..., 0, 2], W[..., 1, 0]], axis=-1)


def _eye(shape, n):
    return np.broadcast_to(np.eye(n), tuple(shape) + (n, n)).copy()


def _sc(c):  # scalar field -> broadcastable over a 3x3 matrix
    return np.asarray(c)[..., None, None]


def so3_exp(w):
    """R = I + A W + B W^2 (Rodrigues)."""
    t = np.linalg.norm(w, axis=-1)
    W = hat3(w)
    return _eye(t.shape, 3) + _sc(coef_A(t)) * W + _sc(coef_B(t)) * (W @ W)


def so3_log(R):
    """theta = atan2(|vee(R - R^T)|/2, (tr R - 1)/2); omega = f(theta) vee(R - R^T)."""
    v = vee3(R - np.swapaxes(R, -1, -2))
    s = np.linalg.norm(v, axis=-1) / 2
    c = (np.trace(R, axis1=-2, axis2=-1) - 1) / 2
    t = np.arctan2(s, c)
    return coef_f(t)[..., None] * v


def so3_jl(w):
    t = np.linalg.norm(w, axis=-1)
    W = hat3(w)
    return _eye(t.shape, 3) + _sc(coef_B(t)) * W + _sc(coef_C(t)) * (W @ W)


def so3_jr(w):
    return so3_jl(-np.asarray(w))


def so3_jr_inv(w):
    """Jr^-1(omega) = I + W/2 + D W^2."""
    t = np.linalg.norm(w, axis=-1)
    W = hat3(w)
    return _eye(t.shape, 3) + 0.5 * W + _sc(coef_D(t)) * (W @ W)


def so3_jl_inv(w):
    """Jl^-1(omega) = I - W/2 + D W^2."""
    t = np.linalg.norm(w, axis=-1)
    W = hat3(w)
    return _eye(t.shape, 3) - 0.5 * W + _sc(coef_D(t)) * (W @ W)


# ----------------------------------------------------------------------------- SE(3)


def se3_from(R, t):
    T = np.zeros(R.shape[:-2] + (4, 4))
    T[..., :3, :3] = R
    T[..., :3, 3] = t
    T[..., 3, 3] = 1.0
    return T


def se3_inv(T):
    R = T[..., :3, :3]
    Rt = np.swapaxes(R, -1, -2)
    return se3_from(Rt, -np.einsum("...ij,...j->...i", Rt, T[..., :3, 3]))


def se3_exp(xi):
    """Exp(rho, omega) = [Exp(omega) | Jl(omega) rho]."""
    xi = np.asarray(xi, dtype=np.float64)
    rho, w = xi[..., :3], xi[..., 3:]
    return se3_from(so3_exp(w), np.einsum("...ij,...j->...i", so3_jl(w), rho))


def se3_log(T):
    """Log(T) = (Jl^-1(omega) t, omega), omega = Log(R)."""
    w = so3_log(T[..., :3, :3])
    rho = np.einsum("...ij,...j->...i", so3_jl_inv(w), T[..., :3, 3])
    return np.concatenate([rho, w], axis=-1)


def se3_adjoint(T):
    """Ad(T) = [[R, t^ R], [0, R]]  (so that T Exp(xi) T^-1 = Exp(Ad_T xi))."""
    R = T[..., :3, :3]
    tR = hat3(T[..., :3, 3]) @ R
    A = np.zeros(T.shape[:-2] + (6, 6))
    A[..., :3, :3] = R
    A[..., :3, 3:] = tR
    A[..., 3:, 3:] = R
    return A


def se3_Q(rho, phi):
    """Barfoot's Q(rho, phi) (the off-diagonal block of the SE(3) left Jacobian)."""
    t = np.linalg.norm(phi, axis=-1)
    P = hat3(phi)
    Rh = hat3(rho)
    PR = P @ Rh
    RP = Rh @ P
    PRP = P @ Rh @ P
    PP = P @ P
    return (0.5 * Rh
            + _sc(coef_C(t)) * (PR + RP + PRP)
            + _sc(coef_c2(t)) * (PP @ Rh + Rh @ PP - 3 * PRP)
            + _sc(coef_c3(t)) * (PRP @ P + PP @ Rh @ P))


def se3_jr(xi):
    """Jr(xi) = [[Jr(omega), Q(-rho, -omega)], [0, Jr(omega)]]."""
    xi = np.asarray(xi, dtype=np.float64)
    rho, w = xi[..., :3], xi[..., 3:]
    J = so3_jr(w)
    out = np.zeros(xi.shape[:-1] + (6, 6))
    out[..., :3, :3] = J
    out[..., :3, 3:] = se3_Q(-rho, -w)
    out[..., 3:, 3:] = J
    return out


def se3_jr_inv(xi):
    """Jr^-1(xi) = [[Jr^-1, -Jr^-1 Q(-rho,-omega) Jr^-1], [0, Jr^-1]]."""
    xi = np.asarray(xi, dtype=np.float64)
    rho, w = xi[..., :3], xi[..., 3:]
    Ji = so3_jr_inv(w)
    out = np.zeros(xi.shape[:-1] + (6, 6))
    out[..., :3, :3] = Ji
    out[..., :3, 3:] = -Ji @ se3_Q(-rho, -w) @ Ji
    out[..., 3:, 3:] = Ji
    return out


def se3_ad(xi):
    """ad_xi = [[omega^, rho^], [0, omega^]]."""
    xi = np.asarray(xi, dtype=np.float64)
    out = np.zeros(xi.shape[:-1] + (6, 6))
    W = hat3(xi[..., 3:])
    out[..., :3, :3] = W
    out[..., :3, 3:] = hat3(xi[..., :3])
    out[..., 3:, 3:] = W
    return out


def se3_hat(xi):
    xi = np.asarray(xi, dtype=np.float64)
    X = np.zeros(xi.shape[:-1] + (4, 4))
    X[..., :3, :3] = hat3(xi[..., 3:])
    X[..., :3, 3] = xi[..., :3]
    return X


# ----------------------------------------------------------------------------- SE(2)


def se2_from(theta, t):
    theta = np.asarray(theta, dtype=np.float64)
    T = np.zeros(theta.shape + (3, 3))
    c, s = np.cos(theta), np.sin(theta)
    T[..., 0, 0] = c
    T[..., 0, 1] = -s
    T[..., 1, 0] = s
    T[..., 1, 1] = c
    T[..., :2, 2] = t
    T[..., 2, 2] = 1.0
    return T


def se2_inv(T):
    R = T[..., :2, :2]
    Rt = np.swapaxes(R, -1, -2)
    out = np.zeros(T.shape)
    out[..., :2, :2] = Rt
    out[..., :2, 2] = -np.einsum("...ij,...j->...i", Rt, T[..., :2, 2])
    out[..., 2, 2] = 1.0
    return out


def _se2_V(w):
    """V(omega) = [[A, -w B], [w B, A]] with A = sin w / w, w B = (1 - cos w)/w."""
    t = np.abs(w)
    A = coef_A(t)
    wB = w * coef_B(t)
    V = np.zeros(np.shape(w) + (2, 2))
    V[..., 0, 0] = A
    V[..., 0, 1] = -wB
    V[..., 1, 0] = wB
    V[..., 1, 1] = A
    return V


def se2_exp(xi):
    """Exp(rho, omega) = [R(omega) | V(omega) rho]."""
    xi = np.asarray(xi, dtype=np.float64)
    w = xi[..., 2]
    return se2_from(w, np.einsum("...ij,...j->...i", _se2_V(w), xi[..., :2]))


def se2_log(T):
    """omega = atan2(R10, R00), rho = V(omega)^-1 t."""
    w = np.arctan2(T[..., 1, 0], T[..., 0, 0])
    rho = np.linalg.solve(_se2_V(w), T[..., :2, 2][..., None])[..., 0]
    return np.concatenate([rho, w[..., None]], axis=-1)


def se2_adjoint(T):
    """Ad(T) = [[R, (t_y, -t_x)^T], [0, 1]]."""
    A = np.zeros(T.shape[:-2] + (3, 3))
    A[..., :2, :2] = T[..., :2, :2]
    A[..., 0, 2] = T[..., 1, 2]
    A[..., 1, 2] = -T[..., 0, 2]
    A[..., 2, 2] = 1.0
    return A


def se2_jr(xi):
    """Closed-form right Jacobian of SE(2):
    [[A, wB, wC r1 - B r2], [-wB, A, B r1 + wC r2], [0, 0, 1]]  (A,B,C of |w|)."""
    xi = np.asarray(xi, dtype=np.float64)
    r1, r2, w = xi[..., 0], xi[..., 1], xi[..., 2]
    t = np.abs(w)
    A, B, C = coef_A(t), coef_B(t), coef_C(t)
    J = np.zeros(xi.shape[:-1] + (3, 3))
    J[..., 0, 0] = A
    J[..., 0, 1] = w * B
    J[..., 0, 2] = w * C * r1 - B * r2
    J[..., 1, 0] = -w * B
    J[..., 1, 1] = A
    J[..., 1, 2] = B * r1 + w * C * r2
    J[..., 2, 2] = 1.0
    return J


def se2_jr_inv(xi):
    """Jr^-1 = [[M^-1, -M^-1 v], [0, 1]] for Jr = [[M, v], [0, 1]]."""
    J = se2_jr(xi)
    M = J[..., :2, :2]
    v = J[..., :2, 2]
    det = M[..., 0, 0] * M[..., 1, 1] - M[..., 0, 1] * M[..., 1, 0]
    Mi = np.zeros(M.shape)
    Mi[..., 0, 0] = M[..., 1, 1] / det
    Mi[..., 0, 1] = -M[..., 0, 1] / det
    Mi[..., 1, 0] = -M[..., 1, 0] / det
    Mi[..., 1, 1] = M[..., 0, 0] / det
    out = np.zeros(J.shape)
    out[..., :2, :2] = Mi
    out[..., :2, 2] = -np.einsum("...ij,...j->...i", Mi, v)
    out[..., 2, 2] = 1.0
    return out


def se2_ad(xi):
    """ad_xi = [[0, -w, rho_y], [w, 0, -rho_x], [0, 0, 0]]."""
    xi = np.asarray(xi, dtype=np.float64)
    out = np.zeros(xi.shape[:-1] + (3, 3))
    out[..., 0, 1] = -xi[..., 2]
    out[..., 1, 0] = xi[..., 2]
    out[..., 0, 2] = xi[..., 1]
    out[..., 1, 2] = -xi[..., 0]
    return out


def se2_hat(xi):
    xi = np.asarray(xi, dtype=np.float64)
    X = np.zeros(xi.shape[:-1] + (3, 3))
    X[..., 0, 1] = -xi[..., 2]
    X[..., 1, 0] = xi[..., 2]
    X[..., :2, 2] = xi[..., :2]
    return X


# ----------------------------------------------------------------------------- second route (pins only)


def jr_series(ad, terms: int = 60):
    """Jr(xi) = sum_{k>=0} (-ad_xi)^k / (k+1)!  -- independent route used only by tests."""
    n = ad.shape[-1]
    out = _eye(ad.shape[:-2], n)
    P = _eye(ad.shape[:-2], n)
    for k in range(1, terms):
        P = -(P @ ad) / (k + 1)
        out = out + P
    return out


# ----------------------------------------------------------------------------- group objects


class _Group:
    name = ""
    d = 0       # tangent dimension
    m = 0       # homogeneous matrix size


class SE3(_Group):
    name, d, m = "SE3", 6, 4
    exp = staticmethod(se3_exp)
    log = staticmethod(se3_log)
    inv = staticmethod(se3_inv)
    adjoint = staticmethod(se3_adjoint)
    jr = staticmethod(se3_jr)
    jr_inv = staticmethod(se3_jr_inv)
    ad = staticmethod(se3_ad)
    hat = staticmethod(se3_hat)


class SE2(_Group):
    name, d, m = "SE2", 3, 3
    exp = staticmethod(se2_exp)
    log = staticmethod(se2_log)
    inv = staticmethod(se2_inv)
    adjoint = staticmethod(se2_adjoint)
    jr = staticmethod(se2_jr)
    jr_inv = staticmethod(se2_jr_inv)
    ad = staticmethod(se2_ad)
    hat = staticmethod(se2_hat)


def group(name_or_d):
    if name_or_d in ("SE3", 6, 3 + 3):
        return SE3
    if name_or_d in ("SE2", 3):
        return SE2
    raise ValueError(f"unknown group {name_or_d!r}")


def to_homog(P):
    """[..., r, r+1] top rows -> [..., r+1, r+1] homogeneous."""
    P = np.asarray(P, dtype=np.float64)
    r = P.shape[-2]
    T = np.zeros(P.shape[:-2] + (r + 1, r + 1))
    T[..., :r, :] = P
    T[..., r, r] = 1.0
    return T


def from_homog(T):
    r = T.shape[-1] - 1
    return np.ascontiguousarray(T[..., :r, :])
