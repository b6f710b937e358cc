"""Pins P1/P2: the oracle's Lie closed forms against
scipy.linalg.expm / logm, the independent ad-series route, mpmath coefficient values,
SPEC.md hand values and group identities."""
import math

import mpmath
import numpy as np
import pytest
from scipy.linalg import expm, logm

from oracle import lie

rng = np.random.default_rng(1234)


def rand_se3(n, rot=1.0, trans=1.0):
    xi = np.concatenate([rng.standard_normal((n, 3)) * trans, rng.standard_normal((n, 3)) * rot], axis=1)
    return xi


# ---------------------------------------------------------------- coefficient functions vs mpmath
mpmath.mp.dps = 60
MP = {
    "A": lambda t: mpmath.sin(t) / t,
    "B": lambda t: (1 - mpmath.cos(t)) / t ** 2,
    "C": lambda t: (t - mpmath.sin(t)) / t ** 3,
    "D": lambda t: 1 / t ** 2 - (1 + mpmath.cos(t)) / (2 * t * mpmath.sin(t)),
    "f": lambda t: t / (2 * mpmath.sin(t)),
    "c2": lambda t: (t ** 2 + 2 * mpmath.cos(t) - 2) / (2 * t ** 4),
    "c3": lambda t: (2 * t - 3 * mpmath.sin(t) + t * mpmath.cos(t)) / (2 * t ** 5),
}
FN = {"A": lie.coef_A, "B": lie.coef_B, "C": lie.coef_C, "D": lie.coef_D, "f": lie.coef_f,
      "c2": lie.coef_c2, "c3": lie.coef_c3}


@pytest.mark.parametrize("name", list(MP))
def test_coefficients_vs_mpmath(name):
    ts = np.concatenate([np.geomspace(1e-9, 3.0, 300), [0.4999999, 0.5, 0.5000001, 0.9999999, 1.0, 1.0000001]])
    got = FN[name](ts)
    for t, g in zip(ts, got):
        ref = float(MP[name](mpmath.mpf(float(t))))
        assert abs(g - ref) <= 1e-14 * max(1.0, abs(ref)), (name, t, g, ref)


def test_coefficients_at_zero():
    assert lie.coef_A(0.0) == 1.0
    assert lie.coef_B(0.0) == 0.5
    assert abs(lie.coef_C(0.0) - 1 / 6) < 1e-17
    assert abs(lie.coef_D(0.0) - 1 / 12) < 1e-17
    assert lie.coef_f(0.0) == 0.5
    assert abs(lie.coef_c2(0.0) - 1 / 24) < 1e-17
    assert abs(lie.coef_c3(0.0) - 1 / 120) < 1e-17


# ---------------------------------------------------------------- SO3 / SE3 exp/log
def test_so3_exp_hand_value():
    # SPEC.md:121  SO3 exp((pi/2, 0, 0)) = [[1,0,0],[0,0,-1],[0,1,0]]
    R = lie.so3_exp(np.array([math.pi / 2, 0, 0]))
    np.testing.assert_allclose(R, [[1, 0, 0], [0, 0, -1], [0, 1, 0]], atol=1e-15)
    np.testing.assert_allclose(lie.so3_exp(np.zeros(3)), np.eye(3), atol=0)


def test_se3_exp_vs_expm():
    xi = rand_se3(200)
    T = lie.se3_exp(xi)
    for k in range(len(xi)):
        np.testing.assert_allclose(T[k], expm(lie.se3_hat(xi[k])), atol=1e-13)


def test_se3_exp_vs_expm_small_angles():
    for s in [1e-9, 1e-6, 1e-4, 1e-2, 0.3, 0.49, 0.51, 0.99, 1.01]:
        xi = rand_se3(20)
        xi[:, 3:] *= s / np.linalg.norm(xi[:, 3:], axis=1, keepdims=True)
        T = lie.se3_exp(xi)
        for k in range(len(xi)):
            np.testing.assert_allclose(T[k], expm(lie.se3_hat(xi[k])), atol=2e-15 * (1 + np.abs(xi[k]).max()) * 10)


def test_se3_log_exp_roundtrip():
    xi = rand_se3(1000)
    n = np.linalg.norm(xi[:, 3:], axis=1, keepdims=True)
    xi[:, 3:] *= np.minimum(1.0, (math.pi - 0.1) / n)
    back = lie.se3_log(lie.se3_exp(xi))
    np.testing.assert_allclose(back, xi, atol=1e-12)


def test_se3_log_vs_logm():
    xi = rand_se3(50, rot=0.8)
    T = lie.se3_exp(xi)
    for k in range(len(xi)):
        X = np.real(logm(T[k]))
        ref = np.array([X[0, 3], X[1, 3], X[2, 3], X[2, 1], X[0, 2], X[1, 0]])
        np.testing.assert_allclose(lie.se3_log(T[k]), ref, atol=1e-11)


def test_se3_adjoint_identity():
    # T Exp(xi) T^-1 = Exp(Ad_T xi)
    T = lie.se3_exp(rand_se3(100))
    xi = rand_se3(100, rot=0.7)
    lhs = T @ lie.se3_exp(xi) @ lie.se3_inv(T)
    rhs = lie.se3_exp(np.einsum("kab,kb->ka", lie.se3_adjoint(T), xi))
    np.testing.assert_allclose(lhs, rhs, atol=1e-12)


def test_se3_jr_closed_vs_series():
    for scale in [1e-7, 1e-3, 0.3, 0.7, 1.5, 2.5]:
        xi = rand_se3(100)
        xi[:, 3:] *= scale / np.linalg.norm(xi[:, 3:], axis=1, keepdims=True)
        Jc = lie.se3_jr(xi)
        Js = lie.jr_series(lie.se3_ad(xi))
        np.testing.assert_allclose(Jc, Js, atol=1e-13)
        np.testing.assert_allclose(lie.se3_jr_inv(xi), np.linalg.inv(Js), atol=1e-12)


def test_se3_jr_inv_product_identity():
    xi = rand_se3(200)
    P = lie.se3_jr(xi) @ lie.se3_jr_inv(xi)
    np.testing.assert_allclose(P, np.broadcast_to(np.eye(6), P.shape), atol=1e-12)


def test_se3_jr_is_derivative_of_exp():
    # Exp(xi + h e_k) ~ Exp(xi) Exp(Jr(xi) h e_k)  (definition of the right Jacobian)
    xi = rand_se3(20)
    h = 1e-6
    for k in range(len(xi)):
        Jr = lie.se3_jr(xi[k])
        for a in range(6):
            e = np.zeros(6)
            e[a] = h
            d = (lie.se3_log(lie.se3_inv(lie.se3_exp(xi[k])) @ lie.se3_exp(xi[k] + e))
                 - lie.se3_log(lie.se3_inv(lie.se3_exp(xi[k])) @ lie.se3_exp(xi[k] - e))) / (2 * h)
            np.testing.assert_allclose(d, Jr[:, a], atol=1e-8)


def test_small_angle_branch_continuity():
    # values on both sides of every switch point agree
    for sw in [0.5, 1.0]:
        lo, hi = np.nextafter(sw, 0.0), np.float64(sw)   # series side / closed-form side
        for f in FN.values():
            assert abs(f(lo) - f(hi)) < 1e-14


# ---------------------------------------------------------------- SE2
def test_se2_hand_inverse():
    # SPEC.md:139  SE2 inverse of (theta=pi/2, t=(1,0)) -> (theta=-pi/2, t=(0,1))
    T = lie.se2_from(math.pi / 2, np.array([1.0, 0.0]))
    Ti = lie.se2_inv(T)
    np.testing.assert_allclose(Ti, lie.se2_from(-math.pi / 2, np.array([0.0, 1.0])), atol=1e-15)


def test_se2_exp_vs_expm_and_log_roundtrip():
    xi = rng.standard_normal((300, 3))
    xi[:, 2] = np.clip(xi[:, 2], -3.0, 3.0)
    T = lie.se2_exp(xi)
    for k in range(len(xi)):
        np.testing.assert_allclose(T[k], expm(lie.se2_hat(xi[k])), atol=1e-13)
    np.testing.assert_allclose(lie.se2_log(T), xi, atol=1e-12)


def test_so2_local_hand_value():
    # SPEC.md:157  SO2 local(rot(0.3), rot(0.8)) = 0.5
    A = lie.se2_from(0.3, np.zeros(2))
    B = lie.se2_from(0.8, np.zeros(2))
    np.testing.assert_allclose(lie.se2_log(lie.se2_inv(A) @ B), [0, 0, 0.5], atol=1e-15)


def test_se2_adjoint_identity():
    T = lie.se2_exp(rng.standard_normal((100, 3)))
    xi = rng.standard_normal((100, 3)) * 0.5
    lhs = T @ lie.se2_exp(xi) @ lie.se2_inv(T)
    rhs = lie.se2_exp(np.einsum("kab,kb->ka", lie.se2_adjoint(T), xi))
    np.testing.assert_allclose(lhs, rhs, atol=1e-12)


def test_se2_jr_closed_vs_series():
    for scale in [1e-8, 1e-3, 0.3, 0.7, 2.0, 3.0]:
        xi = rng.standard_normal((100, 3))
        xi[:, 2] = scale * np.sign(xi[:, 2])
        Js = lie.jr_series(lie.se2_ad(xi))
        np.testing.assert_allclose(lie.se2_jr(xi), Js, atol=1e-13)
        np.testing.assert_allclose(lie.se2_jr_inv(xi), np.linalg.inv(Js), atol=1e-12)


def test_se2_ad_is_commutator():
    a, b = rng.standard_normal(3), rng.standard_normal(3)
    A, Bm = lie.se2_hat(a), lie.se2_hat(b)
    C = A @ Bm - Bm @ A
    np.testing.assert_allclose(lie.se2_ad(a) @ b, [C[0, 2], C[1, 2], C[1, 0]], atol=1e-14)


def test_se3_ad_is_commutator():
    a, b = rand_se3(1)[0], rand_se3(1)[0]
    A, Bm = lie.se3_hat(a), lie.se3_hat(b)
    C = A @ Bm - Bm @ A
    ref = np.array([C[0, 3], C[1, 3], C[2, 3], C[2, 1], C[0, 2], C[1, 0]])
    np.testing.assert_allclose(lie.se3_ad(a) @ b, ref, atol=1e-14)
