"""Golden worked examples (tests/golden/spec_worked_examples.json, each entry cites SPEC.md)
checked against the oracle."""
import json
import os

import numpy as np

from oracle import lie, linalg, nls

G = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_worked_examples.json")))


def test_golden_linear_algebra():
    L, ok = linalg.cholesky(np.array(G["cholesky_2x2"]["H"], float))
    assert ok
    np.testing.assert_allclose(L, G["cholesky_2x2"]["L"], atol=1e-15)
    assert linalg.cholesky(np.array(G["cholesky_fail"]["H"], float))[1] == G["cholesky_fail"]["ok"]
    L, _ = linalg.cholesky(np.array(G["solve_2x2"]["H"], float))
    np.testing.assert_allclose(linalg.chol_solve(L, np.array(G["solve_2x2"]["b"], float)), G["solve_2x2"]["x"], atol=1e-15)
    e = G["linsolve_backward"]
    A = np.array(e["A"], float)
    y = np.linalg.solve(A, np.array(e["b"], float))
    gb, gA = linalg.linear_solve_backward(A, y, np.array(e["gy"], float))
    np.testing.assert_allclose(gb, e["gb"])
    np.testing.assert_allclose(gA, e["gA"])


def test_golden_appb():
    e = G["appb_residual"]
    x, y = np.array(e["x"]), np.array(e["y"], float)
    prob = nls.EuclidProblem(1, 1, lambda v: y - v[0, 0] * np.exp(x), lambda v: -np.exp(x)[:, None])
    v0 = np.full((1, 1), e["v"])
    np.testing.assert_allclose(prob.residual(v0), e["r"], atol=1e-15)
    S, H, b = prob.linearize(v0)
    assert abs(S - e["S"]) < 1e-14 and abs(H[0, 0] - G["appb_system"]["H"]) < 1e-14 and abs(b[0] - G["appb_system"]["b"]) < 1e-14
    r = nls.gauss_newton(prob, v0, nls.Options(max_iterations=1))
    assert abs(r.x[0, 0] - G["appb_gn_step"]["v1"]) < 1e-15
    lm = G["appb_lm_step"]
    r = nls.levenberg_marquardt(prob, v0, nls.Options(optimizer="lm", max_iterations=1, lambda0=lm["lambda"]))
    assert abs(r.x[0, 0] - lm["v1"]) < 1e-15 and abs(r.objective - lm["S1"]) < 1e-14 and abs(r.lam - lm["lambda1"]) < 1e-16


def test_golden_lie():
    e = G["so3_exp"]
    np.testing.assert_allclose(lie.so3_exp(np.array(e["w"])), e["R"], atol=1e-15)
    e = G["se2_inverse"]
    Ti = lie.se2_inv(lie.se2_from(e["theta"], np.array(e["t"], float)))
    np.testing.assert_allclose(Ti, lie.se2_from(e["theta_inv"], np.array(e["t_inv"], float)), atol=1e-15)
