"""Pins P3/P5: oracle cost Jacobians vs central finite differences
with the retraction, prior at target -> J = I,
coordinate independence of the Between cost, hand Cholesky / solve
examples, textbook vs LAPACK Cholesky, linear-solve backward hand
values and FD."""
import numpy as np
import pytest

from oracle import costs, lie, linalg

rng = np.random.default_rng(7)


def rand_pose(G, n, s=1.0):
    return G.exp(rng.standard_normal((n, G.d)) * s)


@pytest.mark.parametrize("G", [lie.SE3, lie.SE2])
def test_between_jacobians_fd(G):
    n = 100
    Ti, Tj = rand_pose(G, n), rand_pose(G, n)
    Z = G.inv(Ti) @ Tj @ G.exp(rng.standard_normal((n, G.d)) * 0.3)   # residual of moderate size
    c, Ci, Cj = costs.between(G, Ti, Tj, Z)
    h = 1e-6
    for a in range(G.d):
        e = np.zeros(G.d)
        e[a] = h
        ci_p, _, _ = costs.between(G, Ti @ G.exp(e), Tj, Z)
        ci_m, _, _ = costs.between(G, Ti @ G.exp(-e), Tj, Z)
        cj_p, _, _ = costs.between(G, Ti, Tj @ G.exp(e), Z)
        cj_m, _, _ = costs.between(G, Ti, Tj @ G.exp(-e), Z)
        fd_i = (ci_p - ci_m) / (2 * h)
        fd_j = (cj_p - cj_m) / (2 * h)
        np.testing.assert_allclose(Ci[:, :, a], fd_i, rtol=0, atol=1e-8 * (1 + np.abs(fd_i).max()))
        np.testing.assert_allclose(Cj[:, :, a], fd_j, rtol=0, atol=1e-8 * (1 + np.abs(fd_j).max()))


@pytest.mark.parametrize("G", [lie.SE3, lie.SE2])
def test_prior_jacobian_fd_and_identity_at_target(G):
    T = rand_pose(G, 50)
    Z = T @ G.exp(rng.standard_normal((50, G.d)) * 0.4)
    c, C = costs.prior(G, T, Z)
    h = 1e-6
    for a in range(G.d):
        e = np.zeros(G.d)
        e[a] = h
        fd = (costs.prior(G, T @ G.exp(e), Z)[0] - costs.prior(G, T @ G.exp(-e), Z)[0]) / (2 * h)
        np.testing.assert_allclose(C[:, :, a], fd, atol=1e-8)
    c0, C0 = costs.prior(G, T, T)
    np.testing.assert_allclose(c0, 0, atol=1e-15)
    np.testing.assert_allclose(C0, np.broadcast_to(np.eye(G.d), C0.shape), atol=1e-15)


@pytest.mark.parametrize("G", [lie.SE3, lie.SE2])
def test_between_coordinate_independence(G):
    # left-composing both poses (and nothing else) by a fixed transform leaves c unchanged
    Ti, Tj = rand_pose(G, 30), rand_pose(G, 30)
    Z = rand_pose(G, 30, 0.3)
    Gt = rand_pose(G, 1)[0]
    c1, _, _ = costs.between(G, Ti, Tj, Z)
    c2, _, _ = costs.between(G, Gt @ Ti, Gt @ Tj, Z)
    np.testing.assert_allclose(c1, c2, atol=1e-12)


def test_objective_has_half_and_weights():
    G = lie.SE2
    T = rand_pose(G, 3)
    Z = G.inv(T[0]) @ T[1] @ G.exp(np.array([0.1, -0.2, 0.05]))
    edges = np.array([[0, 1]])
    c, _, _ = costs.between(G, T[:1], T[1:2], Z[None])
    S1 = costs.objective(G, T, edges, Z[None], np.array([1.0]), [], None, None)
    S2 = costs.objective(G, T, edges, Z[None], np.array([2.0]), [], None, None)
    assert abs(S1 - 0.5 * float(c[0] @ c[0])) < 1e-16
    assert abs(S2 - 4 * S1) < 1e-15            # SPEC.md weight linearity: doubling w quadruples


# ---------------------------------------------------------------- dense linear algebra
def test_cholesky_hand_examples():
    L, ok = linalg.cholesky(np.array([[4.0, 2.0], [2.0, 3.0]]))
    assert ok
    np.testing.assert_allclose(L, [[2, 0], [1, np.sqrt(2)]], atol=1e-15)
    L, ok = linalg.cholesky(np.eye(3))
    assert ok and np.array_equal(L, np.eye(3))
    _, ok = linalg.cholesky(np.array([[1.0, 2.0], [2.0, 1.0]]))         # SPEC.md:353 (pivot -3)
    assert not ok


def test_pivot_tolerance_rule():
    # a pivot <= 1e-13 * max diag fails even though it is positive
    A = np.diag([1.0, 1e-14])
    assert not linalg.cholesky(A)[1]
    assert linalg.cholesky(np.diag([1.0, 1e-12]))[1]


def test_solve_hand_example():
    L, _ = linalg.cholesky(np.array([[4.0, 2.0], [2.0, 3.0]]))
    np.testing.assert_allclose(linalg.chol_solve(L, np.array([8.0, 8.0])), [1, 2], atol=1e-15)


@pytest.mark.parametrize("n", [1, 5, 40, 300])
def test_textbook_cholesky_vs_lapack(n):
    M = rng.standard_normal((n, n))
    A = M @ M.T + n * np.eye(n)
    L, ok = linalg.cholesky(A)
    assert ok
    np.testing.assert_allclose(L, np.linalg.cholesky(A), rtol=0, atol=1e-12 * np.abs(L).max())
    b = rng.standard_normal(n)
    np.testing.assert_allclose(linalg.chol_solve(L, b), np.linalg.solve(A, b), rtol=1e-10, atol=1e-12)


def test_assemble_matches_explicit_jacobian():
    # H = J^T J, b = J^T r with the full stacked Jacobian built independently
    d, nv = 3, 4
    blocks = []
    Jfull, rfull = [], []
    for vids in [(0, 1), (1, 2), (2, 3), (0,), (3, 0)]:
        Js = [rng.standard_normal((d, d)) for _ in vids]
        r = rng.standard_normal(d)
        blocks.append((vids, Js, r))
        row = np.zeros((d, nv * d))
        for v, J in zip(vids, Js):
            row[:, v * d:(v + 1) * d] += J
        Jfull.append(row)
        rfull.append(r)
    Jf, rf = np.vstack(Jfull), np.concatenate(rfull)
    H, b = linalg.assemble(nv, d, blocks)
    np.testing.assert_allclose(H, Jf.T @ Jf, atol=1e-13)
    np.testing.assert_allclose(b, Jf.T @ rf, atol=1e-13)
    # SPEC.md:334 App. B: J=[-1,-2]^T, r=[2,4] -> H=[5], b=[-10]
    H, b = linalg.assemble(1, 1, [((0,), [np.array([[-1.0], [-2.0]])], np.array([2.0, 4.0]))])
    assert H[0, 0] == 5.0 and b[0] == -10.0
    np.testing.assert_allclose(linalg.damp(H, 1.0), [[10.0]])


def test_linear_solve_backward_hand_and_fd():
    # A = diag(2,4), b=(2,4) -> y=(1,1); f = y1+y2
    A = np.diag([2.0, 4.0])
    y = np.linalg.solve(A, np.array([2.0, 4.0]))
    gb, gA = linalg.linear_solve_backward(A, y, np.ones(2))
    np.testing.assert_allclose(gb, [0.5, 0.25])
    np.testing.assert_allclose(gA, [[-0.5, -0.5], [-0.25, -0.25]])
    # FD on a random system, f(y) = c . y
    n = 5
    M = rng.standard_normal((n, n))
    A = M @ M.T + n * np.eye(n)
    bb = rng.standard_normal(n)
    cvec = rng.standard_normal(n)
    y = np.linalg.solve(A, bb)
    gb, gA = linalg.linear_solve_backward(A, y, cvec)
    h = 1e-6
    for i in range(n):
        e = np.zeros(n)
        e[i] = h
        fd = (cvec @ np.linalg.solve(A, bb + e) - cvec @ np.linalg.solve(A, bb - e)) / (2 * h)
        assert abs(fd - gb[i]) < 1e-6 * max(1, abs(fd))
        for j in range(n):
            E = np.zeros((n, n))
            E[i, j] = h
            fd = (cvec @ np.linalg.solve(A + E, bb) - cvec @ np.linalg.solve(A - E, bb)) / (2 * h)
            assert abs(fd - gA[i, j]) < 1e-6 * max(1, abs(fd))
