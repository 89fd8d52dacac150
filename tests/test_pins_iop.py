"""Pins of the oracle's Alg. 2 (IOP): the Eq. 30 factorization, local
orthogonality, Theorem 2 (Eq. 31), Lanczos reduction for symmetric A, breakdown
and the canonical shift chain."""
import numpy as np
import pytest

from oracle import oracle as O


def aug_dense(A, u, nu):
    N, p = A.shape[0], len(u) - 1
    At = np.zeros((N + p, N + p))
    At[:N, :N] = A
    for c in range(p):
        At[:N, N + c] = nu * u[p - c]
    if p:
        At[N:, N:] = np.diag(np.ones(p - 1), 1)
    return At


def rand_case(seed, N=60, p=2, scale=1.0):
    rng = np.random.default_rng(seed)
    A = rng.standard_normal((N, N)) * scale / np.sqrt(N) - 0.5 * np.eye(N)
    u = [rng.standard_normal(N) for _ in range(p + 1)]
    return A, u


@pytest.mark.parametrize("seed,p,q", [(0, 0, 2), (1, 2, 2), (2, 4, 2), (3, 2, 1), (4, 3, 5)])
def test_eq30_factorization(seed, p, q):
    A, u = rand_case(seed, p=p)
    nu = 0.5
    m = 25
    v0 = np.r_[u[0], np.ones(p)] if p else u[0]
    V, H, j, happy = O.iop({"kind": "dense", "nx": len(u[0]), "dense": A}, u, nu, v0, m, q)
    assert j == m and not happy
    At = aug_dense(A, u, nu)
    R = At @ V[:, :m] - V[:, :m] @ H[:m, :m]
    R[:, m - 1] -= H[m, m - 1] * V[:, m]
    assert np.linalg.norm(R) <= 1e-12 * np.linalg.norm(At @ V[:, :m])
    # every column unit norm; H banded: H(i, j) = 0 for i < j - q + 1
    assert np.allclose(np.linalg.norm(V[:, : m + 1], axis=0), 1.0, atol=1e-13)
    for jj in range(m):
        for i in range(0, max(0, jj - q + 1)):
            assert H[i, jj] == 0.0
    # local orthogonality within the window
    for jj in range(1, m + 1):
        for i in range(max(0, jj - q), jj):
            assert abs(V[:, i] @ V[:, jj]) <= 1e-10


def test_theorem2_polynomial_reproduction():
    A, u = rand_case(7, p=2)
    nu, m = 0.5, 10
    v0 = np.r_[u[0], 0.3, 1.0]
    V, H, j, _ = O.iop({"kind": "dense", "nx": len(u[0]), "dense": A}, u, nu, v0, m, 2)
    At = aug_dense(A, u, nu)
    beta = np.linalg.norm(v0)
    x = v0.copy()
    Hm = H[:m, :m]
    Pe = np.eye(m)[:, 0]
    for i in range(m - 1):   # Eq. 31, j < m - 1
        assert np.linalg.norm(x - beta * V[:, :m] @ Pe) <= 1e-9 * np.linalg.norm(x)
        x = At @ x
        Pe = Hm @ Pe


def test_symmetric_tridiagonal_is_lanczos():
    rng = np.random.default_rng(8)
    N = 80
    d = -np.linspace(0.1, 4.0, N)
    A = np.diag(d) + np.diag(0.3 * np.ones(N - 1), 1) + np.diag(0.3 * np.ones(N - 1), -1)
    V, H, j, _ = O.iop({"kind": "dense", "nx": N, "dense": A}, [rng.standard_normal(N)], 1.0,
                       rng.standard_normal(N), 10, 2)
    assert np.allclose(V[:, :11].T @ V[:, :11], np.eye(11), atol=1e-12)
    Hm = H[:10, :10]
    assert np.allclose(Hm, Hm.T, atol=1e-12)
    assert np.allclose(np.triu(Hm, 2), 0) and np.allclose(np.tril(Hm, -2), 0)


def test_identity_breaks_down_at_once():
    N = 12
    V, H, j, happy = O.iop({"kind": "dense", "nx": N, "dense": np.eye(N)}, [np.ones(N)], 1.0,
                           np.arange(1.0, N + 1), 5, 2)
    assert happy == 1 and j == 1 and H[0, 0] == pytest.approx(1.0, rel=1e-15)


def test_shift_chain():
    # A = shift (A e_i = e_{i+1}), v = e_1, m = 3 -> V = [e1, e2, e3], H subdiagonal ones
    N = 8
    A = np.diag(np.ones(N - 1), -1)
    e1 = np.eye(N)[:, 0]
    V, H, j, happy = O.iop({"kind": "dense", "nx": N, "dense": A}, [e1], 1.0, e1, 3, 2)
    assert j == 3 and not happy
    assert np.array_equal(V[:, :4], np.eye(N)[:, :4])
    assert np.array_equal(H[:4, :3], np.diag(np.ones(3), -1)[:4, :3])


def test_full_window_is_arnoldi():
    A, u = rand_case(9, p=1)
    V, H, j, _ = O.iop({"kind": "dense", "nx": len(u[0]), "dense": A}, u, 1.0, np.r_[u[0], 1.0], 15, 15)
    assert np.allclose(V[:, :16].T @ V[:, :16], np.eye(16), atol=1e-12)
