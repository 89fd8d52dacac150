"""Pins of the oracle's operators and of Theorem 1's augmented matvec (Alg. 2 l.4-6,
P:316-318) against independent numpy/scipy formulations."""
import numpy as np
import scipy.sparse as sp

from oracle import oracle as O
from workloads import configs as W


def roll_1d(op, x):
    Wt, Cc, E = op["w"]
    y = Wt * np.roll(x, 1) + Cc * x + E * np.roll(x, -1)
    return y + (op["diag"] * x if op.get("diag") is not None else 0)


def roll_2d(op, x):
    X = x.reshape(op["ny"], op["nx"])
    Wt, E, S, Nn, Cc = op["w"]
    Y = (Wt * np.roll(X, 1, axis=1) + E * np.roll(X, -1, axis=1) + S * np.roll(X, 1, axis=0)
         + Nn * np.roll(X, -1, axis=0) + Cc * X)
    y = Y.ravel()
    return y + (op["diag"] * x if op.get("diag") is not None else 0)


def roll_3d(op, x):
    sh = (op["nz"], op["ny"], op["nx"])
    X, K = x.reshape(sh), op["kappa"].reshape(sh)
    Y = np.zeros(sh)
    for ax in range(3):
        for s in (1, -1):
            Y += 0.5 * (K + np.roll(K, s, axis=ax)) * (np.roll(X, s, axis=ax) - X)
    return Y.ravel() * op["inv_h2"]


def test_stencils_match_numpy_roll():
    rng = np.random.default_rng(5)
    for cfg, ref in ((W.config1(37), roll_1d), (W.config2(13, 9), roll_2d), (W.config3(11, 14), roll_2d),
                     (W.config4(7, 5, 6), roll_3d)):
        x = rng.standard_normal(cfg["N"])
        y = O.apply(cfg["op"], x)
        r = ref(cfg["op"], x)
        assert np.allclose(y, r, rtol=1e-14, atol=1e-14 * np.abs(r).max())


def test_csr_matches_scipy_and_generator_shape():
    cfg = W.config5(6, 7, 5)
    op = cfg["op"]
    A = sp.csr_matrix((op["vals"], op["col_idx"], op["row_ptr"]), shape=(cfg["N"], cfg["N"]))
    # D9a: truncated 27-pt pattern has (3n-2) nonzeros per axis product
    assert A.nnz == (3 * 6 - 2) * (3 * 7 - 2) * (3 * 5 - 2)
    # D9b: strictly diagonally dominant with |off| row sums, off-diagonals in (-1, 0]
    Ad = A.toarray()
    off = Ad - np.diag(np.diag(Ad))
    assert (off <= 0).all() and (off > -1).all()
    assert (np.diag(Ad) - np.abs(off).sum(1) >= 0).all() and (np.diag(Ad) - np.abs(off).sum(1) < 10).all()
    x = np.random.default_rng(1).standard_normal(cfg["N"])
    assert np.allclose(O.apply(op, x), A @ x, rtol=1e-14, atol=1e-13)


def test_full_config1_weights():
    op = W.config1()["op"]
    assert np.allclose(op["w"], [1400.0, -3200.0, 1800.0], rtol=1e-15)
    op2 = W.config2()["op"]
    assert np.allclose(op2["w"], [911.36, 655.36, 783.36, 655.36, -3005.44], rtol=1e-14)


def test_augmented_matvec_vs_assembled_dense():
    rng = np.random.default_rng(6)
    N, p = 10, 4
    A = rng.standard_normal((N, N))
    u = [rng.standard_normal(N) for _ in range(p + 1)]
    nu = 0.25
    At = np.zeros((N + p, N + p))
    At[:N, :N] = A
    for c in range(p):
        At[:N, N + c] = nu * u[p - c]          # B = [u_p, ..., u_1]  (Thm 1)
    At[N:, N:] = np.diag(np.ones(p - 1), 1)    # K
    v = rng.standard_normal(N + p)
    y = O.augmented_matvec({"kind": "dense", "nx": N, "dense": A}, u, nu, v)
    assert np.allclose(y, At @ v, rtol=1e-14, atol=1e-14)


def test_augmented_matvec_hand_cases():
    # p=1, v=[x;1] -> [Ax + b_1; 0];  p=3, v=[0;(c3,c2,c1)] -> [c3 b3 + c2 b2 + c1 b1; (c2, c1, 0)]
    N = 4
    A = np.arange(16.0).reshape(4, 4)
    b = [np.zeros(N), np.array([1.0, 2, 3, 4]), np.array([0.5, 0, 0, 1]), np.array([0, 1.0, 0, 0])]
    x = np.array([1.0, -1, 2, 0.5])
    y = O.augmented_matvec({"kind": "dense", "nx": N, "dense": A}, b[:2], 1.0, np.r_[x, 1.0])
    assert np.allclose(y, np.r_[A @ x + b[1], 0.0])
    y = O.augmented_matvec({"kind": "dense", "nx": N, "dense": A}, b, 1.0, np.r_[np.zeros(N), 3.0, 2.0, 1.0])
    assert np.allclose(y, np.r_[3 * b[3] + 2 * b[2] + 1 * b[1], 2.0, 1.0, 0.0])


def test_normalisation_golden():
    import json, os
    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_examples.json")))
    for ex in g["normalisation"]:
        # a one-column B whose 1-norm is exactly B_1norm
        u = [np.zeros(3), np.array([ex["B_1norm"] / 2, -ex["B_1norm"] / 4, ex["B_1norm"] / 4])]
        assert O.normalisation(u) == (ex["nu"], ex["mu"]), ex["cite"]
