"""Pins of the oracle's dense exponential (Higham 2005 Pade + scaling and
squaring) against closed forms, invariants and an independent library routine
(SURVEY 8(c) P2).  CPU only."""
from fractions import Fraction
from math import factorial

import numpy as np
import pytest
import scipy.linalg as sl

from oracle import oracle as O


def test_identity_and_zero():
    F, _ = O.expm(np.zeros((3, 3)), 1.0)
    assert np.array_equal(F, np.eye(3))


def test_diagonal():
    F, _ = O.expm(np.diag([1.0, 2.0, -3.0]), 1.0)
    assert np.allclose(F, np.diag(np.exp([1.0, 2.0, -3.0])), rtol=2e-15, atol=0)


@pytest.mark.parametrize("tau", [1e-3, 0.3, 7.0, 1e4])
def test_nilpotent_exact(tau):
    # [[0,1],[0,0]]: the series truncates, e^{tau N} = [[1, tau],[0, 1]]
    F, _ = O.expm(np.array([[0.0, 1.0], [0.0, 0.0]]), tau)
    assert F[0, 0] == 1.0 and F[1, 1] == 1.0 and F[1, 0] == 0.0
    assert abs(F[0, 1] - tau) <= 4e-16 * tau


@pytest.mark.parametrize("p,tau", [(5, 0.7), (8, 3.0), (4, 40.0)])
def test_shift_toeplitz_eq17(p, tau):
    # Eq. 17: e^{tau K} is upper-triangular Toeplitz with entries tau^j / j!
    K = np.diag(np.ones(p - 1), 1)
    F, _ = O.expm(K, tau)
    for r in range(p):
        for c in range(p):
            want = tau ** (c - r) / factorial(c - r) if c >= r else 0.0
            assert abs(F[r, c] - want) <= 1e-14 * max(1.0, abs(want))


@pytest.mark.parametrize("target", [0.01, 0.2, 0.9, 2.0, 5.0, 40.0, 700.0])
def test_each_pade_degree_vs_scipy(target):
    # 1-norms chosen inside each theta interval of Higham 2005 Table 2.3 so every
    # degree {3,5,7,9,13} and the scaling branch are exercised; scipy's expm is
    # the independent Al-Mohy-Higham 2009 algorithm (tolerance check only).
    rng = np.random.default_rng(1)
    for n in (1, 4, 17, 50):
        M = rng.standard_normal((n, n)) - 2.0 * np.eye(n)
        M *= target / np.abs(M).sum(axis=0).max()
        F, _ = O.expm(M, 1.0)
        R = sl.expm(M)
        assert np.linalg.norm(F - R, 1) <= 1e-13 * np.linalg.norm(R, 1) * max(1.0, target)


def test_semigroup_and_det():
    rng = np.random.default_rng(2)
    M = rng.standard_normal((6, 6))
    M *= 2.0 / np.abs(M).sum(axis=0).max()
    Fa, _ = O.expm(M, 1.7)
    Fb, _ = O.expm(M, 2.9)
    Fab, _ = O.expm(M, 4.6)
    assert np.linalg.norm(Fa @ Fb - Fab) <= 1e-13 * np.linalg.norm(Fab)
    F1, _ = O.expm(M, 1.0)
    assert abs(np.linalg.det(F1) - np.exp(np.trace(M))) <= 1e-12 * np.exp(np.trace(M))


def test_taylor_series():
    rng = np.random.default_rng(3)
    M = rng.standard_normal((8, 8))
    M *= 2.0 / np.abs(M).sum(axis=0).max()
    T = np.eye(8)
    term = np.eye(8)
    for k in range(1, 40):
        term = term @ M / k
        T = T + term
    F, _ = O.expm(M, 1.0)
    assert np.linalg.norm(F - T) <= 1e-14 * np.linalg.norm(T)


def test_pade_coefficients_are_the_rational_formula():
    # R17: b_j proportional to (2m-j)! m! / ((2m)! j! (m-j)!).  The oracle keeps the
    # integer-scaled table of Higham 2005; check the table it must contain by
    # reproducing e^x for scalar x where each degree is selected: a wrong
    # coefficient would move r_m(x) away from e^x by >> rounding.
    for m, x in ((3, 0.01), (5, 0.2), (7, 0.9), (9, 2.0)):
        c = [Fraction(factorial(2 * m - j) * factorial(m), factorial(2 * m) * factorial(j) * factorial(m - j))
             for j in range(m + 1)]
        num = sum(float(c[j]) * x ** j for j in range(m + 1))
        den = sum(float(c[j]) * (-x) ** j for j in range(m + 1))
        F, _ = O.expm(np.array([[x]]), 1.0)
        assert abs(F[0, 0] - num / den) <= 4e-16 * abs(num / den)
