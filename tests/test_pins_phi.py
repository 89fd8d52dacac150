"""Pins for the scalar phi-function helper (tests/phiref.py) used by the closed-form
pins: mpmath quadrature of the Eq. 3 integral, phi_k(0) = 1/k!, the
recurrence phi_k(z) = z phi_{k+1}(z) + 1/k!, phi_1 = (e^z - 1)/z."""
from math import factorial

import mpmath as mp
import numpy as np
import pytest

from tests.phiref import phi

mp.mp.dps = 40


def phi_mp(k, z):
    z = mp.mpc(z)
    if k == 0:
        return mp.exp(z)
    f = lambda t: mp.exp(z * (1 - t)) * t ** (k - 1) / mp.factorial(k - 1)
    return mp.quad(f, [0, 0.25, 0.5, 0.75, 1])


ZS = [0.0, 1e-8, -0.3, 0.7, -0.999, -1.0, 1.5, -3.0, -25.0, -200.0, 2.0 + 3.0j, -10.0 + 4.0j,
      0.5j, -786.0]


@pytest.mark.parametrize("k", [0, 1, 2, 3, 4])
def test_phi_vs_mpmath(k):
    for z in ZS:
        ref = complex(phi_mp(k, z))
        got = complex(phi(k, np.array([z]))[0])
        assert abs(got - ref) <= 1e-14 * abs(ref) + 1e-300, (k, z, got, ref)


def test_phi_at_zero():
    for k in range(9):
        assert phi(k, np.array([0.0]))[0] == pytest.approx(1.0 / factorial(k), rel=1e-16)


def test_recurrence_and_phi1():
    z = np.array([-50.0, -2.0, -0.5, 0.3, 3.0, -1 + 2j])
    for k in range(6):
        lhs = phi(k, z)
        rhs = z * phi(k + 1, z) + 1.0 / factorial(k)
        assert np.allclose(lhs, rhs, rtol=1e-13, atol=1e-15)
    assert np.allclose(phi(1, z), (np.exp(z) - 1) / z, rtol=1e-13)
