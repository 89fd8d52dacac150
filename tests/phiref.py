"""Closed-form helpers used by the pins (tests only; independent of oracle/ and of
the CUDA path).

phi(k, z): scalar phi-functions of Eq. 3, phi_k(z) = int_0^1
e^{z(1-t)} t^{k-1}/(k-1)! dt, phi_0 = e^z, for complex arrays z.  Series
sum_i z^i/(i+k)! for |z| < 1, else the recurrence phi_{k+1}(z) = (phi_k(z) -
1/k!)/z (which follows from Eq. 3 by integration by parts).  Pinned against an
mpmath quadrature of the Eq. 3 integral in test_pins_phi.py.

circulant_phi_combination: w = IFFT(sum_k tau^k phi_k(tau lambda) FFT(u_k)) for a
periodic constant-coefficient stencil with Fourier symbol lambda.
"""
from math import factorial

import numpy as np


def phi(k, z):
    z = np.asarray(z, dtype=np.complex128)
    out = np.empty_like(z)
    small = np.abs(z) < 1.0
    if small.any():
        zs = z[small]
        s = np.zeros_like(zs)
        term = np.ones_like(zs) / factorial(k)
        for i in range(60):
            s = s + term
            term = term * zs / (i + k + 1)
        out[small] = s
    if (~small).any():
        zb = z[~small]
        f = np.exp(zb)
        for j in range(k):
            f = (f - 1.0 / factorial(j)) / zb
        out[~small] = f
    return out


def symbol_1d(w, n):
    th = 2 * np.pi * np.arange(n) / n
    W, Cc, E = w
    return W * np.exp(-1j * th) + Cc + E * np.exp(1j * th)


def symbol_2d(w, nx, ny, d=0.0):
    """array layout u[y, x]; numpy fft2 convention"""
    W, E, S, Nn, Cc = w
    tx = 2 * np.pi * np.arange(nx) / nx
    ty = 2 * np.pi * np.arange(ny) / ny
    lx = W * np.exp(-1j * tx) + E * np.exp(1j * tx)
    ly = S * np.exp(-1j * ty) + Nn * np.exp(1j * ty)
    return ly[:, None] + lx[None, :] + Cc + d


def symbol_3d_const_kappa(nx, ny, nz, inv_h2):
    t = [2 * np.pi * np.arange(n) / n for n in (nx, ny, nz)]
    cx, cy, cz = (2 * np.cos(a) - 2 for a in t)
    return (cz[:, None, None] + cy[None, :, None] + cx[None, None, :]) * inv_h2


def circulant_phi_combination(lam, u_list, tau, shape):
    acc = np.zeros(shape, dtype=np.complex128)
    for k, u in enumerate(u_list):
        if not np.any(u):
            continue
        U = np.fft.fftn(np.asarray(u).reshape(shape))
        acc += (tau ** k) * phi(k, tau * lam) * U
    return np.real(np.fft.ifftn(acc)).ravel()
