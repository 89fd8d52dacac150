"""Seeded synthetic inputs for the five BASELINE.json configs.

This module holds NO arithmetic of the KIOPS method: it only draws random
fields and writes operator coefficients from the configs' PDE recipes.  It is
the one piece shared by the oracle side (tests, bench cpu_baseline) and the CUDA
side (tests, bench, smoke).  Generation recipe = SURVEY.md 8(d) readings D1-D9:

* unit periodic domain, h = 1/n (D1, D2); lexicographic index i = x + nx*y + nx*ny*z;
* numpy default_rng(seed) (PCG64); draw order: operator random fields first,
  then u_0..u_p (standard_normal, float64); a u_k that is 0 by definition is not drawn;
* smoothed fields: white N(0,1) on the grid, periodic Gaussian blur by FFT
  (multiply by exp(-2 pi^2 sigma^2 |k|^2 / n^2)), then re-standardised to mean 0
  and the target std (D4).

Every generator takes optional smaller grid sizes for parity tests.  By default
a reduced grid keeps the FULL config's stencil weights (its h), so the spectrum
(and therefore Krylov sizes, substeps, rejections) matches the full config.
"""
from __future__ import annotations

import numpy as np

FULL = {1: (400,), 2: (256, 256), 3: (1024, 1024), 4: (256, 256, 256), 5: (160, 160, 160)}


def _blur(rng, shape, sigma, std):
    """White noise -> periodic Gaussian blur (sigma in cells) -> mean 0, given std (D4)."""
    g = rng.standard_normal(shape)
    G = np.fft.fftn(g)
    mult = np.ones(shape)
    for ax, n in enumerate(shape):
        k = np.fft.fftfreq(n) * n
        sh = [1] * len(shape)
        sh[ax] = n
        mult = mult * np.exp(-2.0 * np.pi ** 2 * sigma ** 2 * (k.reshape(sh) ** 2) / n ** 2)
    b = np.real(np.fft.ifftn(G * mult))
    b = b - b.mean()
    return b * (std / b.std())


def _pack(op, u, T, tol, m_init=10, m_min=10, m_max=128, q=2, name=""):
    N = op["nx"] * op["ny"] * op["nz"]
    return {"name": name, "op": op, "u": u, "T": np.asarray(T, dtype=np.float64), "tol": tol,
            "m_init": m_init, "m_min": m_min, "m_max": m_max, "iop_q": q, "N": N, "p": len(u) - 1}


def config1(n=None, seed=0, n_full=400):
    """1D advection-diffusion, periodic, A = eps D2 + alpha D1 (centered), eps=1e-2,
    alpha=1; p=3, u_0..u_3 ~ N(0,1); tau=1e-2, tol=1e-8, m_init=10, q=2."""
    n = n or n_full
    h = 1.0 / n_full
    eps, alpha = 1e-2, 1.0
    w = [eps / h ** 2 - alpha / (2 * h), -2 * eps / h ** 2, eps / h ** 2 + alpha / (2 * h)]
    rng = np.random.default_rng(seed)
    u = [rng.standard_normal(n) for _ in range(4)]
    op = {"kind": "stencil1d3", "nx": n, "ny": 1, "nz": 1, "w": w, "diag": None}
    return _pack(op, u, [1e-2], 1e-8, name=f"c1_adv_diff_1d_n{n}")


def config2(nx=None, ny=None, seed=1, n_full=256):
    """2D ADR, periodic: 5-pt Laplacian eps=1e-2 + upwind advection (1, 0.5) (backward
    differences, D5) + diagonal reaction gamma(1-2v), v ~ U(0,1), gamma=10; p=1,
    u_0 = 0, u_1 ~ N(0,1); tau=1e-3, tol=1e-8, q=2."""
    nx = nx or n_full
    ny = ny or nx
    h = 1.0 / n_full
    e = 1e-2 / h ** 2
    ax, ay = 1.0 / h, 0.5 / h
    w = [e + ax, e, e + ay, e, -4 * e - ax - ay]  # W, E, S, N, C
    rng = np.random.default_rng(seed)
    v = rng.random((ny, nx)).ravel()
    diag = 10.0 * (1.0 - 2.0 * v)
    u1 = rng.standard_normal(nx * ny)
    op = {"kind": "stencil2d5", "nx": nx, "ny": ny, "nz": 1, "w": w, "diag": diag}
    return _pack(op, [np.zeros(nx * ny), u1], [1e-3], 1e-8, name=f"c2_adr_2d_{nx}x{ny}")


def config3(nx=None, ny=None, seed=2, n_full=1024):
    """2D Allen-Cahn Jacobian, periodic: eps Lap (5-pt, eps=1e-3) + diag(1 - 3 v^2),
    v = blur(sigma=8 cells) of N(0,1) re-standardised (D4); p=3, u_k ~ N(0,1);
    tau=5e-3, tol=1e-10, q=2."""
    nx = nx or n_full
    ny = ny or nx
    h = 1.0 / n_full
    e = 1e-3 / h ** 2
    w = [e, e, e, e, -4 * e]
    rng = np.random.default_rng(seed)
    v = _blur(rng, (ny, nx), 8.0, 1.0).ravel()
    diag = 1.0 - 3.0 * v ** 2
    u = [rng.standard_normal(nx * ny) for _ in range(4)]
    op = {"kind": "stencil2d5", "nx": nx, "ny": ny, "nz": 1, "w": w, "diag": diag}
    return _pack(op, u, [5e-3], 1e-10, name=f"c3_allen_cahn_2d_{nx}x{ny}")


def config4(nx=None, ny=None, nz=None, seed=3, n_full=256):
    """3D variable-coefficient diffusion, periodic 7-pt, face kappa = arithmetic mean
    (D6), kappa = exp(g), g = blur(sigma=8, D7) re-standardised to std 0.5 (D8);
    p=2, u_k ~ N(0,1); tau list {1e-4, 5e-4, 1e-3}, tol=1e-10, m_max=128, q=2."""
    nx = nx or n_full
    ny = ny or nx
    nz = nz or nx
    h = 1.0 / n_full
    rng = np.random.default_rng(seed)
    g = _blur(rng, (nz, ny, nx), 8.0, 0.5).ravel()
    kappa = np.exp(g)
    N = nx * ny * nz
    u = [rng.standard_normal(N) for _ in range(3)]
    op = {"kind": "stencil3d7", "nx": nx, "ny": ny, "nz": nz, "kappa": kappa,
          "inv_h2": 1.0 / h ** 2, "diag": None}
    return _pack(op, u, [1e-4, 5e-4, 1e-3], 1e-10, m_max=128, name=f"c4_varkappa_3d_{nx}x{ny}x{nz}")


def csr_27pt(nx, ny, nz, rng):
    """27-point pattern {-1,0,1}^3 truncated at the grid boundary (D9a); rows in
    lexicographic order, ascending columns.  Off-diagonals -U(0,1) drawn in CSR
    order (diagonal skipped); then one U(0,10) per row; diagonal = sum |off| +
    that draw (D9b)."""
    N = nx * ny * nz
    idx = np.arange(N, dtype=np.int64)
    x, y, z = idx % nx, (idx // nx) % ny, idx // (nx * ny)
    offs = [(dx, dy, dz) for dz in (-1, 0, 1) for dy in (-1, 0, 1) for dx in (-1, 0, 1)]
    cols = np.empty((N, 27), dtype=np.int32)
    valid = np.empty((N, 27), dtype=bool)
    for k, (dx, dy, dz) in enumerate(offs):  # ascending column order within a row
        ok = (x + dx >= 0) & (x + dx < nx) & (y + dy >= 0) & (y + dy < ny) & (z + dz >= 0) & (z + dz < nz)
        valid[:, k] = ok
        cols[:, k] = (idx + dx + nx * dy + nx * ny * dz).astype(np.int32)
    counts = valid.sum(axis=1)
    row_ptr = np.zeros(N + 1, dtype=np.int64)
    np.cumsum(counts, out=row_ptr[1:])
    col_idx = cols[valid]
    del cols
    is_diag = np.zeros((N, 27), dtype=bool)
    is_diag[:, 13] = True
    diag_pos = is_diag[valid]
    del is_diag, valid
    nnz = int(row_ptr[-1])
    vals = np.empty(nnz)
    off = -rng.random(nnz - N)
    vals[~diag_pos] = off
    rows = np.repeat(idx, counts)
    offsum = np.bincount(rows[~diag_pos], weights=-off, minlength=N)
    extra = rng.uniform(0.0, 10.0, N)
    vals[diag_pos] = offsum + extra
    return row_ptr, col_idx, vals


def config5(nx=None, ny=None, nz=None, seed=4, n_full=160):
    """General CSR: 27-pt pattern on 160^3 (4.1M rows, nnz = 478^3), off-diagonal
    -U(0,1), diagonal = |off| row sum + U(0,10); p=4, u_k ~ N(0,1); tau=1e-2,
    tol=1e-9, q=2."""
    nx = nx or n_full
    ny = ny or nx
    nz = nz or nx
    rng = np.random.default_rng(seed)
    row_ptr, col_idx, vals = csr_27pt(nx, ny, nz, rng)
    N = nx * ny * nz
    u = [rng.standard_normal(N) for _ in range(5)]
    op = {"kind": "csr", "nx": N, "ny": 1, "nz": 1, "row_ptr": row_ptr, "col_idx": col_idx,
          "vals": vals, "diag": None, "grid": (nx, ny, nz)}
    return _pack(op, u, [1e-2], 1e-9, name=f"c5_csr27_{nx}x{ny}x{nz}")


MAKERS = {1: config1, 2: config2, 3: config3, 4: config4, 5: config5}


def make(idx: int, *dims, **kw):
    return MAKERS[idx](*dims, **kw)


def algorithmic_bytes_per_pass(cfg) -> int:
    """Minimum HBM bytes per Krylov vector: read the operator
    coefficients once, the q-window (2 vectors), B's p vectors, write one vector:
    (q + 1 + p + c) * 8N, plus CSR matrix bytes (12 per nnz + 8 (N+1))."""
    op, N, p, q = cfg["op"], cfg["N"], cfg["p"], cfg["iop_q"]
    c = 0
    if op.get("diag") is not None:
        c += 1
    if op["kind"] == "stencil3d7":
        c += 1
    b = (q + 1 + p + c) * 8 * N
    if op["kind"] == "csr":
        b += 12 * len(op["vals"]) + 8 * (N + 1)
    return b
