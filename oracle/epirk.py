"""EPIRK exponential integrators on top of the oracle's KIOPS.

TEST INFRASTRUCTURE ONLY (same rule as oracle.py: only tests/, __graft_entry__.smoke()
and bench.py's reference legs import it; the product package never does).

What it follows, step by step:
  * the three-stage EPIRK template, Eq. 2 (Sec. 2), with the nonlinear
    remainder r(u) = f(u) - f(u_n) - J_n (u - u_n);
  * EPIRK4s3, Eq. 50 (= Eq. 9) and EPIRK4s3A, Eq. 51;
  * the "mixed implementation" grouping of Sec. 2 (Eqs. 10-11): call 1 is a
    Task-I KIOPS call, phi_1 at the two stage nodes T = [c_a, c_b] on b = h f(u_n) with
    the 1/T^p scaling (Alg. 1 l.31-35); call 2 is a Task-II call at tau = 1 with
    b_1 = h f(u_n), b_2 = 0 and b_3, b_4 written exactly as Eq. 11 prints them (for
    EPIRK4s3A: read off Eq. 51 the same way);
  * constant step size (Sec. 4: "implemented with constant time step
    integration"); KIOPS's m warm-started from the previous step's final m of the same
    call (Sec. 3.6 heuristic, reading E1 in DESIGN.md).
The problems (Sec. 4): the 1D semilinear parabolic problem made autonomous
by appending t to the state (reading E2), with the source discretised so that the
semi-discrete system has the exact solution x(1-x)e^t (reading E3); and a periodic
Allen-Cahn 2D problem (periodic instead of no-flow boundaries: reading E4).
"""
from __future__ import annotations

import numpy as np

from oracle import oracle as O

# Eq. 50 / Eq. 51: stage nodes (U_{n2}, U_{n3}) and the final-stage combination
SCHEMES = ("epirk4s3", "epirk4s3a")
NODES = {"epirk4s3": (1.0 / 8.0, 1.0 / 9.0), "epirk4s3a": (1.0 / 2.0, 2.0 / 3.0)}
# fifth-order schemes, three KIOPS calls per step (Sec. 4)
SCHEMES5 = ("epirk5p1", "exprb5s3")
# Table 1, EPIRK5P1 coefficients as printed
A11, A21, A22 = 0.3512959269505819, 0.8440547201165712, 1.690589160956896
B1, B2, B3 = 1.0, 1.272712731735689, 2.271459926542262
G11, G21, G22 = 0.3512959269505819, 0.8440547201165712, 1.0
G31, G32, G33 = 1.0, 0.71111109536436687, 0.6237811195337149


def final_b34(scheme, h, r2, r3):
    """b_3, b_4 of the Task-II call (Eq. 11 for EPIRK4s3; Eq. 51 for EPIRK4s3A), as printed."""
    if scheme == "epirk4s3":
        d = r3 - 2.0 * r2
        b3 = 1892.0 * h * r2 + 1458.0 * h * d
        b4 = -42336.0 * h * r2 - 34992.0 * h * d
    elif scheme == "epirk4s3a":
        b3 = 32.0 * h * r2 - 13.5 * h * r3
        b4 = -144.0 * h * r2 + 81.0 * h * r3
    else:
        raise ValueError(scheme)
    return b3, b4


# ---------------------------------------------------------------------------
# problems: f(y), J(y) as a KIOPS operator dict scaled by h, and J(y) x
# ---------------------------------------------------------------------------
class Semilinear1D:
    """U_t - U_xx = int_0^1 U dx + Phi(x, t) on (0, 1), U = 0 at x = 0, 1.
    Interior nodes x_i = i dx, dx = 1/(N+1); U_xx by the 3-point difference; the
    integral by the trapezoid rule with the zero boundary values, dx sum_j U_j.
    Phi_i(t) = e^t (x_i(1-x_i) + 2 - Q), Q = dx sum_j x_j(1-x_j): then
    u_i(t) = x_i(1-x_i) e^t solves the semi-discrete system exactly (reading E3).
    State y = (u_1..u_N, t) (autonomous form, reading E2)."""

    def __init__(self, N=200):
        self.N = N
        self.dim = N + 1
        dx = 1.0 / (N + 1)
        self.x = dx * np.arange(1, N + 1)
        A = np.zeros((N, N))
        i = np.arange(N)
        A[i, i] = -2.0 / dx ** 2
        A[i[1:], i[:-1]] = 1.0 / dx ** 2
        A[i[:-1], i[1:]] = 1.0 / dx ** 2
        A += dx  # quadrature row: every row gets dx * sum_j u_j
        self.A = A
        self.g = self.x * (1.0 - self.x) + 2.0 - dx * np.sum(self.x * (1.0 - self.x))

    def exact(self, t):
        return np.r_[self.x * (1.0 - self.x) * np.exp(t), t]

    def f(self, y):
        u, t = y[:-1], y[-1]
        return np.r_[self.A @ u + np.exp(t) * self.g, 1.0]

    def jac_dense(self, y):
        t = y[-1]
        J = np.zeros((self.dim, self.dim))
        J[:-1, :-1] = self.A
        J[:-1, -1] = np.exp(t) * self.g  # d Phi / dt
        return J

    def jmul(self, y, x):
        return self.jac_dense(y) @ x

    def kiops_op(self, y, h):
        return {"kind": "dense", "nx": self.dim, "ny": 1, "nz": 1, "dense": h * self.jac_dense(y)}


class ReactionDiffusion2D:
    """u_t = alpha lap(u) + R(u), R(u) = c0 + c1 u + c2 u^2 + c3 u^3, periodic n x n
    grid of spacing dx (5-point Laplacian).  Allen-Cahn: alpha = 0.1,
    R = u - u^3 on [-1, 1]^2 (dx = 2/n), u_0 = 0.1 + 0.1 cos(2 pi x) cos(2 pi y);
    periodic boundaries (reading E4).  J(u) = alpha lap + diag(R'(u))."""

    def __init__(self, n=64, ny=None, alpha=0.1, coef=(0.0, 1.0, 0.0, -1.0), length=2.0):
        self.nx, self.ny = n, (ny or n)
        self.dim = self.nx * self.ny
        self.dx = length / self.nx
        self.alpha = alpha
        self.c = tuple(float(c) for c in coef)
        self.wa = alpha / self.dx ** 2

    def initial(self):
        xs = -1.0 + self.dx * np.arange(self.nx)
        ys = -1.0 + self.dx * np.arange(self.ny)
        X, Y = np.meshgrid(xs, ys, indexing="xy")
        return (0.1 + 0.1 * np.cos(2 * np.pi * X) * np.cos(2 * np.pi * Y)).ravel()

    def lap(self, u):
        U = u.reshape(self.ny, self.nx)
        L = np.roll(U, 1, 1) + np.roll(U, -1, 1) + np.roll(U, 1, 0) + np.roll(U, -1, 0) - 4.0 * U
        return self.wa * L.ravel()

    def R(self, u):
        c0, c1, c2, c3 = self.c
        return c0 + u * (c1 + u * (c2 + u * c3))

    def dR(self, u):
        _, c1, c2, c3 = self.c
        return c1 + u * (2.0 * c2 + u * 3.0 * c3)

    def f(self, y):
        return self.lap(y) + self.R(y)

    def jmul(self, y, x):
        return self.lap(x) + self.dR(y) * x

    def remainder(self, yn, y):
        """r(y) of P:85 for f = L u + R(u) with L linear: the L terms of
        f(y) - f(y_n) - J_n (y - y_n) cancel identically, leaving the pointwise
        R(y) - R(y_n) - R'(y_n)(y - y_n) (reading E7; no cancellation of large terms)."""
        return self.R(y) - self.R(yn) - self.dR(yn) * (y - yn)

    def kiops_op(self, y, h):
        wa = h * self.wa
        return {"kind": "stencil2d5", "nx": self.nx, "ny": self.ny, "nz": 1,
                "w": [wa, wa, wa, wa, -4.0 * wa], "diag": h * self.dR(y)}


class ReactionDiffusionCSR:
    """u' = L u + R(u) with a general constant linear part L (CSR: row_ptr, col_idx,
    vals; every row holds its diagonal entry) and the pointwise cubic R(u) = c0 + c1 u +
    c2 u^2 + c3 u^3.  J(u) = L + diag(R'(u)); the remainder of P:85 is pointwise as for
    ReactionDiffusion2D (reading E7).  Plain loops / numpy only."""

    def __init__(self, row_ptr, col_idx, vals, coef):
        self.row_ptr = np.asarray(row_ptr, dtype=np.int64)
        self.col_idx = np.asarray(col_idx, dtype=np.int32)
        self.vals = np.asarray(vals, dtype=np.float64)
        self.dim = len(self.row_ptr) - 1
        self.c = tuple(float(c) for c in coef)
        rows = np.repeat(np.arange(self.dim), np.diff(self.row_ptr))
        self._rows = rows
        self.diag_pos = np.full(self.dim, -1, dtype=np.int64)
        on = np.nonzero(self.col_idx == rows)[0]
        self.diag_pos[rows[on]] = on
        if np.any(self.diag_pos < 0):
            raise ValueError("every row of L must hold its diagonal entry")

    def lmul(self, u):
        out = np.zeros(self.dim)
        np.add.at(out, self._rows, self.vals * u[self.col_idx])  # row sums in storage order
        return out

    def R(self, u):
        c0, c1, c2, c3 = self.c
        return c0 + u * (c1 + u * (c2 + u * c3))

    def dR(self, u):
        _, c1, c2, c3 = self.c
        return c1 + u * (2.0 * c2 + u * 3.0 * c3)

    def f(self, y):
        return self.lmul(y) + self.R(y)

    def jmul(self, y, x):
        return self.lmul(x) + self.dR(y) * x

    def remainder(self, yn, y):
        return self.R(y) - self.R(yn) - self.dR(yn) * (y - yn)

    def kiops_op(self, y, h):
        v = self.vals.copy()
        v[self.diag_pos] += self.dR(y)
        return {"kind": "csr", "nx": self.dim, "ny": 1, "nz": 1, "row_ptr": self.row_ptr,
                "col_idx": self.col_idx, "vals": h * v}


def adr_neumann(nx, ny=None, eps=0.01, alpha=-10.0, gamma=100.0):
    """The ADR 2D problem of Sec. 4: u_t = eps lap(u) - alpha (u_x + u_y) +
    gamma u (u - 1/2)(1 - u) on [0, 1]^2 with homogeneous Neumann boundaries, u_0 =
    256 (x y (1-x)(1-y))^2 + 0.3.  Discretisation (reading E10): nodes x_i = i dx,
    i = 0..nx-1, dx = 1/(nx-1) (boundary nodes included), second-order central
    differences for both the Laplacian and the advection term, the Neumann condition by
    the mirrored ghost node u_{-1} = u_{1} (so the boundary Laplacian row is
    (2 u_1 - 2 u_0)/dx^2 and the central first difference vanishes there).  Returns
    (problem, u0); rows in lexicographic order (x fastest), ascending columns."""
    ny = ny or nx
    dx, dy = 1.0 / (nx - 1), 1.0 / (ny - 1)
    row_ptr, col, val = [0], [], []
    for j in range(ny):
        for i in range(nx):
            ent = {}

            def add(ii, jj, w):
                ii = -ii if ii < 0 else (2 * (nx - 1) - ii if ii > nx - 1 else ii)  # mirror
                jj = -jj if jj < 0 else (2 * (ny - 1) - jj if jj > ny - 1 else jj)
                k = ii + nx * jj
                ent[k] = ent.get(k, 0.0) + w

            add(i, j, -2.0 * eps / dx ** 2 - 2.0 * eps / dy ** 2)
            add(i - 1, j, eps / dx ** 2 + alpha / (2.0 * dx))
            add(i + 1, j, eps / dx ** 2 - alpha / (2.0 * dx))
            add(i, j - 1, eps / dy ** 2 + alpha / (2.0 * dy))
            add(i, j + 1, eps / dy ** 2 - alpha / (2.0 * dy))
            for k in sorted(ent):
                col.append(k)
                val.append(ent[k])
            row_ptr.append(len(col))
    prob = ReactionDiffusionCSR(row_ptr, col, val, (0.0, -0.5 * gamma, 1.5 * gamma, -gamma))
    prob.nx, prob.ny = nx, ny
    xs, ys = dx * np.arange(nx), dy * np.arange(ny)
    X, Y = np.meshgrid(xs, ys, indexing="xy")
    u0 = (256.0 * (X * Y * (1.0 - X) * (1.0 - Y)) ** 2 + 0.3).ravel()
    return prob, u0


def allen_cahn_noflow(nx, ny=None, alpha=0.1):
    """Allen-Cahn 2D as printed: u_t = alpha lap(u) + u - u^3 on [-1, 1]^2 with
    NO-FLOW (homogeneous Neumann) boundaries, u_0 = 0.1 + 0.1 cos(2 pi x) cos(2 pi y).
    Same discretisation as adr_neumann (reading E10): nodes x_i = -1 + i dx, dx = 2/(nx-1),
    mirrored ghost nodes.  (ReactionDiffusion2D is the periodic variant, reading E4.)
    Returns (problem, u0)."""
    ny = ny or nx
    dx, dy = 2.0 / (nx - 1), 2.0 / (ny - 1)
    row_ptr, col, val = [0], [], []
    for j in range(ny):
        for i in range(nx):
            ent = {}
            for ii, jj, w in ((i, j, -2.0 * alpha / dx ** 2 - 2.0 * alpha / dy ** 2), (i - 1, j, alpha / dx ** 2),
                              (i + 1, j, alpha / dx ** 2), (i, j - 1, alpha / dy ** 2), (i, j + 1, alpha / dy ** 2)):
                ii = -ii if ii < 0 else (2 * (nx - 1) - ii if ii > nx - 1 else ii)  # mirror
                jj = -jj if jj < 0 else (2 * (ny - 1) - jj if jj > ny - 1 else jj)
                k = ii + nx * jj
                ent[k] = ent.get(k, 0.0) + w
            for k in sorted(ent):
                col.append(k)
                val.append(ent[k])
            row_ptr.append(len(col))
    prob = ReactionDiffusionCSR(row_ptr, col, val, (0.0, 1.0, 0.0, -1.0))
    prob.nx, prob.ny = nx, ny
    xs, ys = -1.0 + dx * np.arange(nx), -1.0 + dy * np.arange(ny)
    X, Y = np.meshgrid(xs, ys, indexing="xy")
    u0 = (0.1 + 0.1 * np.cos(2 * np.pi * X) * np.cos(2 * np.pi * Y)).ravel()
    return prob, u0


# ---------------------------------------------------------------------------
# one step / integration
# ---------------------------------------------------------------------------
def remainder(prob, yn, fn, y):
    """r(y) = f(y) - f(y_n) - J_n (y - y_n); problems with a linear part may
    provide the identical pointwise form (reading E7)."""
    if hasattr(prob, "remainder"):
        return prob.remainder(yn, y)
    return prob.f(y) - fn - prob.jmul(yn, y - yn)


def step(prob, scheme, yn, h, tol=1e-12, m_hint=(10, 10), m_max=128):
    """One EPIRK4s3 / EPIRK4s3A step with the two grouped KIOPS calls.
    Returns (y_{n+1}, (final_m call 1, final_m call 2), [stats1, stats2])."""
    ca, cb = NODES[scheme]
    fn = prob.f(yn)
    b1 = h * fn
    op = prob.kiops_op(yn, h)  # the matrix argument is h J_n
    zero = np.zeros_like(yn)
    # call 1 (Task I): phi_1(T h J) h f at both nodes, T ascending, scaled by 1/T
    T1 = np.array(sorted((ca, cb)))
    w1, s1, tr1, rc = O.kiops(op, [zero, b1], T1, tol=tol, m_init=m_hint[0], m_min=min(10, m_hint[0]),
                              m_max=m_max, task1=1)
    assert rc == "OK", rc
    s1["trace"] = tr1  # the call's decision trace (GPU parity compares it call by call)
    phi = {T1[0]: w1[0], T1[1]: w1[1]}
    U2 = yn + ca * phi[ca]
    U3 = yn + cb * phi[cb]
    r2 = remainder(prob, yn, fn, U2)
    r3 = remainder(prob, yn, fn, U3)
    b3, b4 = final_b34(scheme, h, r2, r3)
    # call 2 (Task II at tau = 1): phi_1 b1 + phi_3 b3 + phi_4 b4 (b0 = b2 = 0)
    w2, s2, tr2, rc = O.kiops(op, [zero, b1, zero, b3, b4], np.array([1.0]), tol=tol, m_init=m_hint[1],
                              m_min=min(10, m_hint[1]), m_max=m_max)
    assert rc == "OK", rc
    s2["trace"] = tr2
    return yn + w2[0], (s1["final_m"], s2["final_m"]), [s1, s2]


def _task1(op, p, b, T, tol, m, m_max):
    """Task I (Sec. 2): phi_p(T_l A) b for every T_l (ascending), from one KIOPS
    call with u_p = b, all other u_k = 0, and the 1/T^p scaling (Alg. 1 l.31-35)."""
    zero = np.zeros_like(b)
    u = [zero] * p + [b]
    w, st, tr, rc = O.kiops(op, u, np.asarray(T, dtype=np.float64), tol=tol, m_init=m, m_min=min(10, m),
                            m_max=m_max, task1=1)
    assert rc == "OK", rc
    st["trace"] = tr
    return w, st


def step5(prob, scheme, yn, h, tol=1e-12, m_hint=(10, 10, 10), m_max=128):
    """One fifth-order step with three grouped KIOPS calls (Sec. 4: "fifth-order methods
    require only three calls").
    EPIRK5P1, Eq. 52 with Table 1 (the U_{n3} line's truncated "+ alpha_22" completed from
    the Eq. 2 template as alpha_22 phi_1(g_22 h J) h r(U_{n2}), reading E8):
      call 1: phi_1 on h f at T = [g11, g21, g31];  call 2: phi_1 on h r(U2) at [g32, g22];
      call 3: phi_3 on h(-2 r(U2) + r(U3)) at [g33].
    EXPRB5s3, Eq. 53:
      call 1: phi_1 on h f at [1/2, 9/10];  call 2: phi_3 on h r(U2) at [1/2, 9/10];
      call 3 (Task II, tau = 1): phi_1 h f + phi_3 b3 + phi_4 b4 with
      b3 = 18 h r2 - 250/81 h r3, b4 = -60 h r2 + 500/27 h r3.
    Returns (y_{n+1}, (final m of calls 1-3), [stats])."""
    fn = prob.f(yn)
    b1 = h * fn
    op = prob.kiops_op(yn, h)
    zero = np.zeros_like(yn)
    if scheme == "epirk5p1":
        w1, s1 = _task1(op, 1, b1, [G11, G21, G31], tol, m_hint[0], m_max)
        U2 = yn + A11 * w1[0]
        r2 = remainder(prob, yn, fn, U2)
        w2, s2 = _task1(op, 1, h * r2, [G32, G22], tol, m_hint[1], m_max)
        U3 = yn + A21 * w1[1] + A22 * w2[1]
        r3 = remainder(prob, yn, fn, U3)
        w3, s3 = _task1(op, 3, h * (-2.0 * r2 + r3), [G33], tol, m_hint[2], m_max)
        y = yn + B1 * w1[2] + B2 * w2[0] + B3 * w3[0]
    elif scheme == "exprb5s3":
        w1, s1 = _task1(op, 1, b1, [0.5, 0.9], tol, m_hint[0], m_max)
        U2 = yn + 0.5 * w1[0]
        r2 = remainder(prob, yn, fn, U2)
        w2, s2 = _task1(op, 3, h * r2, [0.5, 0.9], tol, m_hint[1], m_max)
        U3 = yn + 0.9 * w1[1] + (27.0 / 25.0) * w2[0] + (729.0 / 125.0) * w2[1]
        r3 = remainder(prob, yn, fn, U3)
        b3 = 18.0 * h * r2 - (250.0 / 81.0) * h * r3
        b4 = -60.0 * h * r2 + (500.0 / 27.0) * h * r3
        w3, s3, tr3, rc = O.kiops(op, [zero, b1, zero, b3, b4], np.array([1.0]), tol=tol, m_init=m_hint[2],
                                  m_min=min(10, m_hint[2]), m_max=m_max)
        assert rc == "OK", rc
        s3["trace"] = tr3
        y = yn + w3[0]
    else:
        raise ValueError(scheme)
    return y, (s1["final_m"], s2["final_m"], s3["final_m"]), [s1, s2, s3]


def integrate(prob, scheme, y0, t0, t1, nsteps, tol=1e-12):
    """Constant-step integration over [t0, t1] (Sec. 4); m chained across steps."""
    h = (t1 - t0) / nsteps
    y = np.array(y0, dtype=np.float64)
    five = scheme in SCHEMES5
    m = (10, 10, 10) if five else (10, 10)
    kv = 0
    calls = []  # per step, per call: counts, final m and the decision trace
    for n in range(nsteps):
        y, m, st = (step5 if five else step)(prob, scheme, y, h, tol=tol, m_hint=m)
        kv += sum(s["krylov_vectors"] for s in st)
        calls += [dict(s, step=n, call=c) for c, s in enumerate(st)]
    return y, {"krylov_vectors": kv, "final_m": m, "calls": calls}
