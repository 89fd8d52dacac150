"""Pins of the EPIRK oracle (oracle/epirk.py) against things other
than itself: the exact solution of the 1D semilinear problem (order 4, SPEC's test
idea S:540), the exact exponential of linear problems (scipy.linalg.expm, an
independent routine), a naive per-phi-term evaluation of Eq. 50/51 with phi_k from
scipy's expm of the block matrix [[M, v e_1^T], [0, J_k]], hand-expanded remainders,
and finite-difference Jacobians."""
import numpy as np
import pytest
import scipy.linalg as sla

from oracle import epirk as E


class Linear:
    """f(y) = A y (dense): every remainder vanishes, so a step is exp(hA) y exactly."""

    def __init__(self, A):
        self.A = np.asarray(A, dtype=np.float64)
        self.dim = self.A.shape[0]

    def f(self, y):
        return self.A @ y

    def jmul(self, y, x):
        return self.A @ x

    def kiops_op(self, y, h):
        return {"kind": "dense", "nx": self.dim, "ny": 1, "nz": 1, "dense": h * self.A}


class Square:
    """scalar f(u) = u^2 (SPEC's remainder example)."""

    dim = 1

    def f(self, y):
        return y * y

    def jmul(self, y, x):
        return 2.0 * y * x


def phi_k_v(M, v, k):
    """phi_k(M) v from the exponential of the (n+k)-block matrix (independent of KIOPS)."""
    n = len(v)
    W = np.zeros((n + k, n + k))
    W[:n, :n] = M
    W[:n, n] = v
    for i in range(k - 1):
        W[n + i, n + i + 1] = 1.0
    return sla.expm(W)[:n, n + k - 1]


def naive_step(prob, scheme, y, h, J):
    """Eq. 50 / Eq. 51 term by term, every phi_k(g h J) b evaluated separately."""
    ca, cb = E.NODES[scheme]
    fn = prob.f(y)
    U2 = y + ca * phi_k_v(ca * h * J, h * fn, 1)
    U3 = y + cb * phi_k_v(cb * h * J, h * fn, 1)
    r2 = prob.f(U2) - fn - J @ (U2 - y)
    r3 = prob.f(U3) - fn - J @ (U3 - y)
    M = h * J
    out = y + phi_k_v(M, h * fn, 1)
    if scheme == "epirk4s3":
        terms = [(1892.0, 3, r2), (-42336.0, 4, r2), (1458.0, 3, r3 - 2 * r2), (-34992.0, 4, r3 - 2 * r2)]
    else:
        terms = [(32.0, 3, r2), (-144.0, 4, r2), (-13.5, 3, r3), (81.0, 4, r3)]
    for c, k, r in terms:
        out = out + c * phi_k_v(M, h * r, k)
    return out


def test_remainder_pins():
    sq = Square()
    u_n = np.array([1.0])
    h = 0.1
    r = E.remainder(sq, u_n, sq.f(u_n), u_n + h)
    assert abs(r[0] - h * h) <= 1e-15  # (1+h)^2 - 1 - 2h = h^2
    for prob in (E.Semilinear1D(20), E.ReactionDiffusion2D(8)):
        y = prob.exact(0.3) if hasattr(prob, "exact") else prob.initial()
        assert not np.any(E.remainder(prob, y, prob.f(y), y))  # r(u_n) = 0 exactly


def test_pointwise_remainder_is_the_papers_definition():
    # reading E7: for f = L u + R(u) the L terms of f(U) - f(u_n) - J_n (U - u_n) cancel
    rng = np.random.default_rng(5)
    prob = E.ReactionDiffusion2D(10, alpha=0.01)
    yn = prob.initial()
    y = yn + 0.1 * rng.standard_normal(prob.dim)
    full = prob.f(y) - prob.f(yn) - prob.jmul(yn, y - yn)
    assert np.linalg.norm(prob.remainder(yn, y) - full) <= 1e-12 * np.linalg.norm(full)


@pytest.mark.parametrize("prob", [E.Semilinear1D(30), E.ReactionDiffusion2D(12)], ids=["semilinear", "allen_cahn"])
def test_jacobian_matches_finite_differences(prob):
    rng = np.random.default_rng(7)
    y = prob.exact(0.2) if hasattr(prob, "exact") else prob.initial() + 0.05 * rng.standard_normal(prob.dim)
    x = rng.standard_normal(prob.dim)
    eps = 1e-6 * (1.0 + np.linalg.norm(y) / np.linalg.norm(x))
    fd = (prob.f(y + eps * x) - prob.f(y - eps * x)) / (2 * eps)
    jx = prob.jmul(y, x)
    assert np.linalg.norm(fd - jx) <= 1e-5 * np.linalg.norm(jx)


@pytest.mark.parametrize("scheme", E.SCHEMES)
def test_linear_problem_step_is_the_exponential(scheme):
    rng = np.random.default_rng(11)
    n = 20
    Q = rng.standard_normal((n, n))
    A = -(Q @ Q.T) / n - 0.5 * np.eye(n) + 0.3 * (Q - Q.T) / np.sqrt(n)
    prob = Linear(A)
    y = rng.standard_normal(n)
    h = 0.7
    y1, _, _ = E.step(prob, scheme, y, h, tol=1e-13)
    ref = sla.expm(h * A) @ y
    assert np.linalg.norm(y1 - ref) <= 1e-9 * np.linalg.norm(ref)


@pytest.mark.parametrize("scheme", E.SCHEMES)
def test_scalar_decay(scheme):
    prob = Linear([[-1.0]])
    y, _ = E.integrate(prob, scheme, np.array([1.0]), 0.0, 1.0, 10, tol=1e-13)
    assert abs(y[0] - np.exp(-1.0)) <= 1e-9


@pytest.mark.parametrize("scheme", E.SCHEMES)
def test_grouped_step_equals_naive_per_term_evaluation(scheme):
    # stage-grouping equivalence (SPEC S:540 idea): the two grouped KIOPS calls give the
    # same step as evaluating every phi_k(g h J) b of Eq. 50/51 separately
    for prob, y, h in ((E.ReactionDiffusion2D(8, alpha=0.1), None, 0.05), (E.Semilinear1D(20), None, 0.1)):
        y = prob.exact(0.0) if hasattr(prob, "exact") else prob.initial()
        J = np.column_stack([prob.jmul(y, e) for e in np.eye(prob.dim)])
        got, _, _ = E.step(prob, scheme, y, h, tol=1e-13)
        ref = naive_step(prob, scheme, y, h, J)
        assert np.linalg.norm(got - ref) <= 1e-9 * np.linalg.norm(ref), (scheme, np.linalg.norm(got - ref))


@pytest.mark.parametrize("scheme", E.SCHEMES)
def test_order_four_on_the_semilinear_problem(scheme):
    # Sec. 4 problem with its exact solution x(1-x)e^t; SPEC's order test:
    # slope 4 +- 0.3 under step halving
    prob = E.Semilinear1D(200)
    steps = [4, 8, 16, 32]
    errs = []
    for n in steps:
        y, _ = E.integrate(prob, scheme, prob.exact(0.0), 0.0, 1.0, n, tol=1e-13)
        ex = prob.exact(1.0)
        errs.append(np.linalg.norm(y[:-1] - ex[:-1]) / np.linalg.norm(ex[:-1]))
    slope = np.polyfit(np.log([1.0 / n for n in steps]), np.log(errs), 1)[0]
    print(f"{scheme}: errors {['%.2e' % e for e in errs]}, observed order {slope:.2f}")
    assert 3.7 <= slope <= 4.3, (slope, errs)


@pytest.mark.parametrize("scheme", E.SCHEMES5)
def test_fifth_order_linear_step_is_the_exponential(scheme):
    rng = np.random.default_rng(12)
    n = 16
    Q = rng.standard_normal((n, n))
    A = -(Q @ Q.T) / n - 0.5 * np.eye(n)
    prob = Linear(A)
    y = rng.standard_normal(n)
    y1, _, _ = E.step5(prob, scheme, y, 0.5, tol=1e-13)
    ref = sla.expm(0.5 * A) @ y
    assert np.linalg.norm(y1 - ref) <= 1e-9 * np.linalg.norm(ref)


def test_fifth_order_grouping_equals_naive_per_term_evaluation():
    # Eq. 52 / Eq. 53 term by term with the block-matrix phi_k
    prob = E.ReactionDiffusion2D(8, alpha=0.1)
    y = prob.initial()
    h = 0.05
    J = np.column_stack([prob.jmul(y, e) for e in np.eye(prob.dim)])
    fn = prob.f(y)
    M = h * J
    r = lambda U: prob.f(U) - fn - J @ (U - y)  # noqa: E731
    # EPIRK5P1
    U2 = y + E.A11 * phi_k_v(E.G11 * M, h * fn, 1)
    r2 = r(U2)
    U3 = y + E.A21 * phi_k_v(E.G21 * M, h * fn, 1) + E.A22 * phi_k_v(E.G22 * M, h * r2, 1)
    r3 = r(U3)
    ref = (y + E.B1 * phi_k_v(E.G31 * M, h * fn, 1) + E.B2 * phi_k_v(E.G32 * M, h * r2, 1)
           + E.B3 * phi_k_v(E.G33 * M, h * (-2 * r2 + r3), 3))
    got, _, _ = E.step5(prob, "epirk5p1", y, h, tol=1e-13)
    assert np.linalg.norm(got - ref) <= 1e-9 * np.linalg.norm(ref)
    # EXPRB5s3
    U2 = y + 0.5 * phi_k_v(0.5 * M, h * fn, 1)
    r2 = r(U2)
    U3 = (y + 0.9 * phi_k_v(0.9 * M, h * fn, 1) + 27 / 25 * phi_k_v(0.5 * M, h * r2, 3)
          + 729 / 125 * phi_k_v(0.9 * M, h * r2, 3))
    r3 = r(U3)
    ref = (y + phi_k_v(M, h * fn, 1) + 18 * phi_k_v(M, h * r2, 3) - 60 * phi_k_v(M, h * r2, 4)
           - 250 / 81 * phi_k_v(M, h * r3, 3) + 500 / 27 * phi_k_v(M, h * r3, 4))
    got, _, _ = E.step5(prob, "exprb5s3", y, h, tol=1e-13)
    assert np.linalg.norm(got - ref) <= 1e-9 * np.linalg.norm(ref)


def test_table1_coefficients_as_printed():
    # Table 1 round trip, SPEC's example values
    assert E.A11 == 0.3512959269505819 and E.G33 == 0.6237811195337149 and E.G32 == 0.71111109536436687


class Logistic:
    """u' = u(1-u), u(0) = 0.1: exact 1/(1 + 9 e^-t); non-stiff, so every scheme shows
    its classical order."""

    dim = 1

    def f(self, y):
        return y * (1.0 - y)

    def jmul(self, y, x):
        return (1.0 - 2.0 * y) * x

    def kiops_op(self, y, h):
        return {"kind": "dense", "nx": 1, "ny": 1, "nz": 1, "dense": h * np.array([[1.0 - 2.0 * y[0]]])}


def observed_order(prob, scheme, y0, t1, steps, exact, tol):
    errs = []
    for n in steps:
        y, _ = E.integrate(prob, scheme, y0, 0.0, t1, n, tol=tol)
        errs.append(np.linalg.norm(y - exact) / np.linalg.norm(exact))
    return np.polyfit(np.log([t1 / n for n in steps]), np.log(errs), 1)[0], errs


@pytest.mark.parametrize("scheme", E.SCHEMES5)
def test_fifth_order_schemes_are_classically_fifth_order(scheme):
    slope, errs = observed_order(Logistic(), scheme, np.array([0.1]), 2.0, [4, 8, 16],
                                 np.array([1.0 / (1.0 + 9.0 * np.exp(-2.0))]), 1e-14)
    print(f"{scheme} (logistic): errors {['%.2e' % e for e in errs]}, order {slope:.2f}")
    assert slope >= 4.6, (slope, errs)


def test_stiff_orders_on_the_semilinear_problem():
    # EXPRB5s3 is stiffly accurate: order 5 on the stiff semi-discretisation (h <= 1/8);
    # EPIRK5P1 is "classical (non-stiffly accurate)": it reduces to ~3 there
    prob = E.Semilinear1D(200)
    ex = prob.exact(1.0)
    s5, e5 = observed_order(prob, "exprb5s3", prob.exact(0.0), 1.0, [8, 16, 32], ex, 1e-14)
    s1, e1 = observed_order(prob, "epirk5p1", prob.exact(0.0), 1.0, [8, 16, 32], ex, 1e-14)
    print(f"exprb5s3: {['%.2e' % e for e in e5]} order {s5:.2f}; epirk5p1: {['%.2e' % e for e in e1]} order {s1:.2f}")
    assert 4.6 <= s5 <= 5.4, (s5, e5)
    assert 2.6 <= s1 <= 3.6, (s1, e1)


# ---------------------------------------------------------------------------
# ADR 2D with homogeneous Neumann boundaries (reading E10): the general
# CSR linear part of ReactionDiffusionCSR
# ---------------------------------------------------------------------------
def _adr_f_reference(u, nx, ny, eps, alpha, gamma):
    """f(u) by an independent formulation: numpy's reflect padding IS the mirrored ghost
    node u_{-1} = u_{1}; central differences on the padded array."""
    U = u.reshape(ny, nx)
    dx, dy = 1.0 / (nx - 1), 1.0 / (ny - 1)
    P = np.pad(U, 1, mode="reflect")
    c, w, e, s, n = P[1:-1, 1:-1], P[1:-1, :-2], P[1:-1, 2:], P[:-2, 1:-1], P[2:, 1:-1]
    lap = (w - 2 * c + e) / dx ** 2 + (s - 2 * c + n) / dy ** 2
    adv = (e - w) / (2 * dx) + (n - s) / (2 * dy)
    return (eps * lap - alpha * adv + gamma * c * (c - 0.5) * (1.0 - c)).ravel()


def test_adr_neumann_matches_reflect_padded_differences():
    rng = np.random.default_rng(3)
    for nx, ny in ((9, 9), (12, 7)):
        prob, u0 = E.adr_neumann(nx, ny)
        u = u0 + 0.2 * rng.standard_normal(prob.dim)
        ref = _adr_f_reference(u, nx, ny, 0.01, -10.0, 100.0)
        assert np.linalg.norm(prob.f(u) - ref) <= 1e-12 * np.linalg.norm(ref)
        # constants are in the kernel of the linear part (no-flux boundaries, central advection)
        assert np.abs(prob.lmul(np.ones(prob.dim))).max() <= 1e-10
        # initial condition as printed: 0.3 on the boundary, 256/4^4 + 0.3 = 1.3 at the centre
        assert np.allclose(u0.reshape(ny, nx)[0], 0.3) and np.allclose(u0.reshape(ny, nx)[:, -1], 0.3)
    prob, u0 = E.adr_neumann(9, 9)
    assert abs(u0.reshape(9, 9)[4, 4] - 1.3) <= 1e-15


def test_adr_jacobian_and_remainder():
    rng = np.random.default_rng(9)
    prob, u0 = E.adr_neumann(10, 8)
    y = u0 + 0.05 * rng.standard_normal(prob.dim)
    x = rng.standard_normal(prob.dim)
    h = 1e-6
    fd = (prob.f(y + h * x) - prob.f(y - h * x)) / (2 * h)
    jx = prob.jmul(y, x)
    assert np.linalg.norm(fd - jx) <= 1e-6 * np.linalg.norm(jx)
    full = prob.f(y) - prob.f(u0) - prob.jmul(u0, y - u0)
    assert np.linalg.norm(prob.remainder(u0, y) - full) <= 1e-10 * np.linalg.norm(full)
    # the KIOPS operator h J(y) as CSR against the dense Jacobian
    import scipy.sparse as sp

    op = prob.kiops_op(y, 0.01)
    A = sp.csr_matrix((op["vals"], op["col_idx"], op["row_ptr"]), shape=(prob.dim, prob.dim)).toarray()
    J = np.column_stack([prob.jmul(y, e) for e in np.eye(prob.dim)])
    assert np.abs(A - 0.01 * J).max() <= 1e-12 * np.abs(J).max()


@pytest.mark.parametrize("scheme", E.SCHEMES)
def test_adr_order_four_against_an_independent_integrator(scheme):
    # reference: scipy's implicit Radau at tight tolerances on the same semi-discrete system
    from scipy.integrate import solve_ivp

    prob, u0 = E.adr_neumann(10, 10)
    T = 0.02
    ref = solve_ivp(lambda t, y: prob.f(y), (0.0, T), u0, method="Radau", rtol=1e-12, atol=1e-13,
                    jac=lambda t, y: np.column_stack([prob.jmul(y, e) for e in np.eye(prob.dim)])).y[:, -1]
    steps = [2, 4, 8, 16]
    errs = []
    for n in steps:
        y, _ = E.integrate(prob, scheme, u0, 0.0, T, n, tol=1e-13)
        errs.append(np.linalg.norm(y - ref) / np.linalg.norm(ref))
    slope = np.polyfit(np.log([1.0 / n for n in steps]), np.log(errs), 1)[0]
    print(f"ADR {scheme}: errors {['%.2e' % e for e in errs]}, observed order {slope:.2f}")
    assert 3.6 <= slope <= 4.6, (slope, errs)


@pytest.mark.parametrize("scheme", E.SCHEMES)
def test_adr_grouped_step_equals_naive_per_term_evaluation(scheme):
    prob, y = E.adr_neumann(7, 6)
    h = 0.004
    J = np.column_stack([prob.jmul(y, e) for e in np.eye(prob.dim)])
    got, _, _ = E.step(prob, scheme, y, h, tol=1e-13)
    ref = naive_step(prob, scheme, y, h, J)
    assert np.linalg.norm(got - ref) <= 1e-9 * np.linalg.norm(ref), (scheme, np.linalg.norm(got - ref))


def test_allen_cahn_noflow_matches_reflect_padded_differences():
    # Allen-Cahn with the paper's no-flow boundaries through the CSR linear part
    rng = np.random.default_rng(4)
    for nx, ny in ((9, 9), (11, 6)):
        prob, u0 = E.allen_cahn_noflow(nx, ny)
        u = u0 + 0.3 * rng.standard_normal(prob.dim)
        U = u.reshape(ny, nx)
        dx, dy = 2.0 / (nx - 1), 2.0 / (ny - 1)
        P = np.pad(U, 1, mode="reflect")
        c, w, e, s_, n = P[1:-1, 1:-1], P[1:-1, :-2], P[1:-1, 2:], P[:-2, 1:-1], P[2:, 1:-1]
        ref = (0.1 * ((w - 2 * c + e) / dx ** 2 + (s_ - 2 * c + n) / dy ** 2) + c - c ** 3).ravel()
        assert np.linalg.norm(prob.f(u) - ref) <= 1e-12 * np.linalg.norm(ref)
        assert np.abs(prob.lmul(np.ones(prob.dim))).max() <= 1e-10
    prob, u0 = E.allen_cahn_noflow(9, 9)
    assert abs(u0.reshape(9, 9)[4, 4] - 0.2) <= 1e-15 and abs(u0[0] - 0.2) <= 1e-15  # cos(0) = cos(2 pi) = 1


@pytest.mark.parametrize("scheme", E.SCHEMES)
def test_allen_cahn_noflow_order_four(scheme):
    from scipy.integrate import solve_ivp

    prob, u0 = E.allen_cahn_noflow(10, 10)
    T = 1.0
    ref = solve_ivp(lambda t, y: prob.f(y), (0.0, T), u0, method="Radau", rtol=1e-12, atol=1e-13,
                    jac=lambda t, y: np.column_stack([prob.jmul(y, e) for e in np.eye(prob.dim)])).y[:, -1]
    steps, errs = [2, 4, 8, 16], []
    for n in steps:
        y, _ = E.integrate(prob, scheme, u0, 0.0, T, n, tol=1e-13)
        errs.append(np.linalg.norm(y - ref) / np.linalg.norm(ref))
    slope = np.polyfit(np.log([1.0 / n for n in steps]), np.log(errs), 1)[0]
    print(f"Allen-Cahn no-flow {scheme}: errors {['%.2e' % e for e in errs]}, observed order {slope:.2f}")
    assert 3.5 <= slope <= 4.8, (slope, errs)
