"""End-to-end pins of the oracle's Alg. 1 against results the paper and
the mathematics fix: A = 0 closed form, diagonal A (scalar phi), circulant FFT
closed forms, dense expm of the augmented matrix (Theorem 1, via scipy),
Eq. 15 tail identity, semigroup (Eqs. 23-24), Task I, tol monotonicity
(SURVEY P3, P8-P14).  Absolute l2 error of the top block <= 10 tol (R18)."""
from math import factorial

import numpy as np
import pytest
import scipy.linalg as sl

from oracle import oracle as O
from tests.phiref import (circulant_phi_combination, phi, symbol_1d, symbol_2d,
                          symbol_3d_const_kappa)
from workloads import configs as W


def aug_dense(A, u):
    N, p = A.shape[0], len(u) - 1
    At = np.zeros((N + p, N + p))
    At[:N, :N] = A
    for c in range(p):
        At[:N, N + c] = u[p - c]
    if p:
        At[N:, N:] = np.diag(np.ones(p - 1), 1)
    return At


def dense_ref(A, u, tau):
    """Theorem 1 evaluated with scipy's expm (independent of the oracle's Pade)."""
    N, p = A.shape[0], len(u) - 1
    v = np.r_[u[0], np.eye(p)[-1]] if p else u[0]
    return sl.expm(tau * aug_dense(A, u)) @ v


def err(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b))


def test_theorem1_dense_route_tail_and_partial_sums():
    # Eq. 15 tail identity and Eq. 18 partial sums, with a diagonal A so each
    # entry is a scalar closed form sum_k tau^k phi_k(tau lambda) b_k.
    rng = np.random.default_rng(0)
    N, p, tau = 6, 3, 0.37
    lam = -rng.uniform(0.1, 5.0, N)
    u = [rng.standard_normal(N) for _ in range(p + 1)]
    out = O.dense_phi_combination({"kind": "dense", "nx": N, "dense": np.diag(lam)}, u, tau)
    tail = [tau ** (p - 1 - c) / factorial(p - 1 - c) for c in range(p)]
    assert np.allclose(out[N:], tail, rtol=1e-13, atol=1e-15)
    want = sum((tau ** k) * np.real(phi(k, tau * lam)) * u[k] for k in range(p + 1))
    assert np.allclose(out[:N], want, rtol=1e-13, atol=1e-13)
    # p = 0 reduces to expm(tau A) b_0 ; tau = 0 gives b_0
    A = rng.standard_normal((N, N))
    assert np.allclose(O.dense_phi_combination({"kind": "dense", "nx": N, "dense": A}, u[:1], tau),
                       sl.expm(tau * A) @ u[0], rtol=1e-13)
    assert np.allclose(O.dense_phi_combination({"kind": "dense", "nx": N, "dense": A}, u, 0.0)[:N], u[0])


def test_zero_operator_exact():
    # P8: A = 0 => w(T) = sum_k T^k/k! u_k (phi_k(0) = 1/k!), breakdown within p+1 vectors
    rng = np.random.default_rng(1)
    N, p = 50, 3
    u = [rng.standard_normal(N) for _ in range(p + 1)]
    T = [0.25, 0.5, 2.0]
    w, st, tr, rc = O.kiops({"kind": "dense", "nx": N, "dense": np.zeros((N, N))}, u, T, tol=1e-10)
    assert rc == "OK" and st["substeps"] == 1
    for l, t in enumerate(T):
        want = sum(t ** k / factorial(k) * u[k] for k in range(p + 1))
        assert err(w[l], want) <= 1e-13 * np.linalg.norm(want)
    # the Krylov space of A~ has dimension <= p + 1; with p <= 1 it fits the IOP-2
    # window, so Alg. 2 must stop by happy breakdown (l.12-15) at j = p + 1
    for p in (0, 1):
        w, st, tr, rc = O.kiops({"kind": "dense", "nx": N, "dense": np.zeros((N, N))}, u[: p + 1], T)
        assert rc == "OK" and st["happy_breakdowns"] == 1 and tr[0]["j"] == p + 1 and tr[0]["happy"] == 1
        for l, t in enumerate(T):
            want = sum(t ** k / factorial(k) * u[k] for k in range(p + 1))
            assert err(w[l], want) <= 1e-14 * np.linalg.norm(want)


def test_zero_start_vector_is_zero():
    # R27: p = 0 and u_0 = 0 -> beta = 0 -> w = 0
    w, st, tr, rc = O.kiops({"kind": "dense", "nx": 5, "dense": np.eye(5)}, [np.zeros(5)], [1.0])
    assert rc == "OK" and not np.any(w[0])


def test_diagonal_csr_closed_form():
    # P9: diagonal A, lambda_i = -10^U(-2,4); closed form per entry via scalar phi
    rng = np.random.default_rng(2)
    N, p = 3000, 2
    lam = -(10 ** rng.uniform(-2, 4, N))
    u = [rng.standard_normal(N) for _ in range(p + 1)]
    op = {"kind": "csr", "nx": N, "row_ptr": np.arange(N + 1), "col_idx": np.arange(N, dtype=np.int32),
          "vals": lam}
    T = [0.01, 0.1]
    tol = 1e-10
    w, st, tr, rc = O.kiops(op, u, T, tol=tol)
    assert rc == "OK"
    for l, t in enumerate(T):
        want = sum((t ** k) * np.real(phi(k, t * lam)) * u[k] for k in range(p + 1))
        assert err(w[l], want) <= 10 * tol


def test_config1_vs_dense_expm_and_fft():
    # P10/P11: config 1 at full size vs scipy expm of the 403^2 augmented matrix and
    # vs the circulant FFT closed form; also the survey's independent trace probe.
    c = W.config1()
    w, st, tr, rc = O.kiops(c["op"], c["u"], c["T"], tol=c["tol"])
    assert rc == "OK"
    n = c["N"]
    A = np.zeros((n, n))
    for i in range(n):
        A[i, (i - 1) % n] += c["op"]["w"][0]
        A[i, i] += c["op"]["w"][1]
        A[i, (i + 1) % n] += c["op"]["w"][2]
    ref = dense_ref(A, c["u"], c["T"][0])
    assert err(w[0], ref[:n]) <= 10 * c["tol"]
    fft = circulant_phi_combination(symbol_1d(c["op"]["w"], n), c["u"], c["T"][0], (n,))
    assert err(fft, ref[:n]) <= 1e-13 * np.linalg.norm(ref[:n])
    assert [r["j"] for r in tr] == [10, 14, 19, 26, 35, 43]
    assert st["krylov_vectors"] == 43 and st["rejections"] == 5 and st["final_m"] == 42


def test_fft_closed_form_2d_3d():
    # P10 on the configs' constant-coefficient variants: config 3 with v = 0 (d = 1),
    # config 2 with v = 1/2 (d = 0), config 4 with kappa = 1.
    c3 = W.config3(48, 40)
    c3["op"]["diag"] = np.ones(c3["N"])
    w, st, tr, rc = O.kiops(c3["op"], c3["u"], c3["T"], tol=c3["tol"])
    lam = symbol_2d(c3["op"]["w"], 48, 40, d=1.0)
    ref = circulant_phi_combination(lam, c3["u"], c3["T"][0], (40, 48))
    assert rc == "OK" and err(w[0], ref) <= 10 * c3["tol"]

    c2 = W.config2(32, 24)
    c2["op"]["diag"] = np.zeros(c2["N"])
    w, st, tr, rc = O.kiops(c2["op"], c2["u"], c2["T"], tol=c2["tol"])
    ref = circulant_phi_combination(symbol_2d(c2["op"]["w"], 32, 24), c2["u"], c2["T"][0], (24, 32))
    assert rc == "OK" and err(w[0], ref) <= 10 * c2["tol"]

    c4 = W.config4(12, 10, 8)
    c4["op"]["kappa"] = np.ones(c4["N"])
    w, st, tr, rc = O.kiops(c4["op"], c4["u"], c4["T"], tol=c4["tol"])
    lam = symbol_3d_const_kappa(12, 10, 8, c4["op"]["inv_h2"])
    assert rc == "OK"
    for l, t in enumerate(c4["T"]):
        ref = circulant_phi_combination(lam, c4["u"], t, (8, 10, 12))
        assert err(w[l], ref) <= 10 * c4["tol"], l


@pytest.mark.parametrize("seed", range(50))
def test_random_instances_vs_dense(seed):
    # N in {20, 40, 64}, p in 0..4, ||A||_1 in {1, 50, 500}, negative-shifted diagonal
    rng = np.random.default_rng(100 + seed)
    N = [20, 40, 64][seed % 3]
    p = seed % 5
    nrm = [1.0, 50.0, 500.0][(seed // 3) % 3]
    A = rng.standard_normal((N, N))
    A = A - (np.abs(A).sum(axis=1).max() + 1.0) * np.eye(N)
    A *= nrm / np.abs(A).sum(axis=0).max()
    u = [rng.standard_normal(N) for _ in range(p + 1)]
    tol = 1e-10
    w, st, tr, rc = O.kiops({"kind": "dense", "nx": N, "dense": A}, u, [1.0], tol=tol)
    assert rc == "OK"
    ref = dense_ref(A, u, 1.0)[:N]
    assert err(w[0], ref) <= 10 * tol


def test_semigroup_forced_schedule():
    # P12 (Eqs. 23-24): forced substeps [t1, t2] equal one substep t1 + t2
    c = W.config1(64)
    op, u = c["op"], c["u"]
    one, *_ = O.kiops(op, u, [2e-3], forced=[(2e-3, 64)], m_max=128)
    two, st, tr, rc = O.kiops(op, u, [2e-3], forced=[(7e-4, 64), (1.3e-3, 64)], m_max=128)
    assert rc == "OK" and st["substeps"] == 2
    assert err(one[0], two[0]) <= 1e-9 * np.linalg.norm(one[0])


def test_task1_phi1_two_times():
    # P14: one call, phi_1 at T = [1/9, 1/8], scaled by 1/T^p
    c = W.config1(64)
    op = c["op"]
    b = c["u"][1]
    lam = symbol_1d(op["w"], 64)
    for tol in (1e-6, 1e-10):
        w, st, tr, rc = O.kiops(op, [np.zeros(64), b], [1 / 9, 1 / 8], tol=tol, task1=1)
        assert rc == "OK"
        for l, t in enumerate([1 / 9, 1 / 8]):
            ref = np.real(np.fft.ifft(phi(1, t * lam) * np.fft.fft(b)))
            assert err(w[l], ref) <= 10 * tol / t


def test_tolerance_monotone():
    # P13: halving tol never increases the error on a fixed instance
    c = W.config1(96)
    ref = circulant_phi_combination(symbol_1d(c["op"]["w"], 96), c["u"], c["T"][0], (96,))
    errs = []
    for tol in (1e-4, 1e-6, 1e-8, 1e-10):
        w, *_ = O.kiops(c["op"], c["u"], c["T"], tol=tol)
        errs.append(err(w[0], ref))
    assert all(errs[i + 1] <= errs[i] * 1.0000001 for i in range(3)), errs


def test_invalid_arguments():
    c = W.config1(16)
    for kw in ({"tol": 0.0}, {"m_min": 0}, {"m_min": 20, "m_max": 10}, {"iop_q": 0}):
        args = dict(tol=1e-8)
        args.update(kw)
        *_, rc = O.kiops(c["op"], c["u"], [1.0], **args)
        assert rc == "INVALID_ARG"
    *_, rc = O.kiops(c["op"], c["u"], [1.0, 0.5])
    assert rc == "INVALID_ARG"
    *_, rc = O.kiops(c["op"], c["u"], [0.0])
    assert rc == "INVALID_ARG"


def test_replaying_own_trace_is_bitwise():
    # the forced (tau, m, accept) replay hook reproduces a free run exactly (R26)
    c = W.config4(20, 18, 16)
    w, st, tr, rc = O.kiops(c["op"], c["u"], c["T"], tol=c["tol"])
    sched = [(r["tau"], r["j"], r["accept"]) for r in tr]
    w2, st2, tr2, rc2 = O.kiops(c["op"], c["u"], c["T"], tol=c["tol"], forced=sched)
    assert rc == rc2 == "OK" and st["rejections"] > 0
    assert all(np.array_equal(a, b) for a, b in zip(w, w2))
    assert [(r["j"], r["accept"]) for r in tr] == [(r["j"], r["accept"]) for r in tr2]


def _dense_augmented(A, u):
    """Theorem 1: A~ = [[A, B],[0, K]], B = [u_p..u_1], K the upper shift, v = [u_0; e_p]."""
    from scipy.linalg import expm  # noqa: F401

    N, p = A.shape[0], len(u) - 1
    Bm = np.column_stack([u[p - c] for c in range(p)]) if p else np.zeros((N, 0))
    At = np.block([[A, Bm], [np.zeros((p, N)), np.eye(p, k=1)]])
    v = np.r_[u[0], np.zeros(max(p - 1, 0)), [1.0] if p else []]
    return At, v


def test_corrected_scheme_more_accurate_at_fixed_m():
    """Saad's corrected scheme [46] adds beta h_{m+1,m} (tau e_m^T phi_1(tau H_m)
    e_1) v_{m+1}, one more Krylov direction: at a fixed, forced m its error against the
    dense exponential of A~ (Theorem 1) is markedly below the standard scheme's (Eq. 33)."""
    from scipy.linalg import expm

    rng = np.random.default_rng(21)
    for _ in range(20):
        N, p, tau = 30, 2, 0.2
        A = rng.standard_normal((N, N)) - 3 * np.eye(N)
        u = [rng.standard_normal(N) for _ in range(p + 1)]
        At, v = _dense_augmented(A, u)
        ex = (expm(tau * At) @ v)[:N]
        err = []
        for corr in (0, 1):
            w, st, tr, rc = O.kiops({"kind": "dense", "nx": N, "dense": A}, u, [tau], tol=1e-30, m_init=6, m_min=6,
                                    m_max=6, forced=[(tau, 6, 1)], corrected=corr)
            assert rc == "OK"
            err.append(np.linalg.norm(w[0] - ex) / np.linalg.norm(ex))
        assert err[1] < 0.5 * err[0], err


def test_corrected_scheme_free_run_within_tol_and_same_decisions():
    """Free-running corrected scheme: within 10 tol (absolute, R18) of the dense
    exponential at every output time; the first substep takes the standard scheme's
    decisions (the correction changes only the output update, not eps / omega / Alg. 4)."""
    from scipy.linalg import expm

    rng = np.random.default_rng(22)
    for _ in range(8):
        N, p = 40, 3
        A = 3 * rng.standard_normal((N, N)) - 5 * np.eye(N)
        u = [rng.standard_normal(N) for _ in range(p + 1)]
        At, v = _dense_augmented(A, u)
        T = [0.3, 1.0]
        op = {"kind": "dense", "nx": N, "dense": A}
        w1, s1, t1, rc1 = O.kiops(op, u, T, tol=1e-8, m_init=10, m_min=10, m_max=40, corrected=1)
        w0, s0, t0, rc0 = O.kiops(op, u, T, tol=1e-8, m_init=10, m_min=10, m_max=40, corrected=0)
        assert rc1 == rc0 == "OK"
        # the first substep's attempts are identical (the next substep starts from the
        # corrected running solution, so later rows may differ)
        n1 = next(i for i, r in enumerate(t0) if r["accept"]) + 1
        assert t1[:n1] == t0[:n1]
        for l, t in enumerate(T):
            assert np.linalg.norm(w1[l] - (expm(t * At) @ v)[:N]) <= 10 * 1e-8


def test_corrected_scheme_equals_standard_on_happy_breakdown():
    """A = 0: the Krylov space closes (happy breakdown, h_{j+1,j} = 0, no v_{j+1}), so
    the correction vanishes: corrected == standard bitwise (P8's closed form)."""
    rng = np.random.default_rng(23)
    N, p = 25, 3
    u = [rng.standard_normal(N) for _ in range(p + 1)]
    op = {"kind": "dense", "nx": N, "dense": np.zeros((N, N))}
    w0, _, _, _ = O.kiops(op, u, [0.5, 1.0], tol=1e-10, corrected=0)
    w1, _, _, _ = O.kiops(op, u, [0.5, 1.0], tol=1e-10, corrected=1)
    assert all(np.array_equal(a, b) for a, b in zip(w0, w1))
