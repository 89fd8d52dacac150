"""GPU parity of the EPIRK driver (kiops_epirk_*) against the
oracle's EPIRK (oracle/epirk.py, pinned in test_pins_epirk.py): same problem, scheme,
step, KIOPS tolerance and warm-start rule.

On these problems every omega = T eps/(tau tol) sits at the rounding floor of the
projected exponential (F(j, j+1) ~ 1e-14 of F's largest entries: GPU and oracle omegas
differ by 2-6% at tol 1e-6 .. 1e-12, measured), so a decision near a threshold (omega
~ 1.4, the ceil of Eq. 46) may flip and the two runs then follow different, equally
valid trajectories (R26, as for config 4).  The parity test is therefore a REPLAY: the
oracle's per-call decision traces are forced on the GPU's calls (kiops_epirk_set_
forced_schedule), and every call of every step must show the same attempts (j,
acceptance), counts and final m, with u within 1e-12 of the oracle -- a divergent
computation fails it.  The free run is checked on the result (1e-10) alone."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import epirk as E  # noqa: E402

DEV = "cuda:0"


def rd(n, ny, alpha=0.1):
    prob = E.ReactionDiffusion2D(n, ny, alpha=alpha)
    wa = prob.wa
    return prob, {"nx": n, "ny": ny, "w": [wa, wa, wa, wa, -4.0 * wa], "c": list(prob.c)}


@pytest.mark.parametrize("scheme", E.SCHEMES + E.SCHEMES5)
@pytest.mark.parametrize("dims", [(48, 40), (64, 64)])
def test_epirk_matches_oracle(scheme, dims):
    from paper_1804_05126_b200 import KiopsEpirk

    prob, pb = rd(*dims)
    u0 = prob.initial()
    h, n, tol = 0.05, 3, 1e-12
    yo, so = E.integrate(prob, scheme, u0, 0.0, n * h, n, tol=tol)
    k = KiopsEpirk(pb, scheme, h, device=DEV, tol=tol)
    k.record_history(True)
    # free run: the result
    u = torch.as_tensor(u0.copy(), device=DEV)
    st = k.step(u, n)
    torch.cuda.synchronize()
    rel_free = np.linalg.norm(u.cpu().numpy() - yo) / np.linalg.norm(yo)
    assert st["steps"] == n and rel_free <= 1e-10, rel_free
    # replay: the oracle's decisions, call by call
    k.set_forced_schedules([(oc["step"], oc["call"], [(r["tau"], r["j"], r["accept"]) for r in oc["trace"]])
                            for oc in so["calls"]])
    u = torch.as_tensor(u0.copy(), device=DEV)
    st = k.step(u, n)
    torch.cuda.synchronize()
    rel = np.linalg.norm(u.cpu().numpy() - yo) / np.linalg.norm(yo)
    hist = k.history()
    print(f"EPIRK {scheme} {dims}: free run rel l2 {rel_free:.2e}; replay rel l2 {rel:.2e}, KVs gpu "
          f"{st['krylov_vectors']} oracle {so['krylov_vectors']}, {len(hist)} calls compared")
    assert len(hist) == len(so["calls"]) == n * (3 if scheme in E.SCHEMES5 else 2)
    for gc, oc in zip(hist, so["calls"]):
        where = (scheme, dims, "step", oc["step"], "call", oc["call"])
        assert (gc["step"], gc["call"]) == (oc["step"], oc["call"]), where
        assert gc["n_attempts"] == len(oc["trace"]), where
        assert gc["attempts"] == [(r["j"], r["accept"]) for r in oc["trace"]], where
        for key in ("krylov_vectors", "substeps", "rejections"):
            assert gc[key] == oc[key], where + (key, gc[key], oc[key])
    assert st["krylov_vectors"] == so["krylov_vectors"]
    assert rel <= 1e-12, rel
    k.close()


def test_epirk_linear_reaction_is_the_exponential():
    # R(u) = lam u: every remainder vanishes and a step is exp(h (L + lam I)) u; the
    # periodic 5-point L is diagonalised by the 2D FFT (independent of KIOPS)
    from paper_1804_05126_b200 import KiopsEpirk

    n, lam, alpha, h = 32, -0.5, 0.1, 0.2
    prob = E.ReactionDiffusion2D(n, alpha=alpha, coef=(0.0, lam, 0.0, 0.0))
    wa = prob.wa
    pb = {"nx": n, "ny": n, "w": [wa, wa, wa, wa, -4 * wa], "c": [0.0, lam, 0.0, 0.0]}
    u0 = prob.initial()
    k = KiopsEpirk(pb, "epirk4s3a", h, device=DEV, tol=1e-13)
    u = torch.as_tensor(u0.copy(), device=DEV)
    k.step(u, 2)
    kx = 2 * np.pi * np.fft.fftfreq(n)
    sym = wa * (2 * np.cos(kx)[None, :] + 2 * np.cos(kx)[:, None] - 4) + lam
    ref = np.real(np.fft.ifft2(np.exp(2 * h * sym) * np.fft.fft2(u0.reshape(n, n)))).ravel()
    g = u.cpu().numpy()
    assert np.linalg.norm(g - ref) <= 1e-10 * np.linalg.norm(ref)


# ---------------------------------------------------------------------------
# general CSR linear part: the ADR 2D problem with homogeneous Neumann boundaries
# (reading E10); h J_n is a KIOPS_OP_CSR operator rewritten every step
# ---------------------------------------------------------------------------
def adr(nx, ny):
    prob, u0 = E.adr_neumann(nx, ny)
    pb = {"nx": nx, "ny": ny, "c": list(prob.c),
          "L": {"row_ptr": prob.row_ptr, "col_idx": prob.col_idx, "vals": prob.vals}}
    return prob, u0, pb


@pytest.mark.parametrize("scheme", E.SCHEMES + E.SCHEMES5)
def test_epirk_adr_neumann_matches_oracle(scheme):
    from paper_1804_05126_b200 import KiopsEpirk

    prob, u0, pb = adr(24, 20)
    h, n, tol = 0.0025, 3, 1e-12
    yo, so = E.integrate(prob, scheme, u0, 0.0, n * h, n, tol=tol)
    k = KiopsEpirk(pb, scheme, h, device=DEV, tol=tol)
    k.record_history(True)
    u = torch.as_tensor(u0.copy(), device=DEV)
    st = k.step(u, n)
    torch.cuda.synchronize()
    rel_free = np.linalg.norm(u.cpu().numpy() - yo) / np.linalg.norm(yo)
    assert st["steps"] == n and rel_free <= 1e-10, rel_free
    k.set_forced_schedules([(oc["step"], oc["call"], [(r["tau"], r["j"], r["accept"]) for r in oc["trace"]])
                            for oc in so["calls"]])
    u = torch.as_tensor(u0.copy(), device=DEV)
    st = k.step(u, n)
    torch.cuda.synchronize()
    rel = np.linalg.norm(u.cpu().numpy() - yo) / np.linalg.norm(yo)
    hist = k.history()
    print(f"EPIRK ADR {scheme}: free run rel l2 {rel_free:.2e}; replay rel l2 {rel:.2e}, KVs gpu "
          f"{st['krylov_vectors']} oracle {so['krylov_vectors']}, {len(hist)} calls compared")
    assert len(hist) == len(so["calls"])
    for gc, oc in zip(hist, so["calls"]):
        where = (scheme, "step", oc["step"], "call", oc["call"])
        assert gc["attempts"] == [(r["j"], r["accept"]) for r in oc["trace"]], where
        for key in ("krylov_vectors", "substeps", "rejections"):
            assert gc[key] == oc[key], where + (key, gc[key], oc[key])
    assert rel <= 1e-12, rel
    k.close()


@pytest.mark.parametrize("scheme", E.SCHEMES)
def test_epirk_order_four_on_the_gpu(scheme):
    # the GPU integrator against an independent implicit integrator (scipy Radau) on the
    # ADR problem: slope 4 under step halving (f1's order test, on the device)
    from scipy.integrate import solve_ivp

    from paper_1804_05126_b200 import KiopsEpirk

    prob, u0, pb = adr(10, 10)
    T = 0.02
    ref = solve_ivp(lambda t, y: prob.f(y), (0.0, T), u0, method="Radau", rtol=1e-12, atol=1e-13,
                    jac=lambda t, y: np.column_stack([prob.jmul(y, e) for e in np.eye(prob.dim)])).y[:, -1]
    steps, errs = [2, 4, 8, 16], []
    for n in steps:
        k = KiopsEpirk(pb, scheme, T / n, device=DEV, tol=1e-13)
        u = torch.as_tensor(u0.copy(), device=DEV)
        k.step(u, n)
        torch.cuda.synchronize()
        errs.append(np.linalg.norm(u.cpu().numpy() - ref) / np.linalg.norm(ref))
        k.close()
    slope = np.polyfit(np.log([1.0 / n for n in steps]), np.log(errs), 1)[0]
    print(f"GPU ADR {scheme}: errors {['%.2e' % e for e in errs]}, observed order {slope:.2f}")
    assert 3.6 <= slope <= 4.6, (slope, errs)


def test_epirk_csr_rejects_a_row_without_diagonal():
    from paper_1804_05126_b200 import KiopsEpirk
    from paper_1804_05126_b200.kiops import KiopsError

    n = 8
    rp = np.arange(n + 1, dtype=np.int64)
    ci = ((np.arange(n) + 1) % n).astype(np.int32)  # one off-diagonal entry per row, no diagonal
    pb = {"nx": n, "ny": 1, "c": [0.0, 1.0, 0.0, 0.0], "L": {"row_ptr": rp, "col_idx": ci, "vals": np.ones(n)}}
    with pytest.raises(KiopsError) as ei:
        KiopsEpirk(pb, "epirk4s3", 0.1, device=DEV)
    assert ei.value.status == "KIOPS_ERR_INVALID_ARG"


def test_refresh_operator_csr_values():
    # kiops_refresh_operator: the CSR values rewritten in place between two applies
    from oracle import oracle
    from paper_1804_05126_b200 import Kiops
    from workloads import configs

    c = configs.config5(12, 10, 9)
    k = Kiops(c["op"], c["p"], device=DEV, tol=c["tol"], m_init=c["m_init"], m_min=c["m_min"], m_max=c["m_max"])
    u = [torch.as_tensor(x, device=DEV) for x in c["u"]]
    w0, _ = k.apply(u, c["T"])
    g0 = w0[0].cpu().numpy().copy()
    k.dev["vals"].mul_(0.5)
    k.refresh_operator()
    w1, _ = k.apply(u, c["T"])
    torch.cuda.synchronize()
    op2 = dict(c["op"])
    op2["vals"] = 0.5 * np.asarray(c["op"]["vals"])
    ref0 = oracle.kiops(c["op"], c["u"], c["T"], tol=c["tol"])[0][0]
    ref1 = oracle.kiops(op2, c["u"], c["T"], tol=c["tol"])[0][0]
    assert np.linalg.norm(g0 - ref0) <= 1e-10 * np.linalg.norm(ref0)
    assert np.linalg.norm(w1[0].cpu().numpy() - ref1) <= 1e-10 * np.linalg.norm(ref1)
    assert np.linalg.norm(ref1 - ref0) > 1e-3 * np.linalg.norm(ref0)  # (the two operators differ)
    k.close()


@pytest.mark.parametrize("scheme", E.SCHEMES + E.SCHEMES5)
def test_epirk_allen_cahn_noflow_matches_oracle(scheme):
    # the paper's Allen-Cahn problem with its no-flow boundaries through the CSR linear part
    from paper_1804_05126_b200 import KiopsEpirk

    nx, ny = 30, 22
    prob, u0 = E.allen_cahn_noflow(nx, ny)
    pb = {"nx": nx, "ny": ny, "c": list(prob.c),
          "L": {"row_ptr": prob.row_ptr, "col_idx": prob.col_idx, "vals": prob.vals}}
    h, n, tol = 0.0625, 3, 1e-12
    yo, so = E.integrate(prob, scheme, u0, 0.0, n * h, n, tol=tol)
    k = KiopsEpirk(pb, scheme, h, device=DEV, tol=tol)
    k.record_history(True)
    k.set_forced_schedules([(oc["step"], oc["call"], [(r["tau"], r["j"], r["accept"]) for r in oc["trace"]])
                            for oc in so["calls"]])
    u = torch.as_tensor(u0.copy(), device=DEV)
    st = k.step(u, n)
    torch.cuda.synchronize()
    rel = np.linalg.norm(u.cpu().numpy() - yo) / np.linalg.norm(yo)
    hist = k.history()
    assert len(hist) == len(so["calls"])
    for gc, oc in zip(hist, so["calls"]):
        assert gc["attempts"] == [(r["j"], r["accept"]) for r in oc["trace"]], (scheme, oc["step"], oc["call"])
    assert st["krylov_vectors"] == so["krylov_vectors"]
    assert rel <= 1e-12, rel
    k.close()
