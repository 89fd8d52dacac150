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
