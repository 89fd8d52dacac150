"""GPU parity of the EPIRK driver (kiops_epirk_*) against the
oracle's EPIRK (oracle/epirk.py, pinned in test_pins_epirk.py): same problem, scheme,
step, KIOPS tolerance and warm-start rule; the GPU's two KIOPS calls per step take the
same decisions (up to a rounding flip at a threshold: Krylov counts within 2%), and u
agrees to 1e-10 relative."""
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
    u = torch.as_tensor(u0.copy(), device=DEV)
    st = k.step(u, n)
    torch.cuda.synchronize()
    g = u.cpu().numpy()
    rel = np.linalg.norm(g - yo) / np.linalg.norm(yo)
    print(f"EPIRK {scheme} {dims}: rel l2 vs oracle {rel:.2e}, KVs gpu {st['krylov_vectors']} oracle "
          f"{so['krylov_vectors']}, final m {st['final_m']} / {so['final_m']}")
    assert st["steps"] == n
    # the result is the unique quantity; a decision at a threshold (omega ~ 1.4, the R3
    # breakdown test) may flip on rounding and cost one Krylov vector more or less
    assert abs(st["krylov_vectors"] - so["krylov_vectors"]) <= max(2, so["krylov_vectors"] // 50)
    assert rel <= 1e-10, rel
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
