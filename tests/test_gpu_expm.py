"""The controller's projected exponential (Pade-13 scaling and squaring,
P:359, reading R17) against the oracle's or_expm -- directly, through the test hook
kiops_debug_expm, on both GPU policies (n <= 48: one CTA, every matrix in shared memory,
register-resident elimination; n > 48: the 8-CTA cluster) and every degree branch."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import oracle  # noqa: E402
from workloads import configs  # noqa: E402

DEV = "cuda:0"


@pytest.fixture(scope="module")
def ctx():
    from paper_1804_05126_b200 import Kiops

    c = configs.config1()
    k = Kiops(c["op"], c["p"], device=DEV, tol=c["tol"], m_max=128)
    yield k
    k.close()


def htilde(n, rng, norm):
    """[[H, e_1],[0, 0]] with a tridiagonal H (IOP window 2), scaled to the given 1-norm."""
    j = n - 1
    M = np.zeros((n, n))
    for c in range(j):
        for r in range(max(0, c - 1), min(j, c + 2)):
            M[r, c] = rng.uniform(-0.5, 0.5) - (1.0 if r == c else 0.0)
    if n > 1:
        M[0, j] = 1.0
    nrm = np.abs(M).sum(axis=0).max()
    return M * (norm / nrm) if nrm > 0 else M


def check(k, M, scale=1.0, tol=2e-13):
    Fo, nmo = oracle.expm(M, scale)
    Fg, nmg = k.debug_expm(M, scale)
    assert nmg == nmo, (M.shape, nmg, nmo)  # same degree and number of squarings
    err = np.abs(Fg - Fo).max() / max(np.abs(Fo).max(), 1e-300)
    assert err <= tol, (M.shape, err)
    return err


@pytest.mark.parametrize("n", [1, 2, 3, 7, 11, 12, 16, 24, 25, 33, 39, 40, 47, 48, 49, 64, 85, 113, 128, 129])
def test_expm_matches_oracle_on_projected_matrices(ctx, n):
    rng = np.random.default_rng(100 + n)
    worst = 0.0
    # every degree branch of Higham's cascade (theta_3 .. theta_13) and scaled-and-squared norms
    for norm in (1e-3, 0.1, 0.6, 1.5, 4.0, 30.0, 400.0):
        worst = max(worst, check(ctx, htilde(n, rng, norm)))
    print(f"n = {n}: max |F_gpu - F_oracle| / max |F| = {worst:.2e}")


@pytest.mark.parametrize("n", [5, 20, 48, 60, 129])
def test_expm_dense_and_structured(ctx, n):
    rng = np.random.default_rng(7 + n)
    A = rng.standard_normal((n, n)) / np.sqrt(n)
    check(ctx, A, 1.0)
    check(ctx, A, 7.0)
    check(ctx, A - A.T, 3.0)                      # skew: orthogonal exponential
    check(ctx, np.zeros((n, n)))                  # exp(0) = I (degree 3, no products beyond the cascade)
    check(ctx, np.diag(rng.uniform(-3, 1, n)))    # diagonal
    P = np.roll(np.eye(n), 1, axis=0)             # cyclic shift: every column of V - U has equal-size
    check(ctx, P, 2.0)                            # entries up to symmetry -> exercises pivot ties
    check(ctx, np.ones((n, n)) / n, 5.0)          # rank one, all pivot candidates equal in column 0
    Fg, _ = ctx.debug_expm(np.zeros((n, n)))
    assert np.array_equal(Fg, np.eye(n))


def test_expm_nonfinite_input_is_reported(ctx):
    from paper_1804_05126_b200.kiops import KiopsError

    M = np.eye(6)
    M[2, 3] = np.nan
    with pytest.raises(KiopsError) as ei:
        ctx.debug_expm(M)
    assert ei.value.status == "KIOPS_ERR_NONFINITE"
