"""GPU parity of the NEXT rows f2 (LS-ESPRIT / 2D-ESPRIT) and f3 (Alg. 7 fast
vector forecast) through the C ABI: against the oracle's definitions (oracle.esprit,
oracle.vector_forecast — the latter the plain projector form of P:1416-1460, not Alg. 7) fed the
device's own triples, and against the closed forms of noiseless finite-rank inputs."""
import numpy as np
import pytest

import closed_form as cf
import oracle
import synth
from parity_util import relfro

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _require_gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device")
    from paper_1309_5050_b200 import build
    build.build()


def _pairs_err(lam, mu, lam0, mu0):
    return max(min(abs(lam - a) + abs(mu - b)) for a, b in zip(lam0, mu0))


@pytest.mark.parametrize("dtype", ["f64", "f32"])
@pytest.mark.parametrize("wmask_drop", [0, 5])
def test_esprit_2d_noiseless(dtype, wmask_drop):
    from paper_1309_5050_b200 import Plan
    rng = np.random.default_rng(3)
    t = synth.draw_terms(rng, 2)
    img = synth.separable_image(40, 37, t)
    wm = None
    if wmask_drop:
        wm = np.ones((12, 10), bool)
        wm[rng.choice(12, wmask_drop), rng.choice(10, wmask_drop)] = False
        wm[0, 0] = True
    lam0, mu0, _ = cf.roots(t)
    R = len(lam0)
    p = Plan(img, (12, 10), wmask=wm, dtype=dtype, path="direct", block_k=8)
    p.decompose(R)
    lam, mu = p.esprit(range(R))
    tol = 1e-8 if dtype == "f64" else 2e-4
    assert _pairs_err(lam, mu, lam0, mu0) < tol
    # the same estimation from the same eigenvectors by the oracle's definition
    sh = oracle.shapes(img, (12, 10), wmask=wm)
    lo, mo = oracle.esprit(sh, p.U().astype(np.float64))
    assert _pairs_err(lam, mu, lo, mo) < (1e-9 if dtype == "f64" else 1e-5)


def test_esprit_c3_twin_fp32():
    """2D-ESPRIT at the c3 size (512², window 64², 24 components, fp32 FFT path): the 24 (λ, μ) pairs of
    the six separable terms (closed_form.roots)."""
    w = synth.config3(noise=False)
    from paper_1309_5050_b200 import Plan
    p = Plan(w.data, w.window, dtype="f32", path="fft")
    p.decompose(24)
    lam, mu = p.esprit(range(24))
    lam0, mu0, _ = cf.roots(w.terms)
    assert _pairs_err(lam, mu, lam0, mu0) < 1e-4


def test_esprit_1d_roots():
    from paper_1309_5050_b200 import Plan
    t = np.arange(400.0)
    x = (np.exp(-0.002 * t) * np.cos(2 * np.pi * t / 23 + 0.5) + 0.7 * np.exp(0.001 * t) * np.sin(2 * np.pi * t / 9))
    p = Plan(x[:, None], (80, 1), dtype="f64", path="fft", block_k=8)
    p.decompose(4)
    lam, mu = p.esprit(range(4))
    ref = [np.exp(-0.002 + s_ * 2j * np.pi / 23) for s_ in (1, -1)] + [np.exp(0.001 + s_ * 2j * np.pi / 9) for s_ in (1, -1)]
    assert max(min(abs(lam - r)) for r in ref) < 1e-9
    assert np.allclose(mu, 1.0)


@pytest.mark.parametrize("path", ["fft", "direct"])
def test_forecast_mssa_c2_vs_oracle(path):
    """Alg. 7 on the c2 MSSA system (8 series, L = 1024, signal group {1..6}) against the vector-forecast
    definition (oracle) on the device's own triples: updated reconstruction + 60 forecast values."""
    w = synth.config2()
    from paper_1309_5050_b200 import Plan
    p = Plan(w.data, w.window, dtype="f32", path=path)
    p.decompose(8)
    g = list(range(6))
    f = p.forecast(g, 60)
    x = np.array(w.data, np.float64).astype(np.float32).astype(np.float64)
    sh = oracle.shapes(x, w.window)
    ref = oracle.vector_forecast(x, sh, p.sigma, p.U().astype(np.float64), p.V().astype(np.float64), g, 60)
    assert f.shape == ref.shape
    assert np.array_equal(np.isnan(f), np.isnan(ref))
    assert relfro(f[~np.isnan(ref)], ref[~np.isnan(ref)]) <= 1e-4


def test_forecast_noiseless_unequal_series_fp64():
    """Noiseless finite-rank MSSA system with series of unequal length (NaN-padded): the forecast continues
    each series exactly (fp64)."""
    def sig(t, c):
        return (1 + 0.1 * c) * np.sin(2 * np.pi * t / 17 + 0.4 * c) + 0.5 * np.exp(-0.002 * t) * np.cos(2 * np.pi * t / 7)
    lens, M = [300, 260, 280], 25
    x = np.full((300, 3), np.nan)
    for c, n in enumerate(lens):
        x[:n, c] = sig(np.arange(n), c)
    from paper_1309_5050_b200 import Plan
    p = Plan(x, (60, 1), dtype="f64", path="direct", block_k=8)
    p.decompose(4)
    f = p.forecast(range(4), M)
    for c, n in enumerate(lens):
        np.testing.assert_allclose(f[:n + M, c], sig(np.arange(n + M), c), atol=1e-9)
        assert np.all(np.isnan(f[n + M:, c]))
