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


# ------------------------------------------------------------------ f4: eigen variant, M-2D-SSA packing
@pytest.mark.parametrize("path", ["direct", "fft"])
def test_eigen_svd_method_c1_fp64(path):
    """svd.method = "eigen": S = XXᵀ from the fast products, full eigendecomposition; on c1
    (fp64, L = 256) σ, reconstructions and residuals against the oracle's dense SVD."""
    w = synth.config1()
    from paper_1309_5050_b200 import Plan
    p = Plan(w.data, w.window, dtype="f64", path=path, svd_method="eigen")
    x = np.array(w.data, np.float64)
    sh = oracle.shapes(x, w.window)
    s_or, U_or, V_or, _ = oracle.svd_dense(x, sh, 10)
    info = p.decompose(10)
    np.testing.assert_allclose(p.sigma, s_or, rtol=1e-10)
    assert info["max_rel_residual"] <= 1e-9
    recs = p.reconstruct(w.groups + [list(range(6))])
    ref = oracle.reconstruct(x, sh, s_or, U_or, V_or, w.groups + [list(range(6))])
    for a, b in zip(recs, ref):
        assert relfro(a, b) <= 1e-9


def test_eigen_svd_method_mssa_fp64():
    """The eigen method on an MSSA system (8 series, L = 512, fp64) against the oracle."""
    w = synth.config2(L=512)
    from paper_1309_5050_b200 import Plan
    p = Plan(w.data, w.window, dtype="f64", path="fft", svd_method="eigen")
    x = np.array(w.data, np.float64)
    sh = oracle.shapes(x, w.window)
    s_or, _, _, _ = oracle.svd_dense(x, sh, 12)
    p.decompose(12)
    np.testing.assert_allclose(p.sigma, s_or, rtol=1e-9)


@pytest.mark.parametrize("path", ["direct", "fft"])
def test_m2dssa_packing(path):
    """M-2D-SSA (eq. P:3499-3518) as a shaped array: two images side by side with a one-column NaN separator
    (P:3512-3515); the decomposition is the SVD of [𝒯(𝕏¹) : 𝒯(𝕏²)] (the stacked trajectory matrices, formed
    here from the oracle's trajmat of each image) and each image's reconstruction uses the common basis."""
    rng = np.random.default_rng(71)
    t = synth.draw_terms(rng, 2)
    x1 = synth.separable_image(30, 25, t) + rng.normal(0, 0.2, (30, 25))
    x2 = 0.7 * synth.separable_image(30, 25, t) + rng.normal(0, 0.2, (30, 25))
    packed = np.concatenate([x1, np.full((30, 1), np.nan), x2], axis=1)
    win = (6, 5)
    from paper_1309_5050_b200 import Plan
    p = Plan(packed, win, dtype="f64", path=path, block_k=8)
    sh = oracle.shapes(packed, win)
    T1 = oracle.trajmat(x1, oracle.shapes(x1, win))
    T2 = oracle.trajmat(x2, oracle.shapes(x2, win))
    s_stack = np.linalg.svd(np.hstack([T1, T2]), compute_uv=False)
    assert p.K == T1.shape[1] + T2.shape[1]
    p.decompose(6)
    np.testing.assert_allclose(p.sigma, s_stack[:6], rtol=1e-9)
    s_or, U_or, V_or, _ = oracle.svd_dense(np.nan_to_num(packed), sh, 6)
    rec = p.reconstruct([[0, 1, 2, 3]])[0]
    ref = oracle.reconstruct(np.nan_to_num(packed), sh, s_or, U_or, V_or, [[0, 1, 2, 3]])[0]
    assert np.array_equal(np.isnan(rec), np.isnan(ref))
    assert relfro(rec[~np.isnan(ref)], ref[~np.isnan(ref)]) <= 1e-9
