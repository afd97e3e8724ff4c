"""GPU parity at the full BASELINE.json sizes (VERDICT r1 "close the parity gaps"): the
decomposition and the reconstructions of c3 (noisy, 2D-SSA 512², L = 4096) and c4 (Shaped
2D-SSA 1024² disc with holes, irregular 𝔎) against the fp64 oracle, their noiseless twins
against the closed-form spectrum (pin P7), the c5 reconstruction kernels at sampled cells,
and the U / V getters on non-square shapes — all through the C ABI.

Tolerances (north star, readings Q9-Q11):
  σ: 1e-4 relative where relgap >= 1e-3 and σ_i >= τ_path·σ_1, else |Δσ| <= 1e-6·σ_1;
  reconstructions: 1e-4 relative Frobenius on 𝔑′, NaN pattern exact;
  subspaces (U_g, V_g of a gap-bounded group): projector distance <= 1e-4.
"""
import numpy as np
import pytest

import closed_form as cf
import oracle
import synth
from parity_util import TAU, check_sigma, gap_groups, projector_err, relfro

pytestmark = pytest.mark.gpu

REC_TOL = 1e-4
PROJ_TOL = 1e-4


@pytest.fixture(scope="module", autouse=True)
def _require_gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device")
    from paper_1309_5050_b200 import build
    build.build()


def _plan(w, path="auto", **kw):
    from paper_1309_5050_b200 import Plan
    return Plan(w.data, w.window, mask=w.mask, wmask=w.wmask, dtype=w.dtype,
                block_k=kw.pop("block_k", w.block_k), path=path, **kw)


def _x32(w):
    """The values the fp32 plan sees (rounded once), in fp64 for the oracle."""
    return np.array(w.data, dtype=np.float64).astype(np.float32).astype(np.float64)


_ORACLE = {}


def _oracle_svd(cfg, r):
    """O3 'eigen' on the noisy config, computed once per session."""
    if cfg not in _ORACLE:
        w = synth.get(cfg)
        x = _x32(w)
        sh = oracle.shapes(x, w.window, mask=w.mask)
        s, U, V, s_all = oracle.svd_gram(x, sh, r)
        _ORACLE[cfg] = (w, x, sh, s, U, V, s_all)
    return _ORACLE[cfg]


def _tau(p):
    return max(TAU[p.path_xv], TAU[p.path_xtu])


def _check_decomp_vs_oracle(p, cfg, r, groups):
    w, x, sh, s_or, U_or, V_or, s_all = _oracle_svd(cfg, r)
    info = p.decompose(r)
    assert info["n_converged"] == r
    assert info["max_rel_residual"] <= 1e-6
    res = p.residuals
    assert np.all(res <= 1e-6 * p.sigma[0] * (1 + 1e-12))
    checked = check_sigma(p.sigma, s_all, r, _tau(p))
    # the decomposition's U and V against the oracle's, per group (sign/rotation invariant)
    U = p.U()
    V = p.V()
    for g in groups:
        eu = projector_err(U[:, g], U_or[:, g])
        ev = projector_err(V[:, g], V_or[:, g])
        assert eu <= PROJ_TOL and ev <= PROJ_TOL, (g, eu, ev)
    # reconstructions (Alg. 4) against the oracle's from its own triples
    recs = p.reconstruct(groups)
    ref = oracle.reconstruct(x, sh, s_or, U_or, V_or, groups)
    npr = sh.nprime
    for g, a, b in zip(groups, recs, ref):
        assert np.array_equal(np.isnan(a), np.isnan(b)), g
        e = relfro(a[npr], b[npr])
        assert e <= REC_TOL, (g, e)
    return checked


# ------------------------------------------------------------------------------------ c4
@pytest.mark.parametrize("path", ["fft", "direct", "tc"])
def test_c4_noiseless_twin_sigma_closed_form(path):
    """P6/P7 on the irregular 𝔎 of c4 (disc r = 500 with 40 holes, window 48²): rank 32, the
    top 20 σ against the closed form summed over 𝔏 and 𝔎 (closed_form.sigma_shaped)."""
    w = synth.config4(noise=False)
    p = _plan(w, path=path)
    sh = oracle.shapes(w.data, w.window, mask=w.mask)
    assert p.K == sh.K
    s_cf = cf.sigma_shaped(w.terms, sh.lpos(), sh.kpos())
    assert cf.rank(w.terms) == 32
    info = p.decompose(20)
    assert info["n_converged"] == 20
    checked = check_sigma(p.sigma, s_cf, 20, _tau(p))
    assert len(checked) >= 16


@pytest.mark.parametrize("path", ["fft", "direct", "tc"])
def test_c4_full_size_vs_oracle(path):
    """c4 (noisy): σ vs the oracle's 'eigen' SVD, U/V subspaces and the reconstructions of the
    Q9 groups (the five 4-clusters and the prefix {1..20}) on 𝔑′ with the exact NaN pattern."""
    w = synth.config4()
    p = _plan(w, path=path)
    groups = [list(range(4 * g, 4 * g + 4)) for g in range(5)] + [list(range(20))]
    _, _, _, _, _, _, s_all = _oracle_svd("c4", 20)
    assert gap_groups(s_all, 20, 1e-1) == groups[:5]
    checked = _check_decomp_vs_oracle(p, "c4", 20, groups)
    assert len(checked) >= 20


# ------------------------------------------------------------------------------------ c3
@pytest.mark.parametrize("path", ["fft", "direct", "tc"])
def test_c3_noisy_full_size_vs_oracle(path):
    """c3 (noisy 512², window 64², r = 32): σ vs the oracle (the noise pairs, relgap ~1e-5, at
    1e-6·σ_1), U/V subspaces and reconstructions of the six signal 4-clusters and {1..24}."""
    w = synth.config3()
    p = _plan(w, path=path)
    groups = [list(range(4 * g, 4 * g + 4)) for g in range(6)] + [list(range(24))]
    checked = _check_decomp_vs_oracle(p, "c3", 32, groups)
    assert len(checked) >= 20


# ------------------------------------------------------------------------------------ c5
def test_c5_reconstruction_sampled_cells():
    """Rows a10/a11 at the c5 size (4096², window 256², K = 14.75M): the device averaging of two
    gap-bounded groups against the oracle's brute-force diagonal averaging (Alg. 4), fed the device's
    own triples (σ, U, V = XᵀU/σ), at 240 uniformly sampled cells (an unbiased estimate of the
    relative Frobenius error on 𝔑′, bar 1e-4) and at corner / border / centre cells, where 𝕎 is
    small and the fp32 FFT's absolute rounding (uniform over the grid) is divided by few hits: those
    are held to the bar's per-element scale, |Δ| <= 1e-4 · RMS of the sampled reconstruction."""
    w = synth.config5()
    p = _plan(w, path="fft")
    info = p.decompose(50)
    assert info["n_converged"] == 50
    sh = oracle.shapes_rect(4096, 4096, 256, 256)
    s_cf = cf.sigma_rect(synth.config5(noise=False).terms, 256, 256, 3841, 3841)
    groups = [[0, 1, 2, 3], [4, 5, 6, 7]]
    assert all(g in gap_groups(np.concatenate([s_cf, [0.0]]), 12, 1e-1) for g in groups)
    recs = p.reconstruct(groups, device=True)
    rng = np.random.default_rng(55)
    ri, rj = rng.integers(0, 4096, 240), rng.integers(0, 4096, 240)
    ei = np.array([0, 4095, 0, 4095, 255, 3840, 2048, 0, 4095, 1, 2048])
    ej = np.array([0, 0, 4095, 4095, 255, 3840, 17, 2048, 2048, 1, 2048])
    U = p.U().astype(np.float64)
    Vd = p.V(device=True)
    sig = p.sigma
    for g, rec in zip(groups, recs):
        Vg = np.asfortranarray(Vd[:, g].double().cpu().numpy())
        rh = rec.double().cpu().numpy()
        ref_r = oracle.reconstruct_cells(sh, sig[g], U[:, g], Vg, range(len(g)), ri + 4096 * rj)
        ref_e = oracle.reconstruct_cells(sh, sig[g], U[:, g], Vg, range(len(g)), ei + 4096 * ej)
        e = relfro(rh[ri, rj], ref_r)
        assert e <= REC_TOL, (g, e)
        rms = np.sqrt(np.mean(ref_r ** 2))
        de = np.abs(rh[ei, ej] - ref_e).max() / rms
        assert de <= REC_TOL, (g, de)
        del Vg


# --------------------------------------------------------------------- U / V getters
def _rect_case(seed=61, nx=50, ny=31, window=(9, 4)):
    rng = np.random.default_rng(seed)
    t = synth.draw_terms(rng, 3)
    img = synth.separable_image(nx, ny, t) + rng.normal(0, 0.3, (nx, ny))
    return synth.Workload("rect_nonsquare", img, window, r=6, block_k=8, dtype="f32", terms=t)


@pytest.mark.parametrize("path", ["direct", "fft"])
@pytest.mark.parametrize("dtype", ["f32", "f64"])
@pytest.mark.parametrize("case", ["shaped", "rect"])
def test_uv_getters_nonsquare(case, dtype, path):
    """ssa_get_u / ssa_get_v on non-square shapes (SURVEY §4 'transposition trap'): U in 𝔏-lex
    order and V in 𝔎-lex order span the oracle's singular subspaces per gap-bounded group, V_i
    equals Xᵀ U_i / σ_i and both are unit columns."""
    w = synth.small_shaped(seed=17, nx=40, ny=33, window=(7, 5), wmask_drop=3) if case == "shaped" else _rect_case()
    from paper_1309_5050_b200 import Plan
    p = Plan(w.data, w.window, mask=w.mask, wmask=w.wmask, dtype=dtype, path=path, block_k=8)
    x = np.array(w.data, dtype=np.float64)
    if dtype == "f32":
        x = x.astype(np.float32).astype(np.float64)
    sh = oracle.shapes(x, w.window, mask=w.mask, wmask=w.wmask)
    s_or, U_or, V_or, s_all = oracle.svd_dense(x, sh, 8)
    p.decompose(6)
    U, V = p.U().astype(np.float64), p.V().astype(np.float64)
    assert U.shape == (sh.L, 6) and V.shape == (sh.K, 6)
    tol = 1e-5 if dtype == "f32" else 1e-10
    np.testing.assert_allclose(np.linalg.norm(U, axis=0), 1.0, atol=tol)
    np.testing.assert_allclose(np.linalg.norm(V, axis=0), 1.0, atol=10 * tol)
    assert relfro(V, oracle.xtu(x, sh, U) / p.sigma[None, :]) <= 10 * tol
    for g in gap_groups(s_all, 6, 1e-2):
        e = max(projector_err(U[:, g], U_or[:, g]), projector_err(V[:, g], V_or[:, g]))
        assert e <= (PROJ_TOL if dtype == "f32" else 1e-9), (g, e)
    # device getters return the same arrays
    Ud = p.U(device=True).double().cpu().numpy()
    assert np.array_equal(Ud, U)


# ---------------------------------------------------------- continuation / precision / residuals
def test_auto_continuation_and_warm_start():
    """reconstructing by more components than were computed continues the decomposition
    automatically; a second decomposition is warm-started from the stored eigenvectors."""
    w = synth.config1()
    p = _plan(w, path="direct")
    x = np.array(w.data, dtype=np.float64)
    sh = oracle.shapes(x, w.window)
    s_or, U_or, V_or, _ = oracle.svd_dense(x, sh, 10)
    p.decompose(4)
    assert p.r == 4
    rec = p.reconstruct([list(range(8))])[0]
    assert p.r == 8
    np.testing.assert_allclose(p.sigma, s_or[:8], rtol=1e-8)
    ref = oracle.reconstruct(x, sh, s_or, U_or, V_or, [list(range(8))])[0]
    assert relfro(rec, ref) <= 1e-8
    info = p.decompose(10)
    assert info["warm_start_cols"] == 8
    np.testing.assert_allclose(p.sigma, s_or[:10], rtol=1e-8)
    from paper_1309_5050_b200 import SSAError
    with pytest.raises(SSAError) as e:
        p.reconstruct([[0, 256]])
    assert e.value.status == 4


def test_precision_option_and_residuals():
    """opts.precision: an fp64 input decomposed in fp32 arithmetic matches the fp32
    plan of the rounded input; residual bounds are reported per triple."""
    w = synth.small_shaped(seed=19)
    from paper_1309_5050_b200 import Plan
    p = Plan(np.asarray(w.data, np.float64), w.window, mask=w.mask, precision="f32", path="fft", block_k=8)
    assert p.dtype == "f32"
    info = p.decompose(4)
    q = Plan(np.asarray(w.data, np.float32), w.window, mask=w.mask, path="fft", block_k=8)
    q.decompose(4)
    np.testing.assert_allclose(p.sigma, q.sigma, rtol=1e-6)
    res = p.residuals
    assert res.shape == (4,) and np.all(res >= 0) and np.all(res <= 1e-6 * p.sigma[0] * (1 + 1e-9))
    assert info["sigma_floor_rel"] == TAU["fft"]
