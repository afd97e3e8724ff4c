"""GPU parity tests: the CUDA path (through the C ABI) against the fp64 oracle on the
same seeded inputs, at the tolerances of BASELINE.json's north star:
  * integer shape data (𝔎, 𝕎, counts): bit-exact
  * operator products: relative Frobenius error <= 1e-5 (fp32) / 1e-12 (fp64)
  * singular values: relative error <= 1e-4 where the oracle relgap >= 1e-3 and
    σ_i >= τ σ_1 (reading Q10), |Δσ_i| <= 1e-6 σ_1 below the floor / in clusters
  * grouped reconstructions: relative Frobenius error <= 1e-4 on 𝔑′ (NaN elsewhere)
"""
import numpy as np
import pytest

import closed_form as cf
import oracle
import synth
from parity_util import TAU, check_sigma, gap_groups

pytestmark = pytest.mark.gpu

FP32_PROD_TOL = 1e-5
FP64_PROD_TOL = 1e-12


@pytest.fixture(scope="module", autouse=True)
def _require_gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device")
    from paper_1309_5050_b200 import build
    build.build()


def _plan(w, dtype=None, **kw):
    from paper_1309_5050_b200 import Plan
    return Plan(w.data, w.window, mask=w.mask, wmask=w.wmask, dtype=dtype or w.dtype,
                block_k=kw.pop("block_k", w.block_k), **kw)


def _oracle_input(w, dtype):
    """The exact values the GPU sees (fp32 configs are rounded once)."""
    x = np.array(w.data, dtype=np.float64)
    if dtype == "f32":
        x = x.astype(np.float32).astype(np.float64)
    return x


from parity_util import relfro  # noqa: E402


def _cases():
    return {
        "shaped_small": synth.small_shaped(seed=11),
        "shaped_wmask": synth.small_shaped(seed=12, wmask_drop=6, nx=37, ny=45, window=(9, 6)),
        "shaped_tiny": synth.small_shaped(seed=13, nx=12, ny=10, window=(4, 3), n_holes=1, wmask_drop=2),
        "c1": synth.config1(),
    }


# ---------------------------------------------------------------- shapes: bit-exact
@pytest.mark.parametrize("name", ["shaped_small", "shaped_wmask", "shaped_tiny", "c1"])
def test_shapes_bit_exact(name):
    w = _cases()[name]
    p = _plan(w)
    sh = oracle.shapes(w.data, w.window, mask=w.mask, wmask=w.wmask)
    assert p.L == sh.L and p.K == sh.K
    assert np.array_equal(p.kmask(), sh.kmask.astype(bool))
    assert np.array_equal(p.weights(), sh.weights)
    assert p.n_excluded == int((sh.nmask.astype(bool) & ~sh.nprime).sum())


def test_shapes_fig4_bit_exact():
    import json, os
    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "fig4.json")))
    nx, ny = g["N_box"]
    n = np.zeros((nx, ny), bool)
    for row, (c0, c1) in g["N_rows"].items():
        n[int(row) - 1, c0 - 1:c1] = True
    wm = np.zeros(tuple(g["L_box"]), bool)
    for x, y in g["L"]:
        wm[x - 1, y - 1] = True
    img = np.where(n, 1.0, np.nan)
    from paper_1309_5050_b200 import Plan
    p = Plan(img, tuple(g["L_box"]), wmask=wm)
    got = sorted((a + 1, b + 1) for a, b in zip(*np.nonzero(p.kmask())))
    assert got == sorted(tuple(v) for v in g["K"])
    assert p.n_excluded == len(g["N_minus_Nprime"])


def test_shapes_c4_full_size_bit_exact():
    w = synth.config4()
    p = _plan(w)
    sh = oracle.shapes(w.data, w.window, mask=w.mask)
    assert p.K == sh.K
    assert np.array_equal(p.kmask(), sh.kmask.astype(bool))
    assert np.array_equal(p.weights(), sh.weights)


# ---------------------------------------------------------------- products
PATHS = ["direct", "fft"]


@pytest.mark.parametrize("path", PATHS)
@pytest.mark.parametrize("name", ["shaped_small", "shaped_wmask", "shaped_tiny", "c1"])
@pytest.mark.parametrize("dtype", ["f32", "f64"])
@pytest.mark.parametrize("k", [1, 5, 37, 70])
def test_products_small(name, dtype, k, path):
    w = _cases()[name]
    p = _plan(w, dtype=dtype, path=path)
    assert p.path == path
    x = _oracle_input(w, dtype)
    sh = oracle.shapes(x, w.window, mask=w.mask, wmask=w.wmask)
    rng = np.random.default_rng(k)
    V = rng.normal(size=(sh.K, k))
    U = rng.normal(size=(sh.L, k))
    npd = np.float32 if dtype == "f32" else np.float64
    V = V.astype(npd).astype(np.float64); U = U.astype(npd).astype(np.float64)
    tol = FP32_PROD_TOL if dtype == "f32" else FP64_PROD_TOL
    assert relfro(p.matmul(V), oracle.xv(x, sh, V)) <= tol
    assert relfro(p.matmul(U, transpose=True), oracle.xtu(x, sh, U)) <= tol


def test_products_device_tensors_and_ld():
    import torch
    w = synth.small_shaped(seed=21)
    p = _plan(w)
    x = _oracle_input(w, "f32")
    sh = oracle.shapes(x, w.window, mask=w.mask)
    V = torch.randn(sh.K, 7, device="cuda", dtype=torch.float32)
    U = p.matmul(V)
    ref = oracle.xv(x, sh, V.double().cpu().numpy())
    assert relfro(U.double().cpu().numpy(), ref) <= FP32_PROD_TOL


@pytest.mark.parametrize("path", PATHS)
def test_products_c2_mssa(path):
    w = synth.config2()
    p = _plan(w, path=path)
    x = _oracle_input(w, "f32")
    sh = oracle.shapes(x, w.window)
    rng = np.random.default_rng(2)
    V = rng.normal(size=(sh.K, 32)).astype(np.float32).astype(np.float64)
    U = rng.normal(size=(sh.L, 32)).astype(np.float32).astype(np.float64)
    assert relfro(p.matmul(V), oracle.xv(x, sh, V)) <= FP32_PROD_TOL
    assert relfro(p.matmul(U, transpose=True), oracle.xtu(x, sh, U)) <= FP32_PROD_TOL


@pytest.mark.parametrize("path", PATHS)
@pytest.mark.parametrize("cfg", ["c3", "c4"])
def test_products_full_size_sampled(cfg, path):
    """Full BASELINE sizes, block k = 32: sampled output rows against the oracle."""
    w = synth.get(cfg)
    p = _plan(w, path=path)
    x = _oracle_input(w, "f32")
    sh = oracle.shapes(x, w.window, mask=w.mask)
    rng = np.random.default_rng(3)
    k = 32
    V = rng.normal(size=(sh.K, k)).astype(np.float32)
    U = rng.normal(size=(sh.L, k)).astype(np.float32)
    Ug = p.matmul(V)
    Vg = p.matmul(U, transpose=True)
    rows = rng.choice(sh.L, 24, replace=False)
    ref = oracle.xv_rows(x, sh, V.astype(np.float64), rows)
    assert relfro(Ug[rows], ref) <= FP32_PROD_TOL
    k0 = int(rng.integers(0, sh.K - 2000))
    refv = oracle.xtu(x, sh, U.astype(np.float64), kstart=k0, kcount=2000)
    assert relfro(Vg[k0:k0 + 2000], refv) <= FP32_PROD_TOL
    # adjoint identity over the whole block (P4), fp64 host dots
    lhs = np.sum(Ug.astype(np.float64) * U.astype(np.float64))
    rhs = np.sum(V.astype(np.float64) * Vg.astype(np.float64))
    assert abs(lhs - rhs) <= 1e-5 * np.sqrt(np.sum(Ug.astype(np.float64) ** 2) * np.sum(U.astype(np.float64) ** 2))


@pytest.mark.parametrize("path", PATHS)
def test_products_closed_form_c3_twin(path):
    """P5: noiseless c3 geometry, products against the separable closed form."""
    w = synth.config3(noise=False)
    p = _plan(w, path=path)
    from paper_1309_5050_b200 import Plan  # noqa: F401
    sh = oracle.shapes(w.data, w.window)
    rng = np.random.default_rng(4)
    V = rng.normal(size=(sh.K, 4)).astype(np.float32).astype(np.float64)
    U = rng.normal(size=(sh.L, 4)).astype(np.float32).astype(np.float64)
    Ucf, Vcf = cf.products(w.terms, sh.lpos(), sh.kpos(), V=V, U=U)
    # the GPU sees the fp32-rounded image: allow the input rounding (≈6e-8 relative)
    assert relfro(p.matmul(V), Ucf) <= 2e-5
    assert relfro(p.matmul(U, transpose=True), Vcf) <= 2e-5


def test_products_closed_form_c5_twin_sampled():
    """P5 at the c5 size (4096², window 256², K ≈ 14.75M, k = 64), FFT path: sampled
    output entries of both products against the separable closed form."""
    w = synth.config5(noise=False)
    p = _plan(w, path="fft")
    import torch
    rng = np.random.default_rng(5)
    k = 64
    V = torch.randn(p.K, k, device="cuda", dtype=torch.float32, generator=torch.Generator("cuda").manual_seed(1))
    U = torch.randn(p.L, k, device="cuda", dtype=torch.float32, generator=torch.Generator("cuda").manual_seed(2))
    Ug = p.matmul(V)[:, :4].double().cpu().numpy()
    Vrows = rng.choice(p.K, 4096, replace=False)
    Vg = p.matmul(U, transpose=True)[torch.as_tensor(Vrows, device="cuda")][:, :4].double().cpu().numpy()
    lx, ly = np.meshgrid(np.arange(256), np.arange(256), indexing="ij")
    lpos = (lx.reshape(-1, order="F"), ly.reshape(-1, order="F"))
    kpos_all = (np.arange(p.K) % 3841, np.arange(p.K) // 3841)
    Vh = V[:, :4].double().cpu().numpy()
    Uh = U[:, :4].double().cpu().numpy()
    Ucf = cf.products(w.terms, lpos, kpos_all, V=Vh)
    Vcf = cf.products(w.terms, lpos, (kpos_all[0][Vrows], kpos_all[1][Vrows]), U=Uh)
    # image values reach ~1e7 here (e^{±8} per axis): fp32 input rounding and fp32 FFT
    # rounding are both relative to the largest entries
    assert relfro(Ug, Ucf) <= 2e-5
    assert relfro(Vg, Vcf) <= 2e-5


# ---------------------------------------------------------------- decomposition + reconstruction
def _check_recon(p, x, sh, s_or, U_or, V_or, groups, tol=1e-4):
    recs = p.reconstruct(groups)
    ref = oracle.reconstruct(x, sh, s_or, U_or, V_or, groups)
    npr = sh.nprime
    for g, (a, b) in enumerate(zip(recs, ref)):
        assert np.array_equal(np.isnan(a), np.isnan(b))
        assert relfro(a[npr], b[npr]) <= tol, (g, groups[g], relfro(a[npr], b[npr]))


@pytest.mark.parametrize("path", PATHS)
def test_decompose_c1_fp64(path):
    w = synth.config1()
    p = _plan(w, path=path)
    x = _oracle_input(w, "f64")
    sh = oracle.shapes(x, w.window)
    s_or, U_or, V_or, s_all = oracle.svd_dense(x, sh, 10)
    info = p.decompose(10)
    assert info["n_converged"] == 10
    assert len(check_sigma(p.sigma, s_all, 10, TAU["f64"])) >= 6
    np.testing.assert_allclose(p.sigma, s_or, rtol=1e-8)
    _check_recon(p, x, sh, s_or, U_or, V_or, w.groups + [list(range(6))], tol=1e-8)
    # the residual group returns the image (eq. P:440-443)
    recs = p.reconstruct(w.groups, add_rest=True)
    np.testing.assert_allclose(recs[0] + recs[1] + recs[2], x, rtol=1e-10, atol=1e-10)


@pytest.mark.parametrize("path", PATHS)
def test_decompose_c2_mssa_fp32(path):
    w = synth.config2()
    p = _plan(w, path=path)
    x = _oracle_input(w, "f32")
    sh = oracle.shapes(x, w.window)
    s_or, U_or, V_or, s_all = oracle.svd_dense(x, sh, 17)
    p.decompose(16)
    assert len(check_sigma(p.sigma, s_all, 16, TAU[path])) >= 4
    _check_recon(p, x, sh, s_or, U_or, V_or, [g for g in w.groups if max(g) < 6])


@pytest.mark.parametrize("path", PATHS)
@pytest.mark.parametrize("name", ["shaped_small", "shaped_wmask"])
def test_decompose_shaped_small(name, path):
    w = _cases()[name]
    p = _plan(w, path=path)
    x = _oracle_input(w, "f32")
    sh = oracle.shapes(x, w.window, mask=w.mask, wmask=w.wmask)
    r = w.r
    s_or, U_or, V_or, s_all = oracle.svd_dense(x, sh, r + 1)
    p.decompose(r)
    check_sigma(p.sigma, s_all, r, TAU[path])
    groups = gap_groups(s_all, r)
    if groups:
        _check_recon(p, x, sh, s_or, U_or, V_or, groups)


@pytest.mark.parametrize("path", PATHS)
def test_reconstruct_from_oracle_triples_c1_and_shaped(path):
    for w, dt in [(synth.config1(), "f64"), (synth.small_shaped(seed=14, wmask_drop=4), "f32")]:
        p = _plan(w, dtype=dt, path=path)
        x = _oracle_input(w, dt)
        sh = oracle.shapes(x, w.window, mask=w.mask, wmask=w.wmask)
        s_or, U_or, V_or, _ = oracle.svd_dense(x, sh, 6)
        p.set_triples(s_or, U_or)
        groups = [[0], [1, 2], [3, 4, 5], [0, 1, 2, 3, 4, 5]]
        recs = p.reconstruct(groups, add_rest=True)
        ref = oracle.reconstruct(x, sh, s_or, U_or, V_or, groups, add_rest=True)
        tol = 1e-11 if dt == "f64" else 2e-5
        for a, b in zip(recs, ref):
            assert np.array_equal(np.isnan(a), np.isnan(b))
            m = ~np.isnan(b)
            assert relfro(a[m], b[m]) <= tol


@pytest.mark.parametrize("path", PATHS)
def test_c3_noiseless_closed_form(path):
    """P6/P7/P12 at the full c3 size: rank 24, σ = closed form, {1..24} = the image."""
    w = synth.config3(noise=False)
    p = _plan(w, path=path)
    info = p.decompose(32, allow_not_converged=True)
    s_cf = cf.sigma_rect(w.terms, 64, 64, 449, 449)
    s = p.sigma
    np.testing.assert_allclose(s[:24], s_cf[:24], rtol=1e-4)
    assert np.all(s[24:] <= 1e-5 * s[0])
    rec = p.reconstruct([list(range(24))])[0]
    x = _oracle_input(w, "f32")
    assert relfro(rec, x) <= 1e-4
    assert info["n_block_products"] > 0


def test_c5_noiseless_closed_form_sigma():
    """P7 at the full c5 size (4096², window 256², K ≈ 14.75M, r = 50, k = 64): σ of the
    noiseless twin against the closed form, with reading Q10's floor for fp32 products."""
    w = synth.config5(noise=False)
    p = _plan(w, path="fft")
    info = p.decompose(50)
    assert info["n_converged"] == 50
    s = p.sigma
    s_cf = np.concatenate([cf.sigma_rect(w.terms, 256, 256, 3841, 3841), np.zeros(8)])
    assert cf.rank(w.terms) == 48
    checked = check_sigma(s, s_cf, 50, TAU["fft"])
    assert len(checked) >= 8
    # reading Q10: the library reports the same floor and how many triples lie below it
    assert info["sigma_floor_rel"] == TAU["fft"]
    assert info["n_below_floor"] == int(np.sum(s < TAU["fft"] * s[0]))


@pytest.mark.parametrize("case", ["c1", "shaped"])
def test_wcor_and_contributions(case):
    """Row f1: the w-correlation matrix and the contributions ||X̃_g||²_w / ||X||²_w
     of the device reconstructions against the oracle's (pinned by the trajectory
    inner-product identity, tests/test_oracle_pins.py)."""
    if case == "c1":
        w, dt, groups = synth.config1(), "f64", [[0], [1], [2], [3], [4, 5], list(range(10))]
    else:
        w, dt = synth.small_shaped(seed=23, wmask_drop=3), "f32"
        groups = [[0], [1, 2], [3, 4, 5], list(range(6))]
    p = _plan(w, dtype=dt)
    x = _oracle_input(w, dt)
    sh = oracle.shapes(x, w.window, mask=w.mask, wmask=w.wmask)
    r = max(max(g) for g in groups) + 1
    p.decompose(r)
    R, con = p.wcor(groups, contributions=True)
    np.testing.assert_allclose(np.diag(R), 1.0, rtol=1e-12)
    np.testing.assert_allclose(R, R.T, atol=1e-12)
    # the oracle on the device's own triples isolates the w-correlation / contribution arithmetic
    recs = oracle.reconstruct(x, sh, p.sigma, p.U().astype(np.float64), p.V().astype(np.float64), groups)
    tol = 1e-9 if dt == "f64" else 2e-5
    np.testing.assert_allclose(R, oracle.wcorr(sh, recs), atol=tol)
    np.testing.assert_allclose(con, oracle.contributions(sh, recs, x), rtol=tol, atol=tol)


# ---------------------------------------------------------------- error behaviour
def test_errors():
    from paper_1309_5050_b200 import Plan, SSAError
    x = np.random.default_rng(0).normal(size=(20, 15))
    with pytest.raises(SSAError) as e:
        Plan(x, (21, 3))
    assert e.value.status == 2
    with pytest.raises(SSAError) as e:
        Plan(x, (1, 1))
    assert e.value.status == 2
    m = np.ones_like(x, bool); m[:, 7] = False; m[10, :] = False
    with pytest.raises(SSAError) as e:
        Plan(x, (12, 9), mask=m)
    assert e.value.status == 3
    p = Plan(x, (5, 4))
    with pytest.raises(SSAError) as e:
        p.reconstruct([[0]])
    assert e.value.status == 9
    with pytest.raises(SSAError) as e:
        p.decompose(21)
    assert e.value.status == 4
    p.decompose(3)
    # a group index beyond the computed rank continues the decomposition ...
    p.reconstruct([[0, 3]])
    assert p.r == 4
    # ... up to min(L, K) (here L = 20)
    with pytest.raises(SSAError) as e:
        p.reconstruct([[0, 20]])
    assert e.value.status == 4


# ---------------------------------------------------------------- band partition (rows a12, (e)) on one GPU
@pytest.mark.parametrize("path", ["direct", "fft", "tc"])
def test_band_products_and_decomposition(path):
    """The multi-GPU band plan on one GPU with an identity all-reduce: a rank's plan is
    its sub-image (band + (Ly−1)-column halo); its X·V is the band's partial sum, its Xᵀ·U the band's
    rows, and the decomposition is the SVD of the band operator X[:, κ ∈ band].  The two bands'
    partials add up to the global X·V and their Xᵀ·U rows stack to the global one."""
    from paper_1309_5050_b200.dist import LocalComm, band_plan, band_slices
    w = synth.small_shaped(seed=51, nx=700, ny=10, window=(300, 3), n_holes=2) if path == "tc" else \
        synth.small_shaped(seed=52, nx=40, ny=33, window=(7, 5), wmask_drop=3)
    x = _oracle_input(w, "f32")
    sh = oracle.shapes(x, w.window, mask=w.mask, wmask=w.wmask)
    rng = np.random.default_rng(8)
    U = rng.normal(size=(sh.L, 5)).astype(np.float32).astype(np.float64)
    Vfull = rng.normal(size=(sh.K, 5)).astype(np.float32).astype(np.float64)
    xv_sum, xtu_rows, koff = np.zeros((sh.L, 5)), [], 0
    for rank in range(2):
        (y0, y1), (c0, c1) = band_slices(sh.ny, sh.ly, 2, rank)
        band = oracle.Shapes(sh.nx, sh.ny, sh.lx, sh.ly, sh.nmask, sh.wmask, sh.kmask.copy(order="F"), sh.weights)
        band.kmask[:, :y0] = 0
        band.kmask[:, y1:] = 0
        p = band_plan(w.data, w.window, LocalComm(rank, 2), mask=w.mask, wmask=w.wmask, dtype="f32", path=path,
                      block_k=8)
        kb = int(band.kmask.sum())
        assert p.K == kb and p.ny == c1 - c0
        V = Vfull[koff:koff + kb]
        Ub = p.matmul(V)
        assert relfro(Ub, oracle.xv(x, band, V)) <= FP32_PROD_TOL
        xv_sum += Ub
        Vb = p.matmul(U, transpose=True)
        assert relfro(Vb, oracle.xtu(x, band, U)) <= FP32_PROD_TOL
        xtu_rows.append(Vb)
        koff += kb
        if rank == 0:
            s_or, _, _, s_all = oracle.svd_dense(x, band, 5)
            p.decompose(4)
            check_sigma(p.sigma, s_all, 4, TAU[path])
    assert koff == sh.K
    assert relfro(xv_sum, oracle.xv(x, sh, Vfull)) <= FP32_PROD_TOL
    assert relfro(np.concatenate(xtu_rows), oracle.xtu(x, sh, U)) <= FP32_PROD_TOL


@pytest.mark.parametrize("world", [2, 3])
def test_band_partition_two_threads_end_to_end(world):
    """The whole band-partitioned path on one GPU: `world` host threads, each with its band plan
    (sub-image only) and a thread communicator whose all-reduce really sums the ranks' buffers.
    The decomposition (X·V partials and K-side Grams summed across the bands) gives the σ of the
    global operator, and the assembled reconstructions (bands' numerators and hit counts summed
    over the halos), the rest group, the w-correlations and the contributions equal the global
    ones — all against the oracle."""
    import torch
    from threadcomm import ThreadComm, ThreadGroup, run_threads
    from paper_1309_5050_b200.dist import band_plan
    w = synth.small_shaped(seed=53, nx=48, ny=41, window=(8, 6), n_holes=3, wmask_drop=4)
    x = _oracle_input(w, "f32")
    sh = oracle.shapes(x, w.window, mask=w.mask, wmask=w.wmask)
    s_or, U_or, V_or, s_all = oracle.svd_dense(x, sh, 9)
    groups = gap_groups(s_all, 6)
    assert groups
    grp = ThreadGroup(world)

    def rank_fn(r):
        st = torch.cuda.Stream()
        with torch.cuda.stream(st):
            comm = ThreadComm(grp, r)
            p = band_plan(w.data, w.window, comm, mask=w.mask, wmask=w.wmask, dtype="f32", path="fft", block_k=8,
                          stream=st.cuda_stream)
            info = p.decompose(6)
            recs = p.reconstruct(groups, add_rest=True)
            R, con = p.wcor(groups, contributions=True)
            return p.sigma, info, recs, R, con, comm.calls

    res = run_threads(world, rank_fn)
    for sig, info, recs, R, con, calls in res:
        assert calls > 0 and info["n_converged"] == 6
        np.testing.assert_array_equal(sig, res[0][0])     # identical on every rank
        check_sigma(sig, s_all, 6, TAU["fft"])
        ref = oracle.reconstruct(x, sh, s_or, U_or, V_or, groups, add_rest=True)
        for a, b in zip(recs, ref):
            assert a.shape == (sh.nx, sh.ny)
            assert np.array_equal(np.isnan(a), np.isnan(b))
            m = ~np.isnan(b)
            assert relfro(a[m], b[m]) <= 1e-4
        ro = oracle.reconstruct(x, sh, s_or, U_or, V_or, groups)
        np.testing.assert_allclose(R, oracle.wcorr(sh, ro), atol=1e-4)
        np.testing.assert_allclose(con, oracle.contributions(sh, ro, x), rtol=1e-4)
