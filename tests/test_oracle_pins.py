"""Pins for the fp64 oracle: each test checks oracle/ against
something the paper or mathematics fixes independently of the oracle's own code —
worked examples printed in the paper (tests/golden/, cited), closed forms
(tests/closed_form.py), library routines for special cases (scipy correlate2d /
hankel), invariants (adjointness, completeness) and brute force on tiny inputs.
CPU only (no GPU marker)."""
import json
import os

import numpy as np
import pytest
import scipy.linalg as sla
import scipy.signal as ssig

import oracle
import closed_form as cf
import synth

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


# ---------------------------------------------------------------- P2: Fig. 4 worked example
def test_fig4_kshape_and_nprime():
    g = _gold("fig4.json")
    nx, ny = g["N_box"]
    n = np.zeros((nx, ny), bool)
    for row, (c0, c1) in g["N_rows"].items():
        n[int(row) - 1, c0 - 1:c1] = True
    assert n.sum() == g["N_count"]
    lx, ly = g["L_box"]
    wm = np.zeros((lx, ly), bool)
    for x, y in g["L"]:
        wm[x - 1, y - 1] = True
    img = np.where(n, 1.0, np.nan)
    sh = oracle.shapes(img, (lx, ly), wmask=wm)
    kx, ky = sh.kmask.shape
    got = sorted((a + 1, b + 1) for a in range(kx) for b in range(ky) if sh.kmask[a, b])
    want = sorted(tuple(p) for p in g["K"])
    assert got == want
    excl = sorted((i + 1, j + 1) for i in range(nx) for j in range(ny)
                  if n[i, j] and not sh.nprime[i, j])
    assert excl == sorted(tuple(p) for p in g["N_minus_Nprime"])
    # 𝔑′ = 𝔎 +‐ 𝔏: the Minkowski sum of the golden sets
    mink = {(a + x - 1, b + y - 1) for (a, b) in g["K"] for (x, y) in g["L"]}
    assert mink == {(i + 1, j + 1) for i in range(nx) for j in range(ny) if sh.nprime[i, j]}


# ---------------------------------------------------------------- P1/Alg. 6: 𝔎 by a second algorithm
@pytest.mark.parametrize("seed", range(12))
def test_kshape_matches_alg6_and_library(seed):
    rng = np.random.default_rng(100 + seed)
    nx, ny = rng.integers(6, 21, size=2)
    lx, ly = rng.integers(1, 6, size=2)
    lx, ly = min(lx, nx), min(ly, ny)
    n = rng.random((nx, ny)) > 0.15
    wm = rng.random((lx, ly)) > 0.3
    wm[0, 0] = True
    img = np.where(n, 1.0, np.nan)
    sh = oracle.shapes(img, (lx, ly), wmask=wm)
    # Alg. 6: v = 𝒯_2DSSAᵀ(I^𝔑)·1_𝔏 over the full origin box, 𝔎 = {v = |𝔏|},
    # evaluated with scipy's 2-D correlation (a library routine)
    v = ssig.correlate2d(n.astype(float), wm.astype(float), mode="valid")
    assert np.array_equal(sh.kmask.astype(bool), np.isclose(v, wm.sum()))
    # weights = diagsums(1_𝔏, 1_𝔎) = full 2-D convolution of the indicators (Alg. 4 step 1)
    w = ssig.convolve2d(sh.kmask.astype(float), wm.astype(float), mode="full")
    assert np.array_equal(sh.weights, np.rint(w).astype(np.int32))


# ---------------------------------------------------------------- P3: weights
def test_weights_1d_golden():
    for case in _gold("weights_1d.json")["cases"]:
        N, L = case["N"], case["L"]
        sh = oracle.shapes(np.zeros((N, 1)), (L, 1))
        assert sh.weights[:, 0].tolist() == case["w"]


def test_weights_rectangle_and_sum():
    nx, ny, lx, ly = 23, 17, 6, 4
    sh = oracle.shapes(np.zeros((nx, ny)), (lx, ly))
    wx = np.minimum.reduce([np.arange(1, nx + 1), np.arange(nx, 0, -1),
                            np.full(nx, min(lx, nx - lx + 1))])
    wy = np.minimum.reduce([np.arange(1, ny + 1), np.arange(ny, 0, -1),
                            np.full(ny, min(ly, ny - ly + 1))])
    assert np.array_equal(sh.weights, np.outer(wx, wy))
    assert sh.weights.sum() == sh.L * sh.K


@pytest.mark.parametrize("dims", [(7, 5, 3, 2), (20, 9, 20, 1), (16, 16, 5, 16), (31, 12, 9, 4)])
def test_shapes_rect_equals_brute_force(dims):
    """oracle.shapes_rect (closed form for full rectangles, used at the c5 size) against the
    brute-force 𝔎 / 𝕎 of oracle.shapes."""
    nx, ny, lx, ly = dims
    a = oracle.shapes_rect(nx, ny, lx, ly)
    b = oracle.shapes(np.zeros((nx, ny)), (lx, ly))
    assert np.array_equal(a.kmask, b.kmask) and np.array_equal(a.weights, b.weights)
    assert np.array_equal(a.nmask, b.nmask) and np.array_equal(a.wmask, b.wmask)


def test_weights_sum_shaped():
    w = synth.small_shaped(seed=3, wmask_drop=4)
    sh = oracle.shapes(w.data, w.window, mask=w.mask, wmask=w.wmask)
    assert sh.weights.sum() == sh.L * sh.K
    assert np.all(sh.weights[sh.nmask == 0] == 0)


# ---------------------------------------------------------------- trajectory matrix structure
def test_trajmat_1d_is_hankel():
    x = np.random.default_rng(0).normal(size=19)
    L = 7
    sh = oracle.shapes(x[:, None], (L, 1))
    X = oracle.trajmat(x[:, None], sh)
    assert np.array_equal(X, sla.hankel(x[:L], x[L - 1:]))  # eq. P:340-352


def test_trajmat_2d_is_hankel_block_hankel():
    rng = np.random.default_rng(1)
    nx, ny, lx, ly = 9, 7, 4, 3
    img = rng.normal(size=(nx, ny))
    sh = oracle.shapes(img, (lx, ly))
    X = oracle.trajmat(img, sh)
    kx, ky = nx - lx + 1, ny - ly + 1
    H = [sla.hankel(img[:lx, j], img[lx - 1:, j]) for j in range(ny)]  # H_j = 𝒯_SSA(col j)
    HbH = np.block([[H[a + b] for b in range(ky)] for a in range(ly)])  # eq. P:2423-2441
    assert np.array_equal(X, HbH)


def test_trajmat_mssa_is_stacked_hankel():
    rng = np.random.default_rng(2)
    N, s, L = 15, 3, 5
    x = rng.normal(size=(N, s))
    sh = oracle.shapes(x, (L, 1))
    X = oracle.trajmat(x, sh)
    st = np.hstack([sla.hankel(x[:L, p], x[L - 1:, p]) for p in range(s)])  # eq. P:944-958
    assert np.array_equal(X, st)


# ---------------------------------------------------------------- P1/P4/P14: products
@pytest.mark.parametrize("seed", range(6))
def test_products_vs_library_correlation(seed):
    rng = np.random.default_rng(200 + seed)
    w = synth.small_shaped(seed=seed, wmask_drop=(seed % 3) * 2)
    img = w.data
    sh = oracle.shapes(img, w.window, mask=w.mask, wmask=w.wmask)
    k = 3
    V = rng.normal(size=(sh.K, k))
    U = rng.normal(size=(sh.L, k))
    Uo = oracle.xv(img, sh, V)
    Vo = oracle.xtu(img, sh, U)
    x = np.where(sh.nmask.astype(bool), img, 0.0)
    lx, ly = w.window
    kx, ky = sh.kx, sh.ky
    km, wm = sh.kmask.astype(bool), sh.wmask.astype(bool)
    for j in range(k):
        Phi = np.zeros((kx, ky)); Phi.T[km.T] = V[:, j]     # factor array (𝔎-lex scatter)
        full = ssig.correlate2d(x, Phi, mode="valid")        # Lx x Ly
        np.testing.assert_allclose(Uo[:, j], full.T[wm.T], rtol=1e-12, atol=1e-10)
        Psi = np.zeros((lx, ly)); Psi.T[wm.T] = U[:, j]     # eigenarray
        full = ssig.correlate2d(x, Psi, mode="valid")        # Kx x Ky
        np.testing.assert_allclose(Vo[:, j], full.T[km.T], rtol=1e-12, atol=1e-10)
    # adjoint identity <Xv,u> = <v,Xᵀu> (P4) and linearity (P14)
    assert abs(np.sum(Uo * U) - np.sum(V * Vo)) <= 1e-10 * np.abs(Uo * U).sum()
    np.testing.assert_allclose(oracle.xv(img, sh, 2 * V[:, :1] - V[:, 1:2]),
                               2 * Uo[:, :1] - Uo[:, 1:2], rtol=1e-12, atol=1e-10)


def test_products_closed_form_c3_twin_sampled():
    """P5 at the full c3 geometry (noiseless twin): sampled rows of both products."""
    w = synth.config3(noise=False)
    sh = oracle.shapes(w.data, w.window)
    rng = np.random.default_rng(5)
    V = rng.normal(size=(sh.K, 2))
    U = rng.normal(size=(sh.L, 2))
    Ucf, Vcf = cf.products(w.terms, sh.lpos(), sh.kpos(), V=V, U=U)
    rows = rng.choice(sh.L, 48, replace=False)
    Ur = oracle.xv_rows(w.data, sh, V, rows)
    np.testing.assert_allclose(Ur, Ucf[rows], rtol=1e-9, atol=1e-9 * np.abs(Ucf).max())
    k0 = 123_456
    Vr = oracle.xtu(w.data, sh, U, kstart=k0, kcount=500)
    np.testing.assert_allclose(Vr, Vcf[k0:k0 + 500], rtol=1e-9, atol=1e-9 * np.abs(Vcf).max())


# ---------------------------------------------------------------- P6/P7: closed-form rank and σ
def test_closed_form_roots_reproduce_image():
    w = synth.config3(noise=False)
    np.testing.assert_allclose(cf.image(w.terms, 64, 48), w.data[:64, :48], atol=1e-11)


def test_c1_noiseless_closed_form_sigma_and_rank():
    w = synth.config1(noise=False)
    sh = oracle.shapes(w.data, w.window)
    s, U, V, sall = oracle.svd_dense(w.data, sh, 10)
    assert cf.rank(w.terms) == 6
    scf = cf.sigma_rect(w.terms, 16, 16, 49, 49)
    np.testing.assert_allclose(s[:6], scf[:6], rtol=1e-11)
    assert sall[6] < 1e-11 * sall[0]
    # the values quoted in SURVEY P7 (0-based reading), 6 significant digits
    np.testing.assert_allclose(s[:6], [671.194, 605.306, 602.303, 565.641, 557.733, 498.232],
                               rtol=2e-6)


def test_separable_twin_rank24_closed_form_sigma():
    """c3 generator (6 terms) at a reduced size: rank 24 and σ = closed form."""
    rng = np.random.default_rng(3)
    terms = synth.draw_terms(rng, 6)
    img = synth.separable_image(72, 60, terms)
    sh = oracle.shapes(img, (12, 10))
    s, U, V, sall = oracle.svd_dense(img, sh, 30)
    scf = cf.sigma_rect(terms, 12, 10, 61, 51)
    assert cf.rank(terms) == 24
    np.testing.assert_allclose(s[:24], scf[:24], rtol=1e-8)
    assert sall[24] < 1e-10 * sall[0]


def test_shaped_closed_form_sigma():
    w = synth.small_shaped(seed=7, noise=False, wmask_drop=3)
    sh = oracle.shapes(w.data, w.window, mask=w.mask, wmask=w.wmask)
    s, U, V, sall = oracle.svd_dense(w.data, sh, 14)
    scf = cf.sigma_shaped(w.terms, sh.lpos(), sh.kpos())
    R = cf.rank(w.terms)
    assert R == 12
    np.testing.assert_allclose(s[:R], scf[:R], rtol=1e-8)
    assert sall[R] < 1e-10 * sall[0]


def test_svd_gram_matches_closed_form():
    """The paper's 'eigen' formulation (S = XXᵀ) against the closed form (noiseless)."""
    rng = np.random.default_rng(8)
    terms = synth.draw_terms(rng, 3)
    img = synth.separable_image(48, 40, terms)
    sh = oracle.shapes(img, (9, 8))
    s, U, V, _ = oracle.svd_gram(img, sh, 12, chunk=500)
    scf = cf.sigma_rect(terms, 9, 8, 40, 33)
    np.testing.assert_allclose(s[:12], scf[:12], rtol=1e-7)
    # V = XᵀU/σ has unit norm and X V = σ U for the top triples
    np.testing.assert_allclose(np.linalg.norm(V, axis=0), 1.0, rtol=1e-9)


# ---------------------------------------------------------------- P8/P9: MSSA theory
def test_example_a2_mssa_eigenvalues():
    for c in _gold("example_a2.json")["cases"]:
        k = np.arange(c["N"])
        f1 = c["A"] * np.cos(2 * np.pi * c["omega"] * k + c["phi1"])
        f2 = c["B"] * np.cos(2 * np.pi * c["omega"] * k + c["phi2"])
        L = c["L"]; Kp = c["N"] - L + 1
        sh = oracle.shapes(np.stack([f1, f2], 1), (L, 1))
        s, *_ = oracle.svd_dense(np.stack([f1, f2], 1), sh, 3)
        lam = s ** 2
        want = (c["A"] ** 2 + c["B"] ** 2) * L * Kp / 4
        np.testing.assert_allclose(lam[:2], [want, want], rtol=1e-10)
        assert lam[2] < 1e-9 * want
        sh1 = oracle.shapes(f1[:, None], (L, 1))
        s1, *_ = oracle.svd_dense(f1[:, None], sh1, 2)
        np.testing.assert_allclose(s1 ** 2, [c["A"] ** 2 * L * Kp / 4] * 2, rtol=1e-10)


def test_table2_ranks():
    g = _gold("table2_ranks.json")
    N = g["N"]
    k = np.arange(1, N + 1)
    for name, ex in g["examples"].items():
        h = [a * np.cos(2 * np.pi * k / p + ph) for a, p, ph in (ex["h1"], ex["h2"])]
        L = 24
        sh1 = oracle.shapes(h[0][:, None], (L, 1))
        s1 = oracle.svd_dense(h[0][:, None], sh1, 6)[3]
        assert int(np.sum(s1 > 1e-8 * s1[0])) == ex["SSA"], name
        x2 = np.stack(h, 1)
        sh2 = oracle.shapes(x2, (L, 1))
        s2 = oracle.svd_dense(x2, sh2, 6)[3]
        assert int(np.sum(s2 > 1e-8 * s2[0])) == ex["MSSA"], name


# ---------------------------------------------------------------- P10-P13: reconstruction
def test_completeness_and_norm_identity():
    rng = np.random.default_rng(9)
    w = synth.small_shaped(seed=4, nx=20, ny=17, window=(5, 4), wmask_drop=2)
    sh = oracle.shapes(w.data, w.window, mask=w.mask, wmask=w.wmask)
    s, U, V, sall = oracle.svd_dense(w.data, sh, min(sh.L, sh.K))
    d = int(np.sum(sall > 1e-13 * sall[0]))
    recs = oracle.reconstruct(w.data, sh, s, U, V, [[i] for i in range(d)])
    tot = np.sum([r[sh.nprime] for r in recs], axis=0)
    np.testing.assert_allclose(tot, w.data[sh.nprime], rtol=1e-11, atol=1e-11)   # eq. P:440-443
    x = np.where(sh.nmask.astype(bool), w.data, 0)
    np.testing.assert_allclose(np.sum(sall ** 2), np.sum(sh.weights * x ** 2), rtol=1e-11)
    # w-correlation matrix is symmetric with unit diagonal
    R = oracle.wcorr(sh, recs[:5])
    np.testing.assert_allclose(np.diag(R), 1.0, rtol=1e-12)
    np.testing.assert_allclose(R, R.T, atol=1e-12)


def test_wcorr_equals_trajectory_inner_products():
    """Pin of oracle.wcorr by the identity it rests on, (Y, Z)_w = ⟨𝒯(Y), 𝒯(Z)⟩_F:
    the weighted inner product of two arrays equals the Frobenius inner product of their
    (independently pinned) trajectory matrices, so dropping the weights w_n, summing outside 𝔑′
    or using the wrong normalisation fails here.  Arbitrary arrays (not only reconstructions),
    shaped 𝔑 and a non-rectangular window."""
    rng = np.random.default_rng(21)
    w = synth.small_shaped(seed=6, nx=23, ny=19, window=(6, 4), wmask_drop=3)
    sh = oracle.shapes(w.data, w.window, mask=w.mask, wmask=w.wmask)
    ys = []
    for _ in range(4):
        y = rng.normal(size=(sh.nx, sh.ny))
        y[~sh.nprime] = np.nan          # reconstructions exist only on 𝔑′
        ys.append(y)
    R = oracle.wcorr(sh, ys)
    T = [oracle.trajmat(np.nan_to_num(y), sh) for y in ys]
    G = np.array([[np.sum(a * b) for b in T] for a in T])
    np.testing.assert_allclose(R, G / np.sqrt(np.outer(np.diag(G), np.diag(G))), rtol=1e-12, atol=1e-13)
    # and the unnormalised form: (Y, Z)_w = Σ_n w_n y_n z_n = ⟨𝒯(Y), 𝒯(Z)⟩_F
    y0, y1 = (np.nan_to_num(y) for y in ys[:2])
    np.testing.assert_allclose(np.sum(sh.weights * y0 * y1), G[0, 1], rtol=1e-12)


def test_contributions_pins():
    """Contributions ||X̃_j||²_w / ||X||²_w: the group of all components reconstructs 𝕏
    on 𝔑′ and contributes exactly 1; each contribution equals ||𝒯(X̃_j)||²_F / ||𝒯(𝕏)||²_F (the
    weighted norm is the trajectory norm, via the independently pinned trajmat)."""
    w = synth.small_shaped(seed=7, nx=21, ny=18, window=(5, 4), wmask_drop=2)
    sh = oracle.shapes(w.data, w.window, mask=w.mask, wmask=w.wmask)
    s, U, V, sall = oracle.svd_dense(w.data, sh, min(sh.L, sh.K))
    d = int(np.sum(sall > 1e-13 * sall[0]))
    groups = [[0], [1, 2], list(range(3, d)), list(range(d))]
    recs = oracle.reconstruct(w.data, sh, s, U, V, groups)
    c = oracle.contributions(sh, recs, w.data)
    assert abs(c[-1] - 1.0) <= 1e-12
    tx = np.sum(oracle.trajmat(np.nan_to_num(w.data), sh) ** 2)
    for g, r in enumerate(recs):
        np.testing.assert_allclose(c[g], np.sum(oracle.trajmat(np.nan_to_num(r), sh) ** 2) / tx, rtol=1e-11)


# ---------------------------------------------------------------- f2 / f3: ESPRIT, vector forecast
def _match_pairs(lam, mu, lam0, mu0):
    return max(min(abs(lam - a) + abs(mu - b)) for a, b in zip(lam0, mu0))


@pytest.mark.parametrize("wmask_drop", [0, 5])
def test_esprit_2d_recovers_closed_form_roots(wmask_drop):
    """2D-ESPRIT: on a noiseless separable array (eq. P:4317-4320) the eigenarrays span the
    exact signal subspace, so the jointly diagonalised shift matrices return the array's (λ_k, μ_k)
    pairs (closed_form.roots) — also for a non-rectangular window (shifts only between cells of 𝔏)."""
    rng = np.random.default_rng(3)
    t = synth.draw_terms(rng, 2)
    img = synth.separable_image(40, 37, t)
    wm = None
    if wmask_drop:
        wm = np.ones((12, 10), bool)
        wm[rng.choice(12, wmask_drop), rng.choice(10, wmask_drop)] = False
        wm[0, 0] = True
    sh = oracle.shapes(img, (12, 10), wmask=wm)
    lam0, mu0, _ = cf.roots(t)
    s, U, V, _ = oracle.svd_dense(img, sh, len(lam0))
    lam, mu = oracle.esprit(sh, U)
    assert _match_pairs(lam, mu, lam0, mu0) < 1e-9


def test_esprit_1d_ls_roots():
    """LS-ESPRIT for one series: the shift matrix's eigenvalues are the roots e^{α±2πiω} of a
    sum of damped sines (Table-2-style finite-rank series, eq. P:4317-4320 in one dimension)."""
    t = np.arange(400.0)
    x = (np.exp(-0.002 * t) * np.cos(2 * np.pi * t / 23 + 0.5) + 0.7 * np.exp(0.001 * t) * np.sin(2 * np.pi * t / 9))
    sh = oracle.shapes(x[:, None], (80, 1))
    s, U, V, _ = oracle.svd_dense(x[:, None], sh, 4)
    lam, _ = oracle.esprit(sh, U)
    ref = np.array([np.exp(-0.002 + s_ * 2j * np.pi / 23) for s_ in (1, -1)] +
                   [np.exp(0.001 + s_ * 2j * np.pi / 9) for s_ in (1, -1)])
    assert max(min(abs(lam - r)) for r in ref) < 1e-10


def test_vector_forecast_continues_finite_rank_series():
    """Vector forecast: for noiseless finite-rank series whose signal subspace is the exact
    span of the eigenvectors, the continued lagged vectors stay on the series' trajectory, so the forecast
    equals the generator's continuation — for one series and for an MSSA system of series of unequal
    length (NaN-padded 2-D packing; common subspace, per-series continuation)."""
    def sig(t, c):
        return (1 + 0.1 * c) * np.sin(2 * np.pi * t / 17 + 0.4 * c) + 0.5 * np.exp(-0.002 * t) * np.cos(2 * np.pi * t / 7)
    M = 25
    for lens in ([300], [300, 260, 280]):
        N = max(lens)
        x = np.full((N, len(lens)), np.nan)
        for c, n in enumerate(lens):
            x[:n, c] = sig(np.arange(n), c)
        sh = oracle.shapes(x, (60, 1))
        s, U, V, _ = oracle.svd_dense(np.nan_to_num(x), sh, 4)
        f = oracle.vector_forecast(np.nan_to_num(x), sh, s, U, V, range(4), M)
        for c, n in enumerate(lens):
            np.testing.assert_allclose(f[:n + M, c], sig(np.arange(n + M), c), atol=1e-11)
            assert np.all(np.isnan(f[n + M:, c]))


def test_m2dssa_packing_is_stacked_trajectory():
    """P13-type packing equivalence for M-2D-SSA (eq. P:3499-3518): two arrays side by side with a one-column
    NaN separator have the trajectory matrix [𝒯(𝕏¹) : 𝒯(𝕏²)] (no window straddles the
    separator)."""
    rng = np.random.default_rng(5)
    x1, x2 = rng.normal(size=(9, 7)), rng.normal(size=(9, 7))
    packed = np.concatenate([x1, np.full((9, 1), np.nan), x2], axis=1)
    win = (3, 2)
    T = oracle.trajmat(np.nan_to_num(packed), oracle.shapes(packed, win))
    T1 = oracle.trajmat(x1, oracle.shapes(x1, win))
    T2 = oracle.trajmat(x2, oracle.shapes(x2, win))
    np.testing.assert_array_equal(T, np.hstack([T1, T2]))


def test_averaging_returns_rank_one_image_exactly():
    """P11: x = c·λ^i μ^j has 𝒯(𝕏) = c·a bᵀ; averaging c·a bᵀ returns 𝕏 on 𝔑′ (shaped)."""
    w = synth.small_shaped(seed=5, wmask_drop=3)
    nx, ny = w.data.shape
    lam, mu, c = 0.97, 1.02, 2.5
    img = c * lam ** np.arange(nx)[:, None] * mu ** np.arange(ny)[None, :]
    sh = oracle.shapes(img, w.window, mask=w.mask, wmask=w.wmask)
    lx, ly = sh.lpos(); kx, ky = sh.kpos()
    a = lam ** lx * mu ** ly
    b = lam ** kx * mu ** ky
    rec = oracle.reconstruct(img, sh, [c], a[:, None], b[:, None], [[0]])[0]
    np.testing.assert_allclose(rec[sh.nprime], img[sh.nprime], rtol=1e-13)
    assert np.all(np.isnan(rec[~sh.nprime]))


def test_c1_noiseless_group_reproduces_signal():
    """P12: the union of the signal triples reconstructs the noiseless input exactly."""
    w = synth.config1(noise=False)
    sh = oracle.shapes(w.data, w.window)
    s, U, V, _ = oracle.svd_dense(w.data, sh, 6)
    rec = oracle.reconstruct(w.data, sh, s, U, V, [list(range(6))])[0]
    np.testing.assert_allclose(rec, w.data, atol=1e-11 * np.abs(w.data).max())


def test_rest_group_and_cells():
    w = synth.config1()
    sh = oracle.shapes(w.data, w.window)
    s, U, V, _ = oracle.svd_dense(w.data, sh, 10)
    recs = oracle.reconstruct(w.data, sh, s, U, V, w.groups, add_rest=True)
    np.testing.assert_allclose(recs[0] + recs[1] + recs[2], w.data, rtol=1e-12, atol=1e-12)
    cells = np.array([0, 5, 64 * 10 + 3, 64 * 64 - 1])
    rc = oracle.reconstruct_cells(sh, s, U, V, w.groups[0], cells)
    np.testing.assert_allclose(rc, recs[0].reshape(-1, order="F")[cells], rtol=1e-12)


def test_packing_equivalences():
    """P13: ShSSA with a full mask = 2D-SSA; 2D-SSA with Lx = 1 = MSSA of the rows."""
    rng = np.random.default_rng(10)
    img = rng.normal(size=(7, 30))
    s0 = oracle.svd_dense(img, oracle.shapes(img, (3, 6)), 5)[0]
    s1 = oracle.svd_dense(img, oracle.shapes(img, (3, 6), mask=np.ones_like(img, bool)), 5)[0]
    np.testing.assert_array_equal(s0, s1)
    # Lx = 1: rows of the (7,30) array are the series; MSSA = 2D packing of the transpose
    sA = oracle.svd_dense(img, oracle.shapes(img, (1, 6)), 7)[3]
    X = np.hstack([sla.hankel(img[p, :6], img[p, 5:]) for p in range(7)])
    np.testing.assert_allclose(sA, np.linalg.svd(X, compute_uv=False)[:len(sA)], rtol=1e-12)
