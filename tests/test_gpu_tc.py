"""GPU parity of the tensor-core (tcgen05, 3xTF32) product path against the fp64 oracle.

The tensor-core kernel serves products whose output box has >= 256 rows (polyphase
tiles of 128·S rows along x); the others fall back to FFT / direct, and each test checks
which path the plan actually chose.  Tolerances are BASELINE.json's north star:
products <= 1e-5 relative Frobenius, σ per reading Q10, reconstructions <= 1e-4.
"""
import numpy as np
import pytest

import oracle
import synth
from parity_util import TAU, check_sigma
from test_gpu_parity import FP32_PROD_TOL, _check_recon, _oracle_input, relfro

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _require_gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device")
    from paper_1309_5050_b200 import build
    build.build()


def _plan(w, **kw):
    from paper_1309_5050_b200 import Plan
    return Plan(w.data, w.window, mask=w.mask, wmask=w.wmask, dtype="f32",
                block_k=kw.pop("block_k", w.block_k), **kw)


def _products(w, k, seed=0):
    x = _oracle_input(w, "f32")
    sh = oracle.shapes(x, w.window, mask=w.mask, wmask=w.wmask)
    rng = np.random.default_rng(seed)
    V = rng.normal(size=(sh.K, k)).astype(np.float32).astype(np.float64)
    U = rng.normal(size=(sh.L, k)).astype(np.float32).astype(np.float64)
    return x, sh, V, U


def _cases():
    return {
        # MSSA packings: ragged K_p (not a multiple of 32 / 128), ragged L
        "mssa_ragged": synth.config2(seed=21, n=777, s=3, L=300),
        "mssa_long_window": synth.config2(seed=22, n=1500, s=2, L=1100),
        # 2-D, window wider than 128 rows, shaped (holes + window mask)
        "shaped_wide": synth.small_shaped(seed=23, nx=520, ny=26, window=(150, 5), n_holes=3, wmask_drop=4),
        "rect_wide": synth.small_shaped(seed=24, nx=700, ny=12, window=(300, 3), n_holes=0),
    }


@pytest.mark.parametrize("name", ["mssa_ragged", "mssa_long_window", "shaped_wide", "rect_wide"])
@pytest.mark.parametrize("k", [1, 5, 32, 37, 70])
def test_tc_products_small(name, k):
    w = _cases()[name]
    p = _plan(w, path="tc")
    x, sh, V, U = _products(w, k, seed=k)
    assert p.path_xtu == "tc"                      # output box = 𝔎 box, >= 256 rows here
    assert p.path_xv == ("tc" if w.window[0] >= 256 else p.path_xv)
    assert relfro(p.matmul(V), oracle.xv(x, sh, V)) <= FP32_PROD_TOL
    assert relfro(p.matmul(U, transpose=True), oracle.xtu(x, sh, U)) <= FP32_PROD_TOL


def test_tc_products_c2_full():
    w = synth.config2()
    p = _plan(w, path="tc")
    assert p.path_xv == "tc" and p.path_xtu == "tc"
    x, sh, V, U = _products(w, 32, seed=2)
    assert relfro(p.matmul(V), oracle.xv(x, sh, V)) <= FP32_PROD_TOL
    assert relfro(p.matmul(U, transpose=True), oracle.xtu(x, sh, U)) <= FP32_PROD_TOL


@pytest.mark.parametrize("cfg", ["c3", "c4"])
def test_tc_products_full_size_sampled(cfg):
    """c3/c4 at full size: Xᵀ·U on the tensor cores (𝔎 box rows 449 / 977), X·V falls
    back (𝔏 box has 64 / 48 rows); sampled rows against the oracle (a long reduction:
    4096 / 2304 terms, which exposes accumulation-precision problems)."""
    w = synth.get(cfg)
    p = _plan(w, path="tc")
    assert p.path_xtu == "tc"
    x = _oracle_input(w, "f32")
    sh = oracle.shapes(x, w.window, mask=w.mask)
    rng = np.random.default_rng(7)
    U = rng.normal(size=(sh.L, 32)).astype(np.float32)
    Vg = p.matmul(U, transpose=True)
    k0 = int(rng.integers(0, sh.K - 3000))
    refv = oracle.xtu(x, sh, U.astype(np.float64), kstart=k0, kcount=3000)
    assert relfro(Vg[k0:k0 + 3000], refv) <= FP32_PROD_TOL


def test_tc_decompose_c2():
    w = synth.config2()
    p = _plan(w, path="tc")
    x = _oracle_input(w, "f32")
    sh = oracle.shapes(x, w.window)
    s_or, U_or, V_or, s_all = oracle.svd_dense(x, sh, 17)
    p.decompose(16)
    assert len(check_sigma(p.sigma, s_all, 16, TAU["tc"])) >= 4
    _check_recon(p, x, sh, s_or, U_or, V_or, [g for g in w.groups if max(g) < 6])


def test_auto_choice_is_measured_and_valid():
    """AUTO picks per product among the available paths; whatever it picks is parity-green."""
    w = synth.config2()
    p = _plan(w)
    assert p.path_xv in ("tc", "fft", "direct") and p.path_xtu in ("tc", "fft", "direct")
    x, sh, V, U = _products(w, 32, seed=9)
    assert relfro(p.matmul(V), oracle.xv(x, sh, V)) <= FP32_PROD_TOL
    assert relfro(p.matmul(U, transpose=True), oracle.xtu(x, sh, U)) <= FP32_PROD_TOL
