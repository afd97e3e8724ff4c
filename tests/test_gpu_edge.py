"""GPU edge cases of the hot path against the fp64 oracle (all product paths that apply):

* 1-D SSA as the N x 1 shaped case and MSSA with unequal series lengths
  (NaN padding, P:1658-1687 / the 2-D packing of P:3340-3354);
* degenerate windows: Lx = 1 (row-wise embedding), a window one short of the array
  (K = 2 columns), 1 x Ly windows on a 2-D array;
* a rank-one separable image: r = 1 reconstructs it exactly (pin P11);
* noiseless finite-rank input: the group of all signal triples returns the input
  (pin P12) and the trailing σ are ~0 (reading Q15);
* r = min(L, K) (full rank request) on a tiny case, and block width k > L.
Tolerances: products 1e-5 (fp32) / 1e-12 (fp64); σ per reading Q10; reconstructions 1e-4 / 1e-10.
"""
import numpy as np
import pytest

import oracle
import synth
from parity_util import TAU, check_sigma
from test_gpu_parity import FP32_PROD_TOL, FP64_PROD_TOL, relfro

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _require_gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device")
    from paper_1309_5050_b200 import build
    build.build()


def _plan(x, window, dtype, path, mask=None, wmask=None, block_k=8):
    from paper_1309_5050_b200 import Plan
    return Plan(x, window, mask=mask, wmask=wmask, dtype=dtype, path=path, block_k=block_k)


def _rounded(x, dtype):
    x = np.array(x, dtype=np.float64)
    return x.astype(np.float32).astype(np.float64) if dtype == "f32" else x


def _check_products(p, x, window, dtype, mask=None, wmask=None, k=3, seed=0):
    sh = oracle.shapes(x, window, mask=mask, wmask=wmask)
    assert p.L == sh.L and p.K == sh.K
    rng = np.random.default_rng(seed)
    V = _rounded(rng.normal(size=(sh.K, k)), dtype)
    U = _rounded(rng.normal(size=(sh.L, k)), dtype)
    tol = FP32_PROD_TOL if dtype == "f32" else FP64_PROD_TOL
    assert relfro(p.matmul(V), oracle.xv(x, sh, V)) <= tol
    assert relfro(p.matmul(U, transpose=True), oracle.xtu(x, sh, U)) <= tol
    return sh


PATHS = ["direct", "fft"]


@pytest.mark.parametrize("path", PATHS)
@pytest.mark.parametrize("dtype", ["f32", "f64"])
def test_ssa_1d_as_n_by_1(path, dtype):
    """Plain 1-D SSA: an N x 1 array with window (L, 1) — SSA as a special case of ShSSA."""
    rng = np.random.default_rng(1)
    t = np.arange(300.0)
    x = _rounded((np.sin(2 * np.pi * t / 17) + 0.01 * t + rng.normal(0, 0.2, t.size))[:, None], dtype)
    p = _plan(x, (60, 1), dtype, path)
    sh = _check_products(p, x, (60, 1), dtype)
    s_or, U_or, V_or, s_all = oracle.svd_dense(x, sh, 7)
    p.decompose(6)
    check_sigma(p.sigma, s_all, 6, TAU[path] if dtype == "f32" else TAU["f64"])
    recs = p.reconstruct([[0, 1, 2, 3, 4, 5]], add_rest=True)
    np.testing.assert_allclose(recs[0] + recs[1], x, rtol=0, atol=(1e-4 if dtype == "f32" else 1e-10) * np.abs(x).max())


@pytest.mark.parametrize("path", PATHS)
def test_mssa_unequal_lengths_nan_padded(path):
    """Series of unequal lengths, NaN-padded to a common length (K_p differ per series)."""
    w = synth.config2(seed=31, n=500, s=3, L=100)
    x = np.array(w.data, dtype=np.float64)
    x[450:, 1] = np.nan        # series 1 has 450 points
    x[380:, 2] = np.nan        # series 2 has 380 points
    x = _rounded(x, "f32")
    p = _plan(x, (100, 1), "f32", path)
    sh = _check_products(p, np.nan_to_num(x), (100, 1), "f32", mask=np.isfinite(x))
    assert sh.K == (500 - 99) + (450 - 99) + (380 - 99)
    s_or, U_or, V_or, s_all = oracle.svd_dense(np.nan_to_num(x), sh, 6)
    p.decompose(5)
    check_sigma(p.sigma, s_all, 5, TAU[path])
    rec = p.reconstruct([[0, 1, 2, 3, 4]])[0]
    # values exist only on 𝔑′: NaN exactly where the input is NaN here
    assert np.array_equal(np.isnan(rec), ~np.isfinite(x))


@pytest.mark.parametrize("path", PATHS)
@pytest.mark.parametrize("window", [(1, 5), (39, 3), (6, 1), (40, 32)])
def test_degenerate_windows(path, window):
    """Lx = 1 (row-wise), a window one column/row short of the array (K = 2), 1-D windows."""
    rng = np.random.default_rng(2)
    x = _rounded(rng.normal(size=(40, 33)), "f32")
    p = _plan(x, window, "f32", path)
    _check_products(p, x, window, "f32", k=4)


@pytest.mark.parametrize("path", PATHS)
def test_rank_one_image_reconstructs_exactly(path):
    """x[i, j] = λ^i μ^j (one real exponential per axis): a rank-1 trajectory matrix; r = 1
    and its reconstruction is x (pin P11)."""
    i = np.arange(48.0)[:, None]
    j = np.arange(37.0)[None, :]
    x = _rounded(3.0 * np.exp(0.01 * i) * np.exp(-0.02 * j), "f32")
    p = _plan(x, (9, 7), "f32", path)
    info = p.decompose(1)
    sh = oracle.shapes(x, (9, 7))
    s_or, _, _, _ = oracle.svd_dense(x, sh, 2)
    assert abs(p.sigma[0] - s_or[0]) <= 1e-5 * s_or[0]
    rec = p.reconstruct([[0]])[0]
    assert relfro(rec, x) <= 1e-5
    assert info["n_converged"] == 1


@pytest.mark.parametrize("path", PATHS)
def test_noiseless_finite_rank_union_returns_signal(path):
    """c1's noiseless twin (rank 6, fp64): σ_7.. ~0 and the union of the 6 signal triples
    reconstructs the signal (pin P12; reading Q15 for the excess triples)."""
    w = synth.config1(noise=False)
    x = np.array(w.data, dtype=np.float64)
    p = _plan(x, w.window, "f64", path, block_k=16)
    p.decompose(8, allow_not_converged=True)
    assert np.all(p.sigma[6:] <= 1e-6 * p.sigma[0])
    rec = p.reconstruct([list(range(6))])[0]
    assert relfro(rec, x) <= 1e-10


def test_full_rank_request_and_wide_block():
    """r = min(L, K) on a tiny case (every triple), block width larger than L."""
    rng = np.random.default_rng(3)
    x = rng.normal(size=(9, 8))
    p = _plan(x, (3, 2), "f64", "direct", block_k=16)
    sh = oracle.shapes(x, (3, 2))
    r = min(sh.L, sh.K)
    s_or, U_or, V_or, s_all = oracle.svd_dense(x, sh, r)
    p.decompose(r)
    np.testing.assert_allclose(p.sigma, s_or, rtol=1e-9, atol=1e-12 * s_or[0])
    recs = p.reconstruct([list(range(r))])
    np.testing.assert_allclose(recs[0], x, rtol=1e-9, atol=1e-9)


_DEFER_SCRIPT = r"""
import json
import synth
from paper_1309_5050_b200 import Plan
w = synth.get("c4")
p = Plan(w.data, w.window, mask=w.mask, wmask=w.wmask, dtype=w.dtype, block_k=w.block_k)
info = p.decompose(w.r)
print(json.dumps({"sigma": [float(s) for s in p.sigma], "n_block_products": info["n_block_products"],
                  "max_rel_residual": info["max_rel_residual"]}))
"""


def test_deferred_orthonormalisation_matches_full():
    """The K-side orthonormalisation deferred past a Ritz check (c4: checks after every
    block pair) gives the decomposition of the undeferred solver: same block products, σ to the
    fp32 floor, residual bound below tol in both."""
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = {}
    for flag in ("0", "1"):
        env = dict(os.environ, SSA_DEFER=flag, PYTHONPATH=root + os.pathsep + os.environ.get("PYTHONPATH", ""))
        r = subprocess.run([sys.executable, "-c", _DEFER_SCRIPT], capture_output=True, text=True, env=env, cwd=root,
                           timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        out[flag] = json.loads(r.stdout.strip().splitlines()[-1])
    a, b = out["0"], out["1"]
    assert a["n_block_products"] == b["n_block_products"]
    s0, s1 = np.array(a["sigma"]), np.array(b["sigma"])
    assert np.max(np.abs(s0 - s1)) <= 1e-6 * s0[0]
    assert a["max_rel_residual"] <= 1e-6 and b["max_rel_residual"] <= 1e-6


def test_release_workspace_between_decompositions():
    """The per-thread K-side workspace (grow-only across decompositions) can be released between
    decompositions; the next decomposition re-allocates it and returns the same triples."""
    from paper_1309_5050_b200 import Plan, release_workspace
    w = synth.get("c3")
    s = []
    for _ in range(2):
        p = Plan(w.data, w.window, dtype=w.dtype, block_k=w.block_k)
        p.decompose(w.r)
        s.append(np.array(p.sigma))
        p.close()
        release_workspace()
    assert np.array_equal(s[0], s[1])


def test_large_block_cache_reuse_across_streams():
    """Freed device blocks >= 8 MB are kept per host thread by exact size and handed to the next plan of
    the shape, also when that plan runs on another stream: the reuse is ordered after the
    previous plan's last kernel by an event.  Same input, three plans on alternating streams, products
    issued back to back without a host synchronisation in between: identical results."""
    import torch
    from paper_1309_5050_b200 import Plan
    w = synth.get("c3")
    rng = np.random.default_rng(5)
    K = (w.data.shape[0] - w.window[0] + 1) * (w.data.shape[1] - w.window[1] + 1)
    V = rng.normal(size=(K, w.block_k)).astype(np.float32)
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    outs, sig = [], []
    for i in range(3):
        st = streams[i % 2]
        with torch.cuda.stream(st):
            p = Plan(w.data, w.window, dtype=w.dtype, block_k=w.block_k, stream=st.cuda_stream)
            outs.append(np.array(p.matmul(V)))
            p.decompose(w.r)
            sig.append(np.array(p.sigma))
            p.close()
    assert np.array_equal(outs[0], outs[1]) and np.array_equal(outs[0], outs[2])
    np.testing.assert_allclose(sig[1], sig[0], rtol=1e-6)
    np.testing.assert_allclose(sig[2], sig[0], rtol=1e-6)
