"""ORACLE — TEST INFRASTRUCTURE ONLY.

Plain fp64 CPU implementation of the multidimensional-SSA hot path of arXiv
1309.5050, written from PAPER.md.  Only ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
module.  It shares no code with the CUDA path and never imports it.

Parts:
  O1 shapes      -- 𝔑, 𝔎 (eq. P:3004-3005, brute force), weights 𝕎
  O2 operator    -- X·V and Xᵀ·U by the naive double loop (eq. P:3020-3028)
  O3 SVD         -- step 2: dense LAPACK SVD of the materialised
                    trajectory matrix (small cases), or the paper's own 'eigen'
                    formulation S = X Xᵀ accumulated in
                    fp64 over column chunks, for mid-size cases
  O4 reconstruct -- steps 3-4 (Alg. 4): diagonal averaging
                    of grouped rank-one sums by brute force, ÷ w on 𝔑′, NaN off 𝔑′

The C loops live in oracle_core.c (compiled to liboracle.so by ``build()``);
numpy/LAPACK is used only for the dense factorisations (a library primitive as
one step) and for array plumbing.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle_core.c")
_SO = os.path.join(_HERE, "liboracle.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile oracle_core.c with gcc (-O2, OpenMP; no fast-math)."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-shared", "-fPIC", "-std=c11",
                               _SRC, "-o", _SO + ".tmp"])
        os.replace(_SO + ".tmp", _SO)
    return _SO


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(_SO)
        i64, p = C.c_int64, C.c_void_p
        L.orc_kshape.restype = i64
        L.orc_kshape.argtypes = [i64, i64, p, i64, i64, p, p]
        L.orc_weights.restype = None
        L.orc_weights.argtypes = [i64, i64, i64, i64, p, p, p]
        L.orc_trajcols.restype = None
        L.orc_trajcols.argtypes = [p, i64, i64, i64, i64, p, p, i64, i64, p]
        L.orc_xv.restype = None
        L.orc_xv.argtypes = [p, i64, i64, i64, i64, p, p, p, i64, p]
        L.orc_xv_rows.restype = None
        L.orc_xv_rows.argtypes = [p, i64, i64, i64, i64, p, p, p, i64, p, i64, p]
        L.orc_xtu_rows.restype = None
        L.orc_xtu_rows.argtypes = [p, i64, i64, i64, i64, p, p, p, i64, i64, i64, p]
        L.orc_diagsums.restype = None
        L.orc_diagsums.argtypes = [i64, i64, i64, i64, p, p, p, p, p, i64, p]
        L.orc_diagsums_cells.restype = None
        L.orc_diagsums_cells.argtypes = [i64, i64, i64, i64, p, p, p, p, p, i64, p, i64, p]
        _lib = L
    return _lib


def _ptr(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _fcol(a, dtype):
    """Column-major (x fastest) contiguous copy: the paper's vec() storage."""
    return np.asfortranarray(np.asarray(a, dtype=dtype))


@dataclass
class Shapes:
    """The shapes of one embedding."""
    nx: int
    ny: int
    lx: int
    ly: int
    nmask: np.ndarray   # (nx, ny) uint8, Fortran order — 𝔑 = finite ∩ mask
    wmask: np.ndarray   # (lx, ly) uint8, Fortran order — 𝔏
    kmask: np.ndarray   # (kx, ky) uint8, Fortran order — 𝔎 (eq. P:3004-3005)
    weights: np.ndarray  # (nx, ny) int32 — w_n = |𝒜_n|

    @property
    def kx(self): return self.nx - self.lx + 1

    @property
    def ky(self): return self.ny - self.ly + 1

    @property
    def L(self): return int(self.wmask.sum())

    @property
    def K(self): return int(self.kmask.sum())

    @property
    def nprime(self):
        """𝔑′ = {w > 0} = 𝔎 +‐ 𝔏 (Alg. 4 step 2)."""
        return self.weights > 0

    def lpos(self):
        """(x, y) of the window cells in 𝔏-lex order."""
        iy, ix = np.nonzero(self.wmask.T)  # iterate y-major so x is fastest
        return ix, iy

    def kpos(self):
        iy, ix = np.nonzero(self.kmask.T)
        return ix, iy


def shapes(img, window, mask=None, wmask=None) -> Shapes:
    """Shape ingestion (𝔑 = non-NaN cells ∩ mask; 𝔏 = wmask, full
    rectangle by default), 𝔎 by brute force (eq. P:3004-3005) and the weights."""
    img = np.asarray(img, dtype=np.float64)
    nx, ny = img.shape
    lx, ly = window
    n = np.isfinite(img)
    if mask is not None:
        n &= np.asarray(mask, dtype=bool)
    nmask = _fcol(n, np.uint8)
    wm = _fcol(np.ones((lx, ly), bool) if wmask is None else wmask, np.uint8)
    kx, ky = nx - lx + 1, ny - ly + 1
    kmask = np.zeros((kx, ky), dtype=np.uint8, order="F")
    lib().orc_kshape(nx, ny, _ptr(nmask), lx, ly, _ptr(wm), _ptr(kmask))
    w = np.zeros((nx, ny), dtype=np.int32, order="F")
    lib().orc_weights(nx, ny, lx, ly, _ptr(wm), _ptr(kmask), _ptr(w))
    return Shapes(nx, ny, lx, ly, nmask, wm, kmask, w)


def shapes_rect(nx, ny, lx, ly) -> Shapes:
    """Shapes of a full Nx x Ny array with the full Lx x Ly window, without the brute-force scan
    (for sizes where it is infeasible, e.g. c5): every origin is valid (eq. P:3004-3005 with 𝔑 the
    whole grid), and the weights are the product of the 1-D hit counts w_i = min(i+1, L, K, N−i)
    (P:3702-3704 per axis; for rectangles 𝕎 = w_x ⊗ w_y, pin P3)."""
    def w1(n, l):
        k = n - l + 1
        i = np.arange(n)
        return np.minimum(np.minimum(i + 1, n - i), min(l, k))
    w = np.asfortranarray(np.outer(w1(nx, lx), w1(ny, ly)).astype(np.int32))
    return Shapes(nx, ny, lx, ly, np.ones((nx, ny), np.uint8, order="F"), np.ones((lx, ly), np.uint8, order="F"),
                  np.ones((nx - lx + 1, ny - ly + 1), np.uint8, order="F"), w)


def _image(img, sh: Shapes):
    """Image with cells outside 𝔑 set to 0 (they never enter 𝒯(𝕏))."""
    x = np.array(img, dtype=np.float64, copy=True)
    x[sh.nmask == 0] = 0.0
    return _fcol(x, np.float64)


def trajmat(img, sh: Shapes, kstart=0, kcount=None) -> np.ndarray:
    """𝒯(𝕏) columns [kstart, kstart+kcount) (eq. P:3020-3028)."""
    kcount = sh.K - kstart if kcount is None else kcount
    out = np.zeros((sh.L, kcount), dtype=np.float64, order="F")
    lib().orc_trajcols(_ptr(_image(img, sh)), sh.nx, sh.ny, sh.lx, sh.ly,
                       _ptr(sh.wmask), _ptr(sh.kmask), kstart, kcount, _ptr(out))
    return out


def xv(img, sh: Shapes, V) -> np.ndarray:
    """U = 𝒯(𝕏)·V, V: |𝔎| x k."""
    V = _fcol(np.atleast_2d(np.asarray(V).T).T, np.float64)
    k = V.shape[1]
    U = np.zeros((sh.L, k), dtype=np.float64, order="F")
    lib().orc_xv(_ptr(_image(img, sh)), sh.nx, sh.ny, sh.lx, sh.ly,
                 _ptr(sh.wmask), _ptr(sh.kmask), _ptr(V), k, _ptr(U))
    return U


def xv_rows(img, sh: Shapes, V, rows) -> np.ndarray:
    V = _fcol(np.atleast_2d(np.asarray(V).T).T, np.float64)
    rows = np.ascontiguousarray(rows, dtype=np.int64)
    k = V.shape[1]
    out = np.zeros((len(rows), k), dtype=np.float64, order="F")
    lib().orc_xv_rows(_ptr(_image(img, sh)), sh.nx, sh.ny, sh.lx, sh.ly,
                      _ptr(sh.wmask), _ptr(sh.kmask), _ptr(V), k, _ptr(rows), len(rows), _ptr(out))
    return out


def xtu(img, sh: Shapes, U, kstart=0, kcount=None) -> np.ndarray:
    """V = 𝒯(𝕏)ᵀ·U (rows [kstart, kstart+kcount) of the result), U: |𝔏| x k."""
    U = _fcol(np.atleast_2d(np.asarray(U).T).T, np.float64)
    k = U.shape[1]
    kcount = sh.K - kstart if kcount is None else kcount
    V = np.zeros((kcount, k), dtype=np.float64, order="F")
    lib().orc_xtu_rows(_ptr(_image(img, sh)), sh.nx, sh.ny, sh.lx, sh.ly,
                       _ptr(sh.wmask), _ptr(sh.kmask), _ptr(U), k, kstart, kcount, _ptr(V))
    return V


def fix_signs(U, V):
    """Sign convention: the largest-|·| entry of each U_i is
    positive; V_i flips with it.  Signs are otherwise arbitrary."""
    U = np.array(U, copy=True); V = np.array(V, copy=True)
    for i in range(U.shape[1]):
        m = np.argmax(np.abs(U[:, i]))
        if U[m, i] < 0:
            U[:, i] *= -1; V[:, i] *= -1
    return U, V


def svd_dense(img, sh: Shapes, r: int):
    """Step 2 on the materialised trajectory matrix: LAPACK gesdd."""
    X = trajmat(img, sh)
    Uf, s, Vt = np.linalg.svd(X, full_matrices=False)
    U, V = fix_signs(Uf[:, :r], Vt[:r].T)
    return s[:r].copy(), U, V, s


def svd_gram(img, sh: Shapes, r: int, chunk: int = 4096):
    """Step 2 exactly as the paper states it ('eigen'):
    S = X Xᵀ (accumulated in fp64 over column chunks of the materialised matrix),
    λ_j, U_j = eigenpairs of S, σ_j = √λ_j, V_j = Xᵀ U_j / σ_j."""
    S = np.zeros((sh.L, sh.L), dtype=np.float64)
    for k0 in range(0, sh.K, chunk):
        B = trajmat(img, sh, k0, min(chunk, sh.K - k0))
        S += B @ B.T
    lam, Ue = np.linalg.eigh(S)
    lam = lam[::-1]; Ue = Ue[:, ::-1]
    sig = np.sqrt(np.clip(lam[:r], 0.0, None))
    U = Ue[:, :r]
    V = xtu(img, sh, U) / sig[None, :]
    U, V = fix_signs(U, V)
    return sig, U, V, np.sqrt(np.clip(lam, 0, None))


def diagsums(sh: Shapes, U, V, coef) -> np.ndarray:
    """Σ_i coef_i · diagsums(U_i, V_i) (Alg. 5 definition) on the nx x ny grid."""
    U = _fcol(np.atleast_2d(np.asarray(U).T).T, np.float64)
    V = _fcol(np.atleast_2d(np.asarray(V).T).T, np.float64)
    coef = np.ascontiguousarray(coef, dtype=np.float64)
    out = np.zeros((sh.nx, sh.ny), dtype=np.float64, order="F")
    lib().orc_diagsums(sh.nx, sh.ny, sh.lx, sh.ly, _ptr(sh.wmask), _ptr(sh.kmask),
                       _ptr(U), _ptr(V), _ptr(coef), len(coef), _ptr(out))
    return out


def diagsums_cells(sh: Shapes, U, V, coef, cells) -> np.ndarray:
    U = _fcol(np.atleast_2d(np.asarray(U).T).T, np.float64)
    V = _fcol(np.atleast_2d(np.asarray(V).T).T, np.float64)
    coef = np.ascontiguousarray(coef, dtype=np.float64)
    cells = np.ascontiguousarray(cells, dtype=np.int64)
    out = np.zeros(len(cells), dtype=np.float64)
    lib().orc_diagsums_cells(sh.nx, sh.ny, sh.lx, sh.ly, _ptr(sh.wmask), _ptr(sh.kmask),
                             _ptr(U), _ptr(V), _ptr(coef), len(coef), _ptr(cells), len(cells),
                             _ptr(out))
    return out


def reconstruct(img, sh: Shapes, sigma, U, V, groups, add_rest=False):
    """Steps 3-4 (Alg. 4):
    X̃_g = diagsums(Σ_{i∈I_g} σ_i U_i V_iᵀ) / 𝕎 on 𝔑′, NaN elsewhere
    (values exist only inside the resulting mask).  With add_rest,
    one more array 𝕏 − Σ_g X̃_g on 𝔑′ (the residual group of eq. P:440-443)."""
    w = sh.weights.astype(np.float64)
    npr = sh.nprime
    outs = []
    for g in groups:
        g = list(g)
        num = diagsums(sh, np.asarray(U)[:, g], np.asarray(V)[:, g], np.asarray(sigma)[g])
        rec = np.full((sh.nx, sh.ny), np.nan)
        rec[npr] = num[npr] / w[npr]
        outs.append(rec)
    if add_rest:
        x = np.asarray(img, dtype=np.float64)
        rest = np.full((sh.nx, sh.ny), np.nan)
        tot = np.zeros(int(npr.sum()))
        for rec in outs:
            tot += rec[npr]
        rest[npr] = x[npr] - tot
        outs.append(rest)
    return outs


def reconstruct_cells(sh: Shapes, sigma, U, V, group, cells):
    """X̃_g at listed flat cells (i + nx*j), for sampled checks at full sizes."""
    g = list(group)
    num = diagsums_cells(sh, np.asarray(U)[:, g], np.asarray(V)[:, g], np.asarray(sigma)[g], cells)
    w = sh.weights.reshape(-1, order="F")[np.asarray(cells)].astype(np.float64)
    out = np.full(len(cells), np.nan)
    ok = w > 0
    out[ok] = num[ok] / w[ok]
    return out


def contributions(sh: Shapes, recs, img):
    """Contributions of reconstructed components: ||X̃_j||²_w / ||X||²_w with the
    weighted norm ||Y||²_w = Σ_n w_n y_n² (w_n = 0 off 𝔑′, cells outside 𝔑 are 0)."""
    w = sh.weights.astype(np.float64)
    x = np.where(sh.nmask.astype(bool), np.nan_to_num(np.asarray(img, dtype=np.float64)), 0.0)
    den = np.sum(w * x * x)
    return np.array([np.sum(w * np.nan_to_num(r) ** 2) for r in recs]) / den


def _shift_pairs(wmask, axis):
    """Row pairs (a, b) of the 𝔏-lex basis with cell b = cell a shifted by one along `axis`
    (0 = x, 1 = y), both cells in 𝔏 (the shifted sub-arrays of the eigenarrays)."""
    wm = np.asarray(wmask, dtype=bool)
    lx, ly = wm.shape
    idx = -np.ones((lx, ly), dtype=np.int64)
    iy, ix = np.nonzero(wm.T)
    idx[ix, iy] = np.arange(len(ix))
    a, b = [], []
    for x in range(lx):
        for y in range(ly):
            x2, y2 = (x + 1, y) if axis == 0 else (x, y + 1)
            if x2 < lx and y2 < ly and idx[x, y] >= 0 and idx[x2, y2] >= 0:
                a.append(idx[x, y]); b.append(idx[x2, y2])
    return np.array(a, dtype=np.int64), np.array(b, dtype=np.int64)


def esprit(sh: Shapes, U, comb=0.6180339887 + 0.3090169944j):
    """LS-ESPRIT / 2D-ESPRIT parameter estimation on the eigenvectors U (L x r) of a group
    (P:675-682 LS-ESPRIT after Roy & Kailath; P:2843-2857 2D-ESPRIT after Rouquette & Najim):
    the shift matrices Φ_x = (U_x↑)^† U_x↓ and Φ_y = (U_y↑)^† U_y↓ solve the least-squares problems
    U_x↑ Φ_x ≈ U_x↓ between the eigenarrays restricted to 𝔏 and to 𝔏 shifted by one along x (y);
    their joint diagonalisation (eigenvectors T of a generic combination Φ_x + c·Φ_y) gives the pairs
    λ_k = (T⁻¹Φ_xT)_kk, μ_k = (T⁻¹Φ_yT)_kk with x_{m,n} = Σ_k c_k λ_k^m μ_k^n.  For a window of one
    column (1-D SSA / MSSA) only λ is defined (μ = 1)."""
    U = np.asarray(U, dtype=np.float64)
    a, b = _shift_pairs(sh.wmask, 0)
    phx = np.linalg.lstsq(U[a], U[b], rcond=None)[0]
    if sh.ly == 1:
        lam = np.linalg.eigvals(phx)
        return lam, np.ones_like(lam)
    a, b = _shift_pairs(sh.wmask, 1)
    phy = np.linalg.lstsq(U[a], U[b], rcond=None)[0]
    _, T = np.linalg.eig(phx + comb * phy)
    Ti = np.linalg.inv(T)
    return np.diag(Ti @ phx @ T), np.diag(Ti @ phy @ T)


def vector_forecast(img, sh: Shapes, sigma, U, V, group, M):
    """Column vector forecast of 1-D SSA / MSSA (window (L, 1); series = columns of the 2-D packing)
    by its definition: with P = [U_j, j ∈ group], π = its last row, ν² = ||π||²,
    Π = the orthogonal projector onto span of the first L−1 rows of P and R_L = Σ_j π_j P_j[:-1]/(1−ν²)
    (eq. P:1376), every series p continues its reconstructed lagged vectors X̂_1..X̂_{K_p} by
    Z_j = (Π Z_{j−1}[1:]; R_Lᵀ Z_{j−1}[1:]) for j = K_p+1 .. K_p+M+L−1 (eq. P:1442-1460); the diagonal
    averaging of [Z_1 : ... : Z_{K_p+M+L−1}] gives z_1..z_{N_p+M+L−1}, of which z_1..z_{N_p+M}
    (reconstruction updated near the end, then the M forecast values) are returned, one column per
    series, NaN-padded to max_p N_p + M."""
    assert sh.ly == 1, "vector forecast: 1-D SSA / MSSA packing (window (L, 1))"
    g = list(group)
    P = np.asarray(U, dtype=np.float64)[:, g]
    Vg = np.asarray(V, dtype=np.float64)[:, g] * np.asarray(sigma, dtype=np.float64)[g][None, :]
    L = P.shape[0]
    pi = P[-1, :]
    nu2 = float(pi @ pi)
    Pl = P[:-1, :]
    Pi = Pl @ np.linalg.pinv(Pl)                      # projector onto span(first L−1 rows)
    R = (Pl @ pi) / (1.0 - nu2)
    kx, ky = sh.kx, sh.ky
    kmask = np.asarray(sh.kmask, dtype=bool)
    Kp = kmask.sum(axis=0)
    out = np.full((int(Kp.max()) + L - 1 + M, ky), np.nan)
    koff = np.concatenate([[0], np.cumsum(Kp)])
    for p in range(ky):
        K = int(Kp[p])
        if K == 0:
            continue
        Z = [P @ Vg[koff[p] + j] for j in range(K)]    # X̂_j = Σ_i σ_i U_i V_i[κ_j]
        for _ in range(M + L - 1):
            f = Z[-1][1:]
            Z.append(np.concatenate([Pi @ f, [R @ f]]))
        Zm = np.array(Z).T                               # L x (K + M + L − 1)
        n = L + Zm.shape[1] - 1
        num = np.zeros(n); cnt = np.zeros(n)
        for c in range(Zm.shape[1]):
            num[c:c + L] += Zm[:, c]
            cnt[c:c + L] += 1
        N = K + L - 1
        out[:N + M, p] = (num / cnt)[:N + M]
    return out


def wcorr(sh: Shapes, recs):
    """w-correlation matrix of reconstructed components:
    ρ_ij = (X̃_i, X̃_j)_w / (‖X̃_i‖_w ‖X̃_j‖_w), (Y, Z)_w = Σ_n w_n y_n z_n."""
    w = sh.weights.astype(np.float64)
    npr = sh.nprime
    M = np.array([np.nan_to_num(r)[npr] for r in recs])
    G = (M * w[npr][None, :]) @ M.T
    d = np.sqrt(np.diag(G))
    return G / np.outer(d, d)
