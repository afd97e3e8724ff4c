"""Seeded synthetic inputs for the BASELINE.json workloads (configs c1..c5).

This module holds NO SSA arithmetic: it only evaluates the generator formulas
that BASELINE.json states for each configuration, with the seeding/draw-order
reading Q12 of SURVEY.md §8(c) (also restated in DESIGN.md §3).  Both the oracle
tests and the CUDA path take their inputs from here; nothing else is shared.

Conventions
-----------
* Images are numpy arrays ``img[i, j]`` of shape ``(Nx, Ny)`` with ``i`` = paper's
  x (row, downward) and ``j`` = paper's y (column), 0-based (reading Q12).
  The paper's vec() is column-major (x fastest); callers that need
  that storage use ``np.asfortranarray``.
* MSSA systems are ``(N, s)`` arrays, series as columns (2D packing),
  NaN-padded when lengths differ.
* Random numbers: ``numpy.random.default_rng(seed)`` (PCG64).  Draw order: the
  per-term parameter vectors a, alpha, beta, omega, nu, phi, psi (each of length
  n_terms), then the noise over the (Nx, Ny) grid in C order, then (c4 only) the
  40 holes, each drawn as (h, w, i0, j0).
"""
from __future__ import annotations

from dataclasses import dataclass, field
import numpy as np

TWO_PI = 2.0 * np.pi


@dataclass
class Workload:
    """One synthetic input: the data array plus everything needed to describe it."""
    name: str
    data: np.ndarray                 # (Nx, Ny) float64 image, or (N, s) series system
    window: tuple                    # (Lx, Ly)
    r: int                           # number of eigentriples requested
    block_k: int                     # Lanczos block width
    mask: np.ndarray | None = None   # (Nx, Ny) bool, True = inside N
    wmask: np.ndarray | None = None  # (Lx, Ly) bool window shape, None = full rectangle
    dtype: str = "f32"               # arithmetic type of the path ("f32" or "f64")
    groups: list = field(default_factory=list)  # 0-based eigentriple index groups
    terms: dict | None = None        # separable-term parameters (closed-form pins)
    noise_sigma: float = 0.0
    seed: int = 0


def draw_terms(rng: np.random.Generator, n_terms: int) -> dict:
    """Per-term parameters of the separable generator (BASELINE.json configs 3-5)."""
    a = rng.uniform(0.5, 3.0, n_terms)
    alpha = rng.uniform(-2e-3, 2e-3, n_terms)
    beta = rng.uniform(-2e-3, 2e-3, n_terms)
    omega = rng.uniform(0.01, 0.25, n_terms)
    nu = rng.uniform(0.01, 0.25, n_terms)
    phi = rng.uniform(0.0, TWO_PI, n_terms)
    psi = rng.uniform(0.0, TWO_PI, n_terms)
    return dict(a=a, alpha=alpha, beta=beta, omega=omega, nu=nu, phi=phi, psi=psi)


def separable_image(nx: int, ny: int, t: dict) -> np.ndarray:
    """x[i,j] = sum_k a_k e^{alpha_k i + beta_k j} cos(2 pi omega_k i + phi_k) cos(2 pi nu_k j + psi_k)."""
    i = np.arange(nx, dtype=np.float64)[:, None]
    j = np.arange(ny, dtype=np.float64)[None, :]
    img = np.zeros((nx, ny), dtype=np.float64)
    for k in range(len(t["a"])):
        fx = np.exp(t["alpha"][k] * i) * np.cos(TWO_PI * t["omega"][k] * i + t["phi"][k])
        fy = np.exp(t["beta"][k] * j) * np.cos(TWO_PI * t["nu"][k] * j + t["psi"][k])
        img += t["a"][k] * fx * fy
    return img


def config1(seed: int = 1, noise: bool = True) -> Workload:
    """c1: 64x64 fp64, 3cos(2pi .05 i)cos(2pi .08 j) + 2(.99^i)cos(2pi .2 j + .3) + N(0, .5^2)."""
    rng = np.random.default_rng(seed)
    nx = ny = 64
    i = np.arange(nx, dtype=np.float64)[:, None]
    j = np.arange(ny, dtype=np.float64)[None, :]
    img = 3.0 * np.cos(TWO_PI * 0.05 * i) * np.cos(TWO_PI * 0.08 * j) \
        + 2.0 * (0.99 ** i) * np.cos(TWO_PI * 0.2 * j + 0.3)
    # the same two terms written in separable-parameter form (for the closed-form pins)
    terms = dict(a=np.array([3.0, 2.0]), alpha=np.array([0.0, np.log(0.99)]),
                 beta=np.array([0.0, 0.0]), omega=np.array([0.05, 0.0]),
                 nu=np.array([0.08, 0.2]), phi=np.array([0.0, 0.0]),
                 psi=np.array([0.0, 0.3]))
    sig = 0.5 if noise else 0.0
    if noise:
        img = img + rng.normal(0.0, 0.5, size=(nx, ny))
    return Workload("c1", img, (16, 16), r=10, block_k=16, dtype="f64",
                    groups=[[0, 1, 2, 3], [4, 5]], terms=terms, noise_sigma=sig, seed=seed)


def config2(seed: int = 2, noise: bool = True, n: int = 4096, s: int = 8, L: int = 1024) -> Workload:
    """c2: MSSA, s=8 series of length 4096; window L=1024 (2D packing (L,1))."""
    rng = np.random.default_rng(seed)
    t = np.arange(n, dtype=np.float64)[:, None]
    c = np.arange(s, dtype=np.float64)[None, :]
    x = (1.0 + 0.1 * c) * np.sin(TWO_PI * t / 37.0 + c * 0.4) \
        + 0.5 * np.sin(TWO_PI * t / 11.0) + 0.001 * t * c
    if noise:
        x = x + rng.normal(0.0, 0.3, size=(n, s))
    # block width 16: faster to solution than SURVEY's proposed 32 (decompose 7.3 vs 8.5 ms on B200,
    # scripts/sweep_k.py); BASELINE fixes k only for c3 and c5
    return Workload("c2", x, (L, 1), r=16, block_k=16, dtype="f32",
                    groups=[[0], [1, 2], [3], [4, 5], [0, 1, 2, 3, 4, 5]],
                    noise_sigma=0.3 if noise else 0.0, seed=seed)


def _separable_config(name, seed, n, n_terms, window, r, k, noise, groups):
    rng = np.random.default_rng(seed)
    terms = draw_terms(rng, n_terms)
    img = separable_image(n, n, terms)
    if noise:
        img = img + rng.normal(0.0, 1.0, size=(n, n))
    return Workload(name, img, window, r=r, block_k=k, dtype="f32", groups=groups,
                    terms=terms, noise_sigma=1.0 if noise else 0.0, seed=seed), rng


def config3(seed: int = 3, noise: bool = True) -> Workload:
    """c3: 512x512 fp32, 6 separable terms + N(0,1); window 64x64; r=32, k=32."""
    groups = [list(range(4 * g, 4 * g + 4)) for g in range(6)] + [list(range(24))]
    w, _ = _separable_config("c3", seed, 512, 6, (64, 64), 32, 32, noise, groups)
    return w


def disc_with_holes(rng: np.random.Generator, n: int = 1024, radius: float = 500.0,
                    n_holes: int = 40, hmin: int = 8, hmax: int = 48) -> np.ndarray:
    """Centred disc (i-c)^2+(j-c)^2 <= R^2, c=(n-1)/2, minus seeded rectangular holes."""
    c = (n - 1) / 2.0
    i = np.arange(n, dtype=np.float64)[:, None]
    j = np.arange(n, dtype=np.float64)[None, :]
    mask = (i - c) ** 2 + (j - c) ** 2 <= radius * radius
    for _ in range(n_holes):
        h = int(rng.integers(hmin, hmax + 1))
        w = int(rng.integers(hmin, hmax + 1))
        i0 = int(rng.integers(0, n - h + 1))
        j0 = int(rng.integers(0, n - w + 1))
        mask[i0:i0 + h, j0:j0 + w] = False
    return mask


def config4(seed: int = 4, noise: bool = True) -> Workload:
    """c4: Shaped 2D-SSA, 1024x1024, 8 terms, disc r=500 with 40 holes; window 48x48; r=20."""
    groups = [list(range(4 * g, 4 * g + 4)) for g in range(5)]
    w, rng = _separable_config("c4", seed, 1024, 8, (48, 48), 20, 32, noise, groups)
    w.mask = disc_with_holes(rng)
    return w


def config5(seed: int = 5, noise: bool = True) -> Workload:
    """c5: 4096x4096 fp32, 12 terms + N(0,1), window 256x256; r=50, k=64."""
    groups = [list(range(48))]
    w, _ = _separable_config("c5", seed, 4096, 12, (256, 256), 50, 64, noise, groups)
    return w


def small_shaped(seed: int = 11, nx: int = 40, ny: int = 33, window=(7, 5),
                 n_holes: int = 4, noise: bool = True, wmask_drop: int = 0) -> Workload:
    """A small, non-square shaped case (ragged sizes, holes, optional non-rectangular window)
    for parity tests that must catch x/y transposition bugs (SURVEY §4 'transposition trap')."""
    rng = np.random.default_rng(seed)
    terms = draw_terms(rng, 3)
    img = separable_image(nx, ny, terms)
    if noise:
        img = img + rng.normal(0.0, 0.3, size=(nx, ny))
    mask = np.ones((nx, ny), dtype=bool)
    for _ in range(n_holes):
        h = int(rng.integers(2, 6)); w = int(rng.integers(2, 6))
        i0 = int(rng.integers(0, nx - h + 1)); j0 = int(rng.integers(0, ny - w + 1))
        mask[i0:i0 + h, j0:j0 + w] = False
    wmask = None
    if wmask_drop:
        wmask = np.ones(window, dtype=bool)
        cells = rng.choice(window[0] * window[1], size=wmask_drop, replace=False)
        for c in cells:
            wmask[c % window[0], c // window[0]] = False
        wmask[0, 0] = True  # keep the bounding box anchored
    return Workload("shaped_small", img, window, r=6, block_k=8, dtype="f32",
                    mask=mask, wmask=wmask, terms=terms, noise_sigma=0.3 if noise else 0, seed=seed)


CONFIGS = {"c1": config1, "c2": config2, "c3": config3, "c4": config4, "c5": config5}


def get(name: str, **kw) -> Workload:
    return CONFIGS[name](**kw)
