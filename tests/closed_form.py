"""Closed forms used as PINS for the oracle and the CUDA path.

Independent of oracle/: nothing here materialises the trajectory matrix or runs
the double-loop operator.  It uses the finite-rank parametric form of real arrays
(eq. P:4317-4320):

    x_{m,n} = Σ_q c_q λ_q^m μ_q^n   (0-based m, n)

for which 𝒯(𝕏) = A·diag(c)·Bᵀ with A[ℓ,q] = λ_q^{ℓx} μ_q^{ℓy},
B[κ,q] = λ_q^{κx} μ_q^{κy} (the shifted sum ℓ +‐ κ is plain addition 0-based).
Each real factor e^{αi}cos(2πωi+φ) = ½(e^{iφ}λ₊^i + e^{-iφ}λ₋^i), λ± = e^{α±2πiω}
gives 2 complex roots (1 when ω = 0); equal (λ, μ) pairs are merged.
"""
from __future__ import annotations

import numpy as np


def roots(terms: dict, tol: float = 1e-13):
    """(λ, μ, c) of x_{ij} = Σ_k a_k e^{α_k i+β_k j} cos(2πω_k i+φ_k) cos(2πν_k j+ψ_k)."""
    lam, mu, cc = [], [], []
    for k in range(len(terms["a"])):
        a, al, be = terms["a"][k], terms["alpha"][k], terms["beta"][k]
        om, nu, ph, ps = terms["omega"][k], terms["nu"][k], terms["phi"][k], terms["psi"][k]
        for s in (+1, -1):
            for t in (+1, -1):
                lam.append(np.exp(al + 2j * np.pi * s * om))
                mu.append(np.exp(be + 2j * np.pi * t * nu))
                cc.append(a / 4.0 * np.exp(1j * (s * ph + t * ps)))
    # merge identical (λ, μ) pairs (ω = 0 or ν = 0 factors)
    out = []
    for l, m, c in zip(lam, mu, cc):
        for e in out:
            if abs(e[0] - l) < tol and abs(e[1] - m) < tol:
                e[2] += c
                break
        else:
            out.append([l, m, c])
    out = [e for e in out if abs(e[2]) > 1e-14]
    L = np.array([e[0] for e in out]); M = np.array([e[1] for e in out]); Cc = np.array([e[2] for e in out])
    return L, M, Cc


def image(terms: dict, nx: int, ny: int) -> np.ndarray:
    """The noiseless image from its roots (a check that roots() is right)."""
    lam, mu, c = roots(terms)
    i = np.arange(nx)[:, None, None]; j = np.arange(ny)[None, :, None]
    return np.real(np.sum(c * lam ** i * mu ** j, axis=2))


def rank(terms: dict) -> int:
    """Closed-form trajectory rank (P6): number of distinct (λ, μ) pairs (for windows
    and origin sets large enough)."""
    return len(roots(terms)[0])


def _vander(lam, mu, px, py):
    return (lam[None, :] ** px[:, None]) * (mu[None, :] ** py[:, None])


def products(terms, lpos, kpos, V=None, U=None):
    """P5: X·V = A (c ⊙ (Bᵀ V)) and Xᵀ·U = B (c ⊙ (Aᵀ U)), O((L+K)R) per vector."""
    lam, mu, c = roots(terms)
    A = _vander(lam, mu, *lpos)
    B = _vander(lam, mu, *kpos)
    out = []
    if V is not None:
        out.append(np.real(A @ (c[:, None] * (B.T @ V))))
    if U is not None:
        out.append(np.real(B @ (c[:, None] * (A.T @ U))))
    return out[0] if len(out) == 1 else tuple(out)


def _geo_gram(z1, z2, n):
    """G[p,q] = Σ_{t=0}^{n-1} (conj(z1_p) z2_q)^t (geometric sums)."""
    q = np.conj(z1)[:, None] * z2[None, :]
    with np.errstate(divide="ignore", invalid="ignore"):
        g = (1 - q ** n) / (1 - q)
    near1 = np.abs(q - 1) < 1e-12
    g[near1] = n
    return g


def sigma_rect(terms, lx, ly, kx, ky):
    """P7 for rectangular 𝔏 and 𝔎: σ(X) = σ(R_A · diag(c) · L_B) with
    G_A = AᴴA = R_Aᴴ R_A and H_B = Bᵀ conj(B) = L_B L_Bᴴ.  Both Grams factor
    into products of 1-D geometric sums (Khatri-Rao structure), so this works at
    any size (including c5)."""
    lam, mu, c = roots(terms)
    GA = _geo_gram(lam, lam, lx) * _geo_gram(mu, mu, ly)
    HB = np.conj(_geo_gram(lam, lam, kx) * _geo_gram(mu, mu, ky))  # Σ_κ b_p conj(b_q)
    return _sigma_from_grams(GA, HB, c)


def sigma_shaped(terms, lpos, kpos, chunk=1 << 16):
    """P7 with irregular shapes: Grams summed explicitly over 𝔏 and 𝔎, O((L+K)R²)."""
    lam, mu, c = roots(terms)
    A = _vander(lam, mu, *lpos)
    GA = A.conj().T @ A
    R = len(lam)
    HB = np.zeros((R, R), dtype=complex)
    kx, ky = kpos
    for s in range(0, len(kx), chunk):
        B = _vander(lam, mu, kx[s:s + chunk], ky[s:s + chunk])
        HB += B.T @ B.conj()
    return _sigma_from_grams(GA, HB, c)


def _sigma_from_grams(GA, HB, c):
    RA = np.linalg.cholesky(GA).conj().T          # GA = RAᴴ RA
    LB = np.linalg.cholesky(HB)                    # HB = LB LBᴴ
    M = RA @ (c[:, None] * LB)
    return np.linalg.svd(M, compute_uv=False)
