"""Shared parity helpers for the GPU tests (tolerances of BASELINE.json's north star with
SURVEY §8(c) readings Q9-Q11)."""
import numpy as np

# Reading Q10: σ floor τ of the fp32 paths — the smallest σ_i/σ_1 down to which σ_i
# meets the σ bar (relative error <= 1e-4), MEASURED on the noiseless c5 twin (σ spread 1.2e-7)
# against the closed form (scripts/measure_tau.py -> profiles/r02/tau.json): FFT and tensor-core
# paths both hold it down to σ_28/σ_1 = 8.7e-5 (below it the r = 50 decomposition, converged at
# ||Xᵀu − σv|| <= 1e-6·σ_1, resolves σ only to ~1e-6·σ_1 absolute).  The library reports the same
# value (ssa_decomp_info.sigma_floor_rel).
TAU = {"fft": 8.7e-5, "direct": 8.7e-5, "tc": 8.7e-5, "f64": 1e-12}


def relfro(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return np.linalg.norm(a - b) / np.linalg.norm(b)


def relgaps(s_all, r):
    """relgap_i = min(σ_{i−1} − σ_i, σ_i − σ_{i+1}) / σ_i (σ_0 = ∞), reading Q10."""
    s = np.asarray(s_all, np.float64)
    g = np.full(r, np.inf)
    for i in range(r):
        left = s[i - 1] - s[i] if i > 0 else np.inf
        right = s[i] - s[i + 1] if i + 1 < len(s) else np.inf
        g[i] = min(left, right) / s[i] if s[i] > 0 else 0.0
    return g


def check_sigma(s_gpu, s_ref_all, r, tau, rel=1e-4, floor_abs=1e-6):
    """Reading Q10: |Δσ_i| <= rel·σ_i where relgap_i >= 1e-3 and σ_i >= τ·σ_1; elsewhere
    (clusters, below the floor) |Δσ_i| <= floor_abs·σ_1.  Returns the indices checked at `rel`."""
    s_gpu = np.asarray(s_gpu, np.float64)
    s_ref = np.asarray(s_ref_all[:r], np.float64)
    gaps = relgaps(s_ref_all, r)
    s1 = s_ref[0]
    checked = []
    for i in range(r):
        if gaps[i] >= 1e-3 and s_ref[i] >= tau * s1:
            assert abs(s_gpu[i] - s_ref[i]) <= rel * s_ref[i], (i, s_gpu[i], s_ref[i])
            checked.append(i)
        else:
            assert abs(s_gpu[i] - s_ref[i]) <= floor_abs * s1, (i, s_gpu[i], s_ref[i], abs(s_gpu[i] - s_ref[i]) / s1)
    return checked


def gap_groups(s_all, r, thr=1e-3):
    """Reading Q9: maximal clusters of the first r indices bounded by relative gaps >= thr
    (a cluster cut by r itself is dropped)."""
    s = np.asarray(s_all, np.float64)
    groups, cur = [], [0]
    for i in range(1, r + 1):
        if (s[i - 1] - s[i]) / s[i - 1] >= thr:
            groups.append(cur)
            cur = [i]
        elif i == r:
            break
        else:
            cur.append(i)
    return [g for g in groups if max(g) < r]


def projector_err(A, B):
    """Distance of the subspaces spanned by A and B (sign / rotation invariant, reading Q11):
    ||P_A − P_B||_F / ||P_B||_F = sqrt(2)·||(I − Q_B Q_Bᵀ) Q_A||_F / sqrt(k) for equal dimensions k,
    formed from the residual directly (no cancellation: accurate down to rounding)."""
    qa, _ = np.linalg.qr(np.asarray(A, np.float64))
    qb, _ = np.linalg.qr(np.asarray(B, np.float64))
    r = qa - qb @ (qb.T @ qa)
    return np.sqrt(2.0) * np.linalg.norm(r) / np.sqrt(qb.shape[1])
