// Parameter estimation and forecasting on the decomposition:
//
//  * LS-ESPRIT / 2D-ESPRIT: shift matrices Φ_x, Φ_y between the
//    eigenarrays of a group restricted to 𝔏 and to 𝔏 shifted by one cell along x (y), as the
//    least-squares solutions of U↑ Φ ≈ U↓, and their joint diagonalisation (the eigenvectors T of a
//    generic combination Φ_x + c·Φ_y; λ_k = (T⁻¹Φ_xT)_kk, μ_k = (T⁻¹Φ_yT)_kk).  The tall-skinny
//    Grams U↑ᵀU↑, U↑ᵀU↓ (L rows) run on the device (gather of the shifted rows, then the solver's
//    Gram kernel); the r x r algebra (Cholesky solve, complex Hessenberg-QR eigenvalues, inverse
//    iteration) is host code like the solver's small dense steps.
//  * Alg. 7, fast column vector forecast (Remark 1: D is the LS-ESPRIT shift matrix):
//    per series p of a 1-D / MSSA plan, W_k = (σ_i V_i[κ_k])_i for its K_p window positions,
//    W_k = D W_{k−1} for k = K_p+1 .. K_p+M+L−1, and the rank-r matrix P·[W_1 : ... ] is
//    hankelized (diagonal averaging) on the device: z_1 .. z_{N_p+M}.
#include <algorithm>
#include <cmath>
#include <complex>
#include <cstring>
#include <vector>

#include "common.h"
#include "hostla.h"
#include "kernels.h"
#include "plan.h"

namespace ssa {

using cd = std::complex<double>;

// ---------------------------------------------------------------- small dense algebra (host)
// Φ = G⁻¹ C with G = AᵀA (SPD, r x r) and C = AᵀB: the normal equations of min ||A Φ − B||_F
static std::vector<double> ls_solve(int r, const std::vector<double> &G, const std::vector<double> &C) {
    std::vector<double> R((size_t)r * r);
    if (!hostla::cholesky_upper(r, G.data(), 0.0, 1e-300, R.data()))
        throw Error(SSA_ERR_ARG, "ESPRIT: the shifted eigenvectors are rank deficient");
    std::vector<double> X = C;
    for (int c = 0; c < r; ++c) {
        double *x = X.data() + (size_t)r * c;
        for (int i = 0; i < r; ++i) {            // Rᵀ y = c
            double v = x[i];
            for (int t = 0; t < i; ++t) v -= R[t + (size_t)r * i] * x[t];
            x[i] = v / R[i + (size_t)r * i];
        }
        for (int i = r - 1; i >= 0; --i) {       // R x = y
            double v = x[i];
            for (int t = i + 1; t < r; ++t) v -= R[i + (size_t)r * t] * x[t];
            x[i] = v / R[i + (size_t)r * i];
        }
    }
    return X;
}

// eigenvalues of a complex n x n matrix (column-major): Householder reduction to Hessenberg form,
// then the shifted QR algorithm (Wilkinson shifts, Givens rotations, deflation)
static std::vector<cd> eigvals(int n, std::vector<cd> A) {
    auto at = [&](int i, int j) -> cd & { return A[i + (size_t)n * j]; };
    for (int k = 0; k + 2 < n; ++k) {
        double nrm = 0.0;
        for (int i = k + 1; i < n; ++i) nrm += std::norm(at(i, k));
        nrm = std::sqrt(nrm);
        if (nrm == 0.0) continue;
        std::vector<cd> v(n, 0.0);
        const cd x0 = at(k + 1, k);
        const cd alpha = -std::polar(nrm, std::arg(x0));
        v[k + 1] = x0 - alpha;
        for (int i = k + 2; i < n; ++i) v[i] = at(i, k);
        double vn = 0.0;
        for (int i = k + 1; i < n; ++i) vn += std::norm(v[i]);
        if (vn == 0.0) continue;
        for (int j = 0; j < n; ++j) {            // A ← (I − 2vvᴴ/vᴴv) A
            cd s = 0.0;
            for (int i = k + 1; i < n; ++i) s += std::conj(v[i]) * at(i, j);
            s *= 2.0 / vn;
            for (int i = k + 1; i < n; ++i) at(i, j) -= v[i] * s;
        }
        for (int i = 0; i < n; ++i) {            // A ← A (I − 2vvᴴ/vᴴv)
            cd s = 0.0;
            for (int j = k + 1; j < n; ++j) s += at(i, j) * v[j];
            s *= 2.0 / vn;
            for (int j = k + 1; j < n; ++j) at(i, j) -= s * std::conj(v[j]);
        }
    }
    std::vector<cd> ev(n);
    int hi = n - 1, iter = 0;
    while (hi >= 0) {
        if (hi == 0) { ev[0] = at(0, 0); break; }
        int lo = hi;
        while (lo > 0) {
            const double sc = std::abs(at(lo, lo)) + std::abs(at(lo - 1, lo - 1));
            if (std::abs(at(lo, lo - 1)) <= 1e-15 * (sc > 0 ? sc : 1.0)) { at(lo, lo - 1) = 0.0; break; }
            --lo;
        }
        if (lo == hi) { ev[hi] = at(hi, hi); --hi; iter = 0; continue; }
        if (++iter > 200 * n) throw Error(SSA_ERR_NOT_CONVERGED, "ESPRIT: eigenvalue iteration did not converge");
        // Wilkinson shift from the trailing 2 x 2 block
        const cd a = at(hi - 1, hi - 1), b = at(hi - 1, hi), c = at(hi, hi - 1), d = at(hi, hi);
        const cd tr = a + d, det = a * d - b * c;
        const cd disc = std::sqrt(tr * tr - 4.0 * det);
        cd m1 = (tr + disc) * 0.5, m2 = (tr - disc) * 0.5;
        cd mu = std::abs(m1 - d) < std::abs(m2 - d) ? m1 : m2;
        if (iter % 11 == 10) mu += std::abs(at(hi, hi - 1));   // exceptional shift
        for (int i = lo; i <= hi; ++i) at(i, i) -= mu;
        std::vector<cd> cs(hi - lo), sn(hi - lo);
        for (int k = lo; k < hi; ++k) {          // QR of the active window by Givens rotations
            const cd x = at(k, k), y = at(k + 1, k);
            const double r = std::sqrt(std::norm(x) + std::norm(y));
            const cd c0 = r > 0 ? x / r : 1.0, s0 = r > 0 ? y / r : 0.0;
            cs[k - lo] = c0; sn[k - lo] = s0;
            for (int j = k; j < n; ++j) {
                const cd u = at(k, j), w = at(k + 1, j);
                at(k, j) = std::conj(c0) * u + std::conj(s0) * w;
                at(k + 1, j) = -s0 * u + c0 * w;
            }
        }
        for (int k = lo; k < hi; ++k) {          // RQ
            const cd c0 = cs[k - lo], s0 = sn[k - lo];
            for (int i = 0; i <= std::min(k + 2, hi); ++i) {
                const cd u = at(i, k), w = at(i, k + 1);
                at(i, k) = u * c0 + w * s0;
                at(i, k + 1) = -u * std::conj(s0) + w * std::conj(c0);
            }
        }
        for (int i = lo; i <= hi; ++i) at(i, i) += mu;
    }
    return ev;
}

// complex LU with partial pivoting (in place), solve
struct LU {
    int n;
    std::vector<cd> a;
    std::vector<int> piv;
    LU(int n_, const std::vector<cd> &A) : n(n_), a(A), piv(n_) {
        for (int k = 0; k < n; ++k) {
            int p = k;
            for (int i = k + 1; i < n; ++i)
                if (std::abs(a[i + (size_t)n * k]) > std::abs(a[p + (size_t)n * k])) p = i;
            piv[k] = p;
            if (p != k)
                for (int j = 0; j < n; ++j) std::swap(a[k + (size_t)n * j], a[p + (size_t)n * j]);
            cd d = a[k + (size_t)n * k];
            if (std::abs(d) == 0.0) d = a[k + (size_t)n * k] = 1e-300;
            for (int i = k + 1; i < n; ++i) {
                const cd f = a[i + (size_t)n * k] /= d;
                for (int j = k + 1; j < n; ++j) a[i + (size_t)n * j] -= f * a[k + (size_t)n * j];
            }
        }
    }
    void solve(cd *x) const {
        for (int k = 0; k < n; ++k) std::swap(x[k], x[piv[k]]);
        for (int i = 0; i < n; ++i)
            for (int t = 0; t < i; ++t) x[i] -= a[i + (size_t)n * t] * x[t];
        for (int i = n - 1; i >= 0; --i) {
            for (int t = i + 1; t < n; ++t) x[i] -= a[i + (size_t)n * t] * x[t];
            x[i] /= a[i + (size_t)n * i];
        }
    }
};

// eigenvectors by inverse iteration on the eigenvalues of eigvals()
static std::vector<cd> eigvecs(int n, const std::vector<cd> &A, const std::vector<cd> &ev) {
    std::vector<cd> T((size_t)n * n);
    double anorm = 0.0;
    for (const cd &v : A) anorm = std::max(anorm, std::abs(v));
    for (int k = 0; k < n; ++k) {
        std::vector<cd> B = A;
        const cd sh = ev[k] + cd(1e-10 * std::max(anorm, 1e-300), 1e-10 * std::max(anorm, 1e-300));
        for (int i = 0; i < n; ++i) B[i + (size_t)n * i] -= sh;
        LU lu(n, B);
        std::vector<cd> x(n);
        for (int i = 0; i < n; ++i) x[i] = cd(1.0 + 0.37 * i, 0.11 * (i % 5));
        for (int it = 0; it < 3; ++it) {
            lu.solve(x.data());
            double nr = 0.0;
            for (const cd &v : x) nr += std::norm(v);
            nr = std::sqrt(nr);
            for (cd &v : x) v /= nr;
        }
        for (int i = 0; i < n; ++i) T[i + (size_t)n * k] = x[i];
    }
    return T;
}

// ---------------------------------------------------------------- device helpers
template <typename T>
__global__ void gather_rows_kernel(const T *__restrict__ U, int64_t ldu, const int *__restrict__ rows, int nrows,
                                   const int *__restrict__ cols, int ncols, T *__restrict__ out) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < (int64_t)nrows * ncols;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int i = (int)(t % nrows), c = (int)(t / nrows);
        out[t] = U[rows[i] + ldu * cols[c]];
    }
}

// z[n] = Σ_{l + k = n} Σ_i P[l, i] Wf[k, i] / #{(l, k)}, n < nout; one warp per n (Alg. 7 step 3:
// the rank-r matrix P·Wfᵀ (L x K') hankelized)
template <typename T>
__global__ void hankel_rank_r_kernel(const T *__restrict__ P, int L, const double *__restrict__ Wf, int Kp, int r,
                                     int nout, T *__restrict__ z) {
    const int lane = threadIdx.x & 31;
    const int n = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (n >= nout) return;
    const int l0 = max(0, n - Kp + 1), l1 = min(L - 1, n);
    double acc = 0.0;
    for (int l = l0 + lane; l <= l1; l += 32) {
        const int k = n - l;
        for (int i = 0; i < r; ++i) acc += (double)P[l + (int64_t)L * i] * Wf[k + (int64_t)Kp * i];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) z[n] = (T)(acc / (double)(l1 - l0 + 1));
}

// Wf[k, i] = σ_{idx[i]} · V[koff + k, idx[i]] for k < K (the reconstructed part of W), fp64
template <typename T>
__global__ void scaled_rows_kernel(const T *__restrict__ V, int64_t ldv, const int *__restrict__ idx, const double *sig,
                                   int r, int64_t koff, int K, double *Wf, int ldw) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < (int64_t)K * r;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int k = (int)(t % K), i = (int)(t / K);
        Wf[k + (int64_t)ldw * i] = sig[idx[i]] * (double)V[koff + k + ldv * idx[i]];
    }
}

template <typename T> void get_v_cols(PlanImpl &p, const std::vector<int> &need);   // api.cu

// G (r x r) = Aᵀ B over the `rows` pairs of the group's eigenvectors (device gather + Gram)
template <typename T>
static void shifted_grams(PlanImpl &p, const std::vector<int> &idx, const std::vector<int> &ra, const std::vector<int> &rb,
                          std::vector<double> &G, std::vector<double> &C) {
    const int r = (int)idx.size(), nr = (int)ra.size();
    SSA_REQUIRE(nr >= r, SSA_ERR_ARG, "ESPRIT: fewer shifted rows than components");
    DevBuf d_idx, d_ra, d_rb, ua, ub, g;
    d_idx.alloc(sizeof(int) * r, p.st); d_ra.alloc(sizeof(int) * nr, p.st); d_rb.alloc(sizeof(int) * nr, p.st);
    SSA_CUDA(cudaMemcpyAsync(d_idx.p, idx.data(), sizeof(int) * r, cudaMemcpyHostToDevice, p.st));
    SSA_CUDA(cudaMemcpyAsync(d_ra.p, ra.data(), sizeof(int) * nr, cudaMemcpyHostToDevice, p.st));
    SSA_CUDA(cudaMemcpyAsync(d_rb.p, rb.data(), sizeof(int) * nr, cudaMemcpyHostToDevice, p.st));
    ua.alloc(sizeof(T) * (size_t)nr * r, p.st);
    ub.alloc(sizeof(T) * (size_t)nr * r, p.st);
    const unsigned grid = (unsigned)std::min<int64_t>(cdiv((int64_t)nr * r, 256), 8 * num_sms());
    gather_rows_kernel<T><<<grid, 256, 0, p.st>>>(p.U.as<T>(), p.L, d_ra.as<int>(), nr, d_idx.as<int>(), r, ua.as<T>());
    after_launch("gather_rows");
    gather_rows_kernel<T><<<grid, 256, 0, p.st>>>(p.U.as<T>(), p.L, d_rb.as<int>(), nr, d_idx.as<int>(), r, ub.as<T>());
    after_launch("gather_rows");
    g.alloc(sizeof(double) * 2 * 64 * 64, p.st);
    G.assign((size_t)r * r, 0.0);
    C.assign((size_t)r * r, 0.0);
    gram_tn<T>(nr, ua.as<T>(), nr, r, ua.as<T>(), nr, r, g.as<double>(), p.ws_gram.as<double>(), p.ws_gram.bytes, p.st);
    gram_tn<T>(nr, ua.as<T>(), nr, r, ub.as<T>(), nr, r, g.as<double>() + 64 * 64, p.ws_gram.as<double>(),
               p.ws_gram.bytes, p.st);
    SSA_CUDA(cudaMemcpyAsync(G.data(), g.p, sizeof(double) * r * r, cudaMemcpyDeviceToHost, p.st));
    SSA_CUDA(cudaMemcpyAsync(C.data(), g.as<double>() + 64 * 64, sizeof(double) * r * r, cudaMemcpyDeviceToHost, p.st));
    SSA_CUDA(cudaStreamSynchronize(p.st));
}

// row pairs (a, b) of the 𝔏-lex basis with b = a shifted by one cell along axis (both in 𝔏)
static void shift_pairs(const PlanImpl &p, int axis, std::vector<int> &ra, std::vector<int> &rb) {
    ra.clear(); rb.clear();
    for (int y = 0; y < p.ly; ++y)
        for (int x = 0; x < p.lx; ++x) {
            const int x2 = axis == 0 ? x + 1 : x, y2 = axis == 0 ? y : y + 1;
            if (x2 >= p.lx || y2 >= p.ly) continue;
            const int a = p.lmap_host[(size_t)x + (size_t)p.lx * y], b = p.lmap_host[(size_t)x2 + (size_t)p.lx * y2];
            if (a >= 0 && b >= 0) { ra.push_back(a); rb.push_back(b); }
        }
}

template <typename T>
static std::vector<double> shift_matrix(PlanImpl &p, const std::vector<int> &idx, int axis) {
    std::vector<int> ra, rb;
    shift_pairs(p, axis, ra, rb);
    std::vector<double> G, C;
    shifted_grams<T>(p, idx, ra, rb, G, C);
    return ls_solve((int)idx.size(), G, C);
}

template <typename T>
static void esprit_impl(PlanImpl &p, const std::vector<int> &idx, double *lam, double *mu) {
    const int r = (int)idx.size();
    const std::vector<double> phx = shift_matrix<T>(p, idx, 0);
    std::vector<cd> ax(phx.begin(), phx.end());
    if (p.ly == 1 || !mu) {
        const std::vector<cd> ev = eigvals(r, ax);
        for (int k = 0; k < r; ++k) { lam[2 * k] = ev[k].real(); lam[2 * k + 1] = ev[k].imag(); }
        if (mu)
            for (int k = 0; k < r; ++k) { mu[2 * k] = 1.0; mu[2 * k + 1] = 0.0; }
        return;
    }
    const std::vector<double> phy = shift_matrix<T>(p, idx, 1);
    std::vector<cd> ay(phy.begin(), phy.end()), comb((size_t)r * r);
    const cd c(0.6180339887, 0.3090169944);   // a generic combination: distinct eigenvalues
    for (size_t t = 0; t < comb.size(); ++t) comb[t] = ax[t] + c * ay[t];
    const std::vector<cd> ev = eigvals(r, comb);
    const std::vector<cd> Tm = eigvecs(r, comb, ev);
    LU lu(r, Tm);
    // λ_k = (T⁻¹ Φ_x T)_kk, μ_k = (T⁻¹ Φ_y T)_kk
    for (int k = 0; k < r; ++k) {
        std::vector<cd> vx(r, 0.0), vy(r, 0.0);
        for (int i = 0; i < r; ++i)
            for (int j = 0; j < r; ++j) {
                vx[i] += ax[i + (size_t)r * j] * Tm[j + (size_t)r * k];
                vy[i] += ay[i + (size_t)r * j] * Tm[j + (size_t)r * k];
            }
        lu.solve(vx.data());
        lu.solve(vy.data());
        lam[2 * k] = vx[k].real(); lam[2 * k + 1] = vx[k].imag();
        mu[2 * k] = vy[k].real(); mu[2 * k + 1] = vy[k].imag();
    }
}

template <typename T>
static void forecast_impl(PlanImpl &p, const std::vector<int> &idx, int M, T *out, int64_t nrow) {
    const int r = (int)idx.size(), L = (int)p.L;
    get_v_cols<T>(p, idx);
    const std::vector<double> D = shift_matrix<T>(p, idx, 0);   // Alg. 7 step 1 (LS-ESPRIT shift matrix)
    // per-series window positions: contiguous prefixes of the origin-box columns
    std::vector<uint8_t> km((size_t)p.kx * p.ky);
    SSA_CUDA(cudaMemcpyAsync(km.data(), p.kmask.p, km.size(), cudaMemcpyDeviceToHost, p.st));
    DevBuf d_idx, d_sig, Wf, wlast;
    d_idx.alloc(sizeof(int) * r, p.st);
    d_sig.alloc(sizeof(double) * p.r, p.st);
    SSA_CUDA(cudaMemcpyAsync(d_idx.p, idx.data(), sizeof(int) * r, cudaMemcpyHostToDevice, p.st));
    SSA_CUDA(cudaMemcpyAsync(d_sig.p, p.sigma.data(), sizeof(double) * p.r, cudaMemcpyHostToDevice, p.st));
    SSA_CUDA(cudaStreamSynchronize(p.st));
    std::vector<T> nanrow(nrow, (T)NAN);
    int64_t koff = 0;
    for (int s = 0; s < p.ky; ++s) {
        int K = 0;
        while (K < p.kx && km[(size_t)K + (size_t)p.kx * s]) ++K;
        for (int t = K; t < p.kx; ++t)
            SSA_REQUIRE(!km[(size_t)t + (size_t)p.kx * s], SSA_ERR_ARG,
                        "forecast: every series' window positions must be a contiguous prefix (NaN-padding at the end)");
        T *col = out + nrow * s;
        SSA_CUDA(cudaMemcpyAsync(col, nanrow.data(), sizeof(T) * nrow, cudaMemcpyHostToDevice, p.st));
        if (K == 0) continue;
        const int Kp = K + M + L - 1;           // columns of Z = P·[W_1 : ... : W_{K+M+L−1}]
        Wf.alloc(sizeof(double) * (size_t)Kp * r, p.st);
        scaled_rows_kernel<T><<<(unsigned)std::min<int64_t>(cdiv((int64_t)K * r, 256), 8 * num_sms()), 256, 0, p.st>>>(
            p.V.as<T>(), p.K, d_idx.as<int>(), d_sig.as<double>(), r, koff, K, Wf.as<double>(), Kp);
        after_launch("scaled_rows");
        // Alg. 7 step 2: W_k = D W_{k−1} from W_K (host, r x r per step)
        std::vector<double> w(r), ext((size_t)(Kp - K) * r);
        for (int i = 0; i < r; ++i)
            SSA_CUDA(cudaMemcpyAsync(&w[i], Wf.as<double>() + (K - 1) + (size_t)Kp * i, sizeof(double),
                                     cudaMemcpyDeviceToHost, p.st));
        SSA_CUDA(cudaStreamSynchronize(p.st));
        for (int m = 0; m < Kp - K; ++m) {
            std::vector<double> nw(r, 0.0);
            for (int j = 0; j < r; ++j)
                for (int i = 0; i < r; ++i) nw[i] += D[i + (size_t)r * j] * w[j];
            w.swap(nw);
            for (int i = 0; i < r; ++i) ext[(size_t)m + (size_t)(Kp - K) * i] = w[i];
        }
        SSA_CUDA(cudaMemcpy2DAsync(Wf.as<double>() + K, sizeof(double) * Kp, ext.data(), sizeof(double) * (Kp - K),
                                   sizeof(double) * (Kp - K), r, cudaMemcpyHostToDevice, p.st));
        // Alg. 7 step 3: hankelization of P·Wfᵀ; z_1..z_{N_p+M}
        DevBuf Pg;
        Pg.alloc(sizeof(T) * (size_t)L * r, p.st);
        for (int i = 0; i < r; ++i)
            SSA_CUDA(cudaMemcpyAsync(Pg.as<T>() + (size_t)L * i, p.U.as<T>() + (size_t)L * idx[i], sizeof(T) * L,
                                     cudaMemcpyDeviceToDevice, p.st));
        const int nout = K + L - 1 + M;
        hankel_rank_r_kernel<T><<<(unsigned)cdiv(nout, 8), 256, 0, p.st>>>(Pg.as<T>(), L, Wf.as<double>(), Kp, r, nout, col);
        after_launch("hankel_rank_r");
        SSA_CUDA(cudaStreamSynchronize(p.st));
        koff += K;
    }
}

}  // namespace ssa

using namespace ssa;

static std::vector<int> group_list(const PlanImpl &P, const int32_t *idx, int32_t n) {
    if (!idx || n < 1 || n > 64) throw Error(SSA_ERR_ARG, "1..64 eigentriple indices");
    if (P.r == 0) throw Error(SSA_ERR_STATE, "no decomposition");
    std::vector<int> v(idx, idx + n);
    for (int i : v)
        if (i < 0 || i >= P.r) throw Error(SSA_ERR_RANK, "eigentriple index >= computed rank");
    return v;
}

extern "C" {

ssa_status ssa_esprit(ssa_plan p, const int32_t *idx, int32_t n, double *lambda, double *mu) {
    try {
        if (!p || !lambda) throw Error(SSA_ERR_ARG, "null argument");
        PlanImpl &P = ssa_plan_impl(p);
        const std::vector<int> g = group_list(P, idx, n);
        if (P.dt == SSA_F64) esprit_impl<double>(P, g, lambda, mu);
        else esprit_impl<float>(P, g, lambda, mu);
        return SSA_OK;
    } catch (const Error &e) {
        ssa_set_error(e.what());
        return e.code;
    } catch (const std::exception &e) {
        ssa_set_error(e.what());
        return SSA_ERR_ARG;
    }
}

ssa_status ssa_forecast(ssa_plan p, const int32_t *idx, int32_t n, int32_t M, void *out, int64_t ld_out, int on_device) {
    try {
        if (!p || !out || M < 0) throw Error(SSA_ERR_ARG, "bad forecast arguments");
        PlanImpl &P = ssa_plan_impl(p);
        const std::vector<int> g = group_list(P, idx, n);
        if (P.ly != 1 || !P.full_window) throw Error(SSA_ERR_ARG, "forecast: 1-D SSA / MSSA plans only (window (L, 1))");
        if (P.has_comm && P.comm.world > 1) throw Error(SSA_ERR_ARG, "forecast: not on band plans");
        const int64_t nrow = P.nx + M;      // max_p N_p + M
        if (ld_out == 0) ld_out = nrow;
        if (ld_out < nrow) throw Error(SSA_ERR_ARG, "forecast: ld_out < nx + M");
        const size_t es = P.elem();
        DevBuf tmp;
        void *dout = out;
        if (!on_device || ld_out != nrow) {
            tmp.alloc(es * nrow * P.ky, P.st);
            dout = tmp.p;
        }
        if (P.dt == SSA_F64) forecast_impl<double>(P, g, M, (double *)dout, nrow);
        else forecast_impl<float>(P, g, M, (float *)dout, nrow);
        if (dout != out)
            SSA_CUDA(cudaMemcpy2DAsync(out, es * ld_out, dout, es * nrow, es * nrow, P.ky,
                                       on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, P.st));
        SSA_CUDA(cudaStreamSynchronize(P.st));
        return SSA_OK;
    } catch (const Error &e) {
        ssa_set_error(e.what());
        return e.code;
    } catch (const std::exception &e) {
        ssa_set_error(e.what());
        return SSA_ERR_ARG;
    }
}

}  // extern "C"
