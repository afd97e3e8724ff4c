// The small-L "eigen" decomposition (svd.method = "eigen"):
// S = X Xᵀ formed with the fast trajectory products — Xᵀ·I_L block by block, then X·(XᵀI_L), "O(LN log N)
// flops using the fast matrix-vector multiplication" — then the full symmetric eigendecomposition of the
// L x L matrix S (the solver's device one-sided Jacobi, fp64: for SPD S the singular values are the
// eigenvalues and the left singular vectors the eigenvectors), σ_i = √λ_i, U_i = eigenvectors; V_i = XᵀU_i/σ_i
// on request as for the Lanczos path.  Squaring the operator squares its condition number
// (SURVEY finding 6): in fp32 plans σ_i below ~1e-3·σ_1 lose accuracy; the Lanczos path remains the default.
#include <algorithm>
#include <cmath>
#include <numeric>
#include <vector>

#include "common.h"
#include "kernels.h"
#include "plan.h"

namespace ssa {

void jacobi_svd_blocked(int m, int n, double *T, int *counters, int *sweeps, cudaStream_t st, double tol, double early);
bool jacobi_blocked_fits(int m, int n);

template <typename T>
__global__ void identity_block_kernel(T *I, int64_t ld, int c0, int kc) {
    const int64_t n = ld * kc;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = t % ld, c = t / ld;
        I[t] = (i == c0 + c) ? T(1) : T(0);
    }
}

// Sd = (S + Sᵀ)/2 in fp64 (the two products leave S symmetric only to rounding)
template <typename T>
__global__ void symmetrize_kernel(const T *S, int L, double *Sd) {
    const int64_t n = (int64_t)L * L;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
        const int i = (int)(t % L), j = (int)(t / L);
        Sd[t] = 0.5 * ((double)S[i + (int64_t)L * j] + (double)S[j + (int64_t)L * i]);
    }
}

template <typename T>
__global__ void take_columns_kernel(const double *A, int L, const int *cols, const double *inv, int r, T *U) {
    const int64_t n = (int64_t)L * r;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
        const int i = (int)(t % L), c = (int)(t / L);
        U[t] = (T)(A[i + (int64_t)L * cols[c]] * inv[c]);
    }
}

template <typename T>
void decompose_eigen(PlanImpl &p, int r, ssa_decomp_info *info) {
    const int L = (int)p.L;
    const int64_t K = p.K;
    SSA_REQUIRE(jacobi_blocked_fits(L, L), SSA_ERR_ARG, "eigen decomposition: L <= 768 (device eigensolver)");
    SSA_REQUIRE(!(p.has_comm && p.comm.world > 1), SSA_ERR_ARG, "eigen decomposition: not on band plans");
    cudaStream_t st = p.st;
    const int kb = 64;
    DevBuf I, VI, S, Sd, ints;
    I.alloc(sizeof(T) * (size_t)L * kb, st);
    VI.alloc(sizeof(T) * (size_t)K * kb, st);
    S.alloc(sizeof(T) * (size_t)L * L, st);
    int64_t nvec = 0, nblk = 0;
    cudaEvent_t e0, e1;
    SSA_CUDA(cudaEventCreate(&e0)); SSA_CUDA(cudaEventCreate(&e1));
    SSA_CUDA(cudaEventRecord(e0, st));
    for (int c0 = 0; c0 < L; c0 += kb) {        // S[:, c0:c0+kc] = X · (Xᵀ · I[:, c0:c0+kc])
        const int kc = std::min(kb, L - c0);
        identity_block_kernel<T><<<(unsigned)std::min<int64_t>(cdiv((int64_t)L * kc, 256), 8 * num_sms()), 256, 0, st>>>(
            I.as<T>(), L, c0, kc);
        after_launch("identity_block");
        op_xtu<T>(p, I.as<T>(), L, VI.as<T>(), K, kc);
        op_xv<T>(p, VI.as<T>(), K, S.as<T>() + (size_t)L * c0, L, kc);
        nvec += 2 * kc; nblk += 2;
    }
    SSA_CUDA(cudaEventRecord(e1, st));
    Sd.alloc(sizeof(double) * (size_t)L * L, st);
    symmetrize_kernel<T><<<(unsigned)std::min<int64_t>(cdiv((int64_t)L * L, 256), 8 * num_sms()), 256, 0, st>>>(
        S.as<T>(), L, Sd.as<double>());
    after_launch("symmetrize");
    ints.alloc(sizeof(int) * 128, st);
    jacobi_svd_blocked(L, L, Sd.as<double>(), ints.as<int>(), ints.as<int>() + 64, st, 1e-12, 1e-8);
    // λ_j = ||column j of S·J||, eigenvector = column / λ_j; order by λ descending
    std::vector<double> A((size_t)L * L);
    SSA_CUDA(cudaMemcpyAsync(A.data(), Sd.p, sizeof(double) * A.size(), cudaMemcpyDeviceToHost, st));
    SSA_CUDA(cudaStreamSynchronize(st));
    std::vector<double> lam(L);
    for (int j = 0; j < L; ++j) {
        double s = 0.0;
        for (int i = 0; i < L; ++i) s += A[i + (size_t)L * j] * A[i + (size_t)L * j];
        lam[j] = std::sqrt(s);
    }
    std::vector<int> ord(L);
    std::iota(ord.begin(), ord.end(), 0);
    std::stable_sort(ord.begin(), ord.end(), [&](int a, int b) { return lam[a] > lam[b]; });
    std::vector<int> cols(ord.begin(), ord.begin() + r);
    std::vector<double> inv(r);
    p.sigma.assign(r, 0.0);
    for (int i = 0; i < r; ++i) {
        p.sigma[i] = std::sqrt(std::max(lam[cols[i]], 0.0));
        inv[i] = lam[cols[i]] > 0 ? 1.0 / lam[cols[i]] : 0.0;
    }
    DevBuf dc, di;
    dc.alloc(sizeof(int) * r, st); di.alloc(sizeof(double) * r, st);
    SSA_CUDA(cudaMemcpyAsync(dc.p, cols.data(), sizeof(int) * r, cudaMemcpyHostToDevice, st));
    SSA_CUDA(cudaMemcpyAsync(di.p, inv.data(), sizeof(double) * r, cudaMemcpyHostToDevice, st));
    p.U.alloc(sizeof(T) * (size_t)L * r, st);
    take_columns_kernel<T><<<(unsigned)std::min<int64_t>(cdiv((int64_t)L * r, 256), 8 * num_sms()), 256, 0, st>>>(
        Sd.as<double>(), L, dc.as<int>(), di.as<double>(), r, p.U.as<T>());
    after_launch("take_columns");
    // sign convention (largest-|.| entry of U_i positive)
    DevBuf sg;
    sg.alloc(sizeof(double) * r, st);
    absmax_sign<T>(L, p.U.as<T>(), L, r, sg.as<double>(), st);
    scale_columns<T>(L, p.U.as<T>(), L, r, sg.as<double>(), st);
    p.r = r;
    p.v_valid = false;
    p.v_have.clear();
    // residual ||X v_i − σ_i u_i|| with v_i = Xᵀu_i/σ_i  (= ||S u_i − λ_i u_i|| / σ_i)
    DevBuf Vr, XV;
    Vr.alloc(sizeof(T) * (size_t)K * r, st);
    XV.alloc(sizeof(T) * (size_t)L * r, st);
    op_xtu<T>(p, p.U.as<T>(), L, Vr.as<T>(), K, r);
    op_xv<T>(p, Vr.as<T>(), K, XV.as<T>(), L, r);
    nvec += 2 * r; nblk += 2;
    std::vector<T> hu((size_t)L * r), hx((size_t)L * r);
    SSA_CUDA(cudaMemcpyAsync(hu.data(), p.U.p, sizeof(T) * hu.size(), cudaMemcpyDeviceToHost, st));
    SSA_CUDA(cudaMemcpyAsync(hx.data(), XV.p, sizeof(T) * hx.size(), cudaMemcpyDeviceToHost, st));
    SSA_CUDA(cudaStreamSynchronize(st));
    p.residuals.assign(r, 0.0);
    double maxres = 0.0;
    for (int i = 0; i < r; ++i) {
        const double s = p.sigma[i];
        double e2 = 0.0;
        for (int l = 0; l < L; ++l) {
            const double d = (s > 0 ? (double)hx[l + (size_t)L * i] / s : 0.0) - s * (double)hu[l + (size_t)L * i];
            e2 += d * d;
        }
        p.residuals[i] = std::sqrt(e2);
        maxres = std::max(maxres, p.residuals[i] / std::max(p.sigma[0], 1e-300));
    }
    float ms = 0.f;
    SSA_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    cudaEventDestroy(e0); cudaEventDestroy(e1);
    if (info) {
        info->r_requested = r;
        info->n_converged = r;
        info->block_k = kb;
        info->n_block_products = nblk;
        info->n_vector_products = nvec;
        info->max_rel_residual = maxres;
        info->ms_products = ms;
        info->sigma_floor_rel = sigma_floor(p);
        info->n_below_floor = 0;
        for (int i = 0; i < r; ++i) info->n_below_floor += p.sigma[i] < info->sigma_floor_rel * p.sigma[0] ? 1 : 0;
    }
}
template void decompose_eigen<float>(PlanImpl &, int, ssa_decomp_info *);
template void decompose_eigen<double>(PlanImpl &, int, ssa_decomp_info *);

}  // namespace ssa
