// Projected-matrix SVD on the GPU ("mk x mk SVD (fp64)"):
// one-sided (Hestenes) Jacobi in fp64.
//   * the rotation angle t is computed in fp32 (cheap MUFU ops); c = 1/√(1+t²)
//     and s = c·t are then formed in fp64, so every applied rotation is exactly
//     orthogonal to working precision — an fp32-accurate angle only means a pair
//     may need another visit, which the sweep loop provides;
//   * σ_j = ||a_j||, left vectors y_j = a_j / σ_j; the right vectors are
//     recovered by the caller as z_j = Tᵀ y_j / σ_j (rotations not accumulated,
//     every access stays on-chip).  σ never comes from eigenvalues of TᵀT.
#include "common.h"
#include "kernels.h"

#include <cooperative_groups.h>

namespace ssa {

// ---------------------------------------------------------------------------
// Block one-sided Jacobi over a cooperative grid (the production path).
// Columns live in global memory (L2-resident); the n columns are split into nb
// blocks of kBW columns (nb even, zero padding).  Each outer round pairs the
// blocks by the circle method; CTA c loads its two blocks (2·kBW columns) into
// shared memory, runs one inner one-sided Jacobi sweep over all column pairs of
// those 2·kBW columns (one warp per pair per inner round), writes them back,
// and the grid synchronises.  A sweep is nb-1 outer rounds; sweeps repeat until
// no rotation happened anywhere.  Same fp32-angle / fp64-rotation scheme as
// above.
// ---------------------------------------------------------------------------
constexpr int kBW = 8;   // columns per block; a CTA holds 2*kBW columns and runs kBW warps

// Rotate columns (ap, aq) of length m so that they become orthogonal.  Each lane
// caches its MR-strided slice of both columns in registers: one load burst, the
// three dot products and the rotation all from registers, one store burst.
template <int MR>
__device__ __forceinline__ bool jacobi_pair(double *ap, double *aq, int m, int lane, float tol) {
    double x[MR], y[MR];
#pragma unroll
    for (int u = 0; u < MR; ++u) {
        const int i = lane + 32 * u;
        x[u] = (i < m) ? ap[i] : 0.0;
        y[u] = (i < m) ? aq[i] : 0.0;
    }
    double al = 0.0, be = 0.0, ga = 0.0;
#pragma unroll
    for (int u = 0; u < MR; ++u) { al = fma(x[u], x[u], al); be = fma(y[u], y[u], be); ga = fma(x[u], y[u], ga); }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        al += __shfl_xor_sync(0xffffffffu, al, o);
        be += __shfl_xor_sync(0xffffffffu, be, o);
        ga += __shfl_xor_sync(0xffffffffu, ga, o);
    }
    // convergence test and angle in fp32 (magnitudes only need a few digits)
    const float fa = (float)al, fb = (float)be, fg = (float)ga;
    if (!(fabsf(fg) > tol * sqrtf(fa) * sqrtf(fb))) return false;
    const float zeta = (float)(be - al) / (2.0f * fg);
    float tf = copysignf(1.0f, zeta) / (fabsf(zeta) + sqrtf(fmaf(zeta, zeta, 1.0f)));
    if (!isfinite(zeta)) tf = 0.0f;
    const double t = (double)tf;
    const double c = rsqrt(fma(t, t, 1.0)), s = c * t;
#pragma unroll
    for (int u = 0; u < MR; ++u) {
        const int i = lane + 32 * u;
        if (i < m) {
            ap[i] = c * x[u] - s * y[u];
            aq[i] = s * x[u] + c * y[u];
        }
    }
    return true;
}

template <int MR>
__global__ void __launch_bounds__(32 * kBW)
jacobi_block_kernel(int m, int n, int nb, double *__restrict__ A, float tol, int max_sweeps,
                    int *__restrict__ counters, int *__restrict__ sweeps_out) {
    namespace cg = cooperative_groups;
    cg::grid_group grid = cg::this_grid();
    extern __shared__ __align__(16) double C[];          // [2*kBW][ldc]
    __shared__ int any_rot;
    const int ldc = m | 1;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int c = blockIdx.x;                              // this CTA's pair slot
    constexpr int NP = 2 * kBW;                            // players in the inner circle
    int sweep = 0;
    for (; sweep < max_sweeps; ++sweep) {
        if (tid == 0) any_rot = 0;
        for (int round = 0; round < nb - 1; ++round) {
            int bp, bq;
            if (c == 0) { bp = round; bq = nb - 1; }
            else { bp = (round + c) % (nb - 1); bq = (round - c + (nb - 1)) % (nb - 1); }
            // load the 2*kBW columns (zero padding beyond n): warp w moves columns w and w+kBW,
            // each lane issuing its MR strided elements at once
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int jl = warp + h * kBW;
                const int col = (h == 0 ? bp : bq) * kBW + warp;
                const double *src = A + (int64_t)m * col;
                double v[MR];
#pragma unroll
                for (int u = 0; u < MR; ++u) {
                    const int i = lane + 32 * u;
                    v[u] = (col < n && i < m) ? src[i] : 0.0;
                }
#pragma unroll
                for (int u = 0; u < MR; ++u) {
                    const int i = lane + 32 * u;
                    if (i < m) C[i + ldc * jl] = v[u];
                }
            }
            __syncthreads();
            // one inner sweep: circle method over NP players, kBW pairs per inner round
            for (int ir = 0; ir < NP - 1; ++ir) {
                int p, q;
                if (warp == 0) { p = ir; q = NP - 1; }
                else { p = (ir + warp) % (NP - 1); q = (ir - warp + (NP - 1)) % (NP - 1); }
                if (jacobi_pair<MR>(C + ldc * p, C + ldc * q, m, lane, tol) && lane == 0) any_rot = 1;
                __syncthreads();
            }
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int jl = warp + h * kBW;
                const int col = (h == 0 ? bp : bq) * kBW + warp;
                if (col < n) {
                    double *dst = A + (int64_t)m * col;
#pragma unroll
                    for (int u = 0; u < MR; ++u) {
                        const int i = lane + 32 * u;
                        if (i < m) dst[i] = C[i + ldc * jl];
                    }
                }
            }
            __threadfence();
            grid.sync();
        }
        if (tid == 0 && any_rot) atomicAdd(&counters[sweep], 1);
        __threadfence();
        grid.sync();
        if (counters[sweep] == 0) break;
    }
    if (c == 0 && tid == 0 && sweeps_out) *sweeps_out = sweep + 1;
}

void jacobi_svd_blocked(int m, int n, double *T, int *counters, int *sweeps, cudaStream_t st) {
    int nb = (int)cdiv(n, kBW);
    nb += nb & 1;
    if (nb < 2) nb = 2;
    const int grid = nb / 2;
    const size_t smem = sizeof(double) * (size_t)(m | 1) * 2 * kBW;
    SSA_REQUIRE(grid <= num_sms() && smem <= 200 * 1024 && m <= 32 * 24, SSA_ERR_ARG,
                "projected matrix too large for the device Jacobi");
    SSA_CUDA(cudaMemsetAsync(counters, 0, sizeof(int) * 64, st));
    float tol = 1e-12f;
    int max_sweeps = 60;
    void *args[] = {&m, &n, &nb, &T, &tol, &max_sweeps, &counters, &sweeps};
    void *kern = m <= 32 * 4 ? (void *)jacobi_block_kernel<4>
               : m <= 32 * 8 ? (void *)jacobi_block_kernel<8>
               : m <= 32 * 16 ? (void *)jacobi_block_kernel<16> : (void *)jacobi_block_kernel<24>;
    SSA_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    SSA_CUDA(cudaLaunchCooperativeKernel(kern, dim3(grid), dim3(32 * kBW), args, smem, st));
    after_launch("jacobi_block");
}

bool jacobi_blocked_fits(int m, int n) {
    int nb = (int)cdiv(n, kBW);
    nb += nb & 1;
    return nb / 2 <= num_sms() && sizeof(double) * (size_t)(m | 1) * 2 * kBW <= 200 * 1024 && m <= 32 * 24;
}

}  // namespace ssa

// ---- ABI utility: the solver's small SVD, exposed for tests and micro-benchmarks
extern "C" ssa_status ssa_small_svd(int32_t m, int32_t n, double *A, int32_t *sweeps, double *ms) {
    using namespace ssa;
    try {
        if (m < n || n < 1 || !A) throw Error(SSA_ERR_ARG, "ssa_small_svd needs m >= n >= 1");
        if (!jacobi_blocked_fits(m, n)) throw Error(SSA_ERR_ARG, "matrix too large for the device Jacobi");
        DevBuf d;
        d.alloc(sizeof(double) * ((size_t)m * n + 80), nullptr);
        int *ds = reinterpret_cast<int *>(d.as<double>() + (size_t)m * n);
        int *dc = ds + 16;
        SSA_CUDA(cudaMemcpy(d.p, A, sizeof(double) * m * n, cudaMemcpyHostToDevice));
        cudaEvent_t e0, e1;
        SSA_CUDA(cudaEventCreate(&e0)); SSA_CUDA(cudaEventCreate(&e1));
        SSA_CUDA(cudaEventRecord(e0, nullptr));
        jacobi_svd_blocked(m, n, d.as<double>(), dc, ds, nullptr);
        SSA_CUDA(cudaEventRecord(e1, nullptr));
        SSA_CUDA(cudaEventSynchronize(e1));
        float t = 0.f;
        SSA_CUDA(cudaEventElapsedTime(&t, e0, e1));
        cudaEventDestroy(e0); cudaEventDestroy(e1);
        if (ms) *ms = t;
        SSA_CUDA(cudaMemcpy(A, d.p, sizeof(double) * m * n, cudaMemcpyDeviceToHost));
        if (sweeps) SSA_CUDA(cudaMemcpy(sweeps, ds, sizeof(int32_t), cudaMemcpyDeviceToHost));
        return SSA_OK;
    } catch (const Error &e) {
        ssa_set_error(e.what());
        return e.code;
    }
}
