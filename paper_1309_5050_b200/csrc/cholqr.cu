// One CholeskyQR pass in a single cooperative launch (the CholeskyQR2 second
// pass of the block orthonormalisation, P:… block Lanczos with full reorthogonalisation):
//
//     G = WᵀW (fp64),   G (+ shift·I) = RᵀR,   W ← W R⁻¹          (W: M x kc fp32, in place)
//
// The separate path costs a Gram launch + reduction + host round trip + coefficient upload +
// update launch, and re-reads W from HBM for the update.  Here every CTA keeps its row slice
// of W in shared memory: phase 1 forms the slice's partial Gram (fp64 FMAs from the fp32
// data), a grid barrier, CTA 0 sums the partials in a fixed order (deterministic) and factors
// (Cholesky, shifted retry, triangular inverse) in shared memory, a second grid barrier, and
// every CTA applies R⁻¹ to its slice straight from shared memory.  W is read once and written
// once.  The factor R, the flags and max|G − I| go back to the host (one small D2H copy) for
// the solver's coefficient bookkeeping; a failed factorisation leaves W untouched.
#include <cooperative_groups.h>

#include "common.h"
#include "kernels.h"

namespace cg = cooperative_groups;

namespace ssa {

namespace cholqr {
constexpr int NT = 256;
constexpr int SMEM_SLICE = 220 * 1024;   // dynamic shared memory cap (scratch + W slice)
}

// out layout (doubles): R [KC*KC] | [0] ok, [1] shifted, [2] max|G − I|, [3] max diag.
// ws: partials [grid][KC*KC] | G [KC*KC] | S (fp32) [KC*KC]
template <int KC>
__global__ void __launch_bounds__(cholqr::NT, 1)
cholqr_fused_kernel(int64_t M, float *W, int64_t ld, int rows_per, double shift_rel, double thr_chol,
                    double *__restrict__ ws, double *__restrict__ out) {
    static_assert(KC == 32, "tiling below assumes 32 columns");
    cg::grid_group grid = cg::this_grid();
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int ldw = rows_per + 1;                      // odd stride
    // dynamic shared memory: reduction / factor scratch (static smem is capped at 48 KB), then the slice
    double *red = reinterpret_cast<double *>(smem_raw);                 // [4][KC*KC] (phase 1)
    double *G = red, *R = red + KC * KC, *S = R + KC * KC;              // CTA 0, phase 2 (aliases red)
    float *Ss = reinterpret_cast<float *>(red + 4 * KC * KC);           // [KC*KC]
    float *wsl = Ss + KC * KC;                                          // slice [KC][ldw]
    double *partials = ws, *Gg = ws + (size_t)gridDim.x * KC * KC;
    float *Sf = reinterpret_cast<float *>(Gg + KC * KC);
    const int tid = threadIdx.x;
    const int64_t r0 = (int64_t)blockIdx.x * rows_per;
    const int nr = (int)max((int64_t)0, min((int64_t)rows_per, M - r0));

    // ---- phase 1: slice -> shared memory; partial Gram, fp64, register-blocked 4 x 4:
    // thread = (4x4 tile of the 32 x 32 Gram: 64 tiles) x (row group: 4)
    for (int c = 0; c < KC; ++c)
        for (int r = tid; r < nr; r += cholqr::NT) wsl[c * ldw + r] = W[r0 + r + ld * c];
    __syncthreads();
    {
        const int tile = tid & 63, rg = tid >> 6;
        const int a0 = 4 * (tile & 7), b0 = 4 * (tile >> 3);
        double acc[4][4];
#pragma unroll
        for (int x = 0; x < 4; ++x)
#pragma unroll
            for (int y = 0; y < 4; ++y) acc[x][y] = 0.0;
        if (a0 <= b0 + 3) {
            for (int r = rg; r < nr; r += 4) {
                double va[4], vb[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    va[q] = (double)wsl[(a0 + q) * ldw + r];
                    vb[q] = (double)wsl[(b0 + q) * ldw + r];
                }
#pragma unroll
                for (int x = 0; x < 4; ++x)
#pragma unroll
                    for (int y = 0; y < 4; ++y) acc[x][y] = fma(va[x], vb[y], acc[x][y]);
            }
        }
        // sum the 4 row groups (the slice stays in the dynamic buffer for phase 3)
#pragma unroll
        for (int x = 0; x < 4; ++x)
#pragma unroll
            for (int y = 0; y < 4; ++y) red[rg * KC * KC + (a0 + x) + KC * (b0 + y)] = acc[x][y];
        __syncthreads();
        for (int e = tid; e < KC * KC; e += cholqr::NT)
            partials[(int64_t)blockIdx.x * KC * KC + e] =
                (red[e] + red[KC * KC + e]) + (red[2 * KC * KC + e] + red[3 * KC * KC + e]);
    }
    grid.sync();

    // ---- phase 2a: fixed-order reduction of the partials, entries spread over the CTAs
    for (int e = blockIdx.x * cholqr::NT + tid; e < KC * KC; e += gridDim.x * cholqr::NT) {
        const int i = e % KC, l = e / KC;
        if (i > l) continue;
        double s = 0.0;
        for (int c = 0; c < (int)gridDim.x; ++c) s += partials[(int64_t)c * KC * KC + e];
        Gg[i + KC * l] = s;
        Gg[l + KC * i] = s;
    }
    grid.sync();

    // ---- phase 2b (CTA 0): Cholesky (+ shifted retry) and R⁻¹ in shared memory
    __shared__ int s_fail;
    __shared__ double s_dmax, s_dev;
    if (blockIdx.x == 0) {
        for (int e = tid; e < KC * KC; e += cholqr::NT) G[e] = Gg[e];
        __syncthreads();
        if (tid < 32) {
            double dmax = 0.0, dev = 0.0;
            int bad = 0;
            for (int e = tid; e < KC * KC; e += 32) {
                const bool dg = (e % KC) == (e / KC);
                if (dg) dmax = fmax(dmax, G[e]);
                const double v = G[e] - (dg ? 1.0 : 0.0);
                if (!isfinite(v)) bad = 1;
                dev = fmax(dev, fabs(v));
            }
            for (int o = 16; o; o >>= 1) {
                dmax = fmax(dmax, __shfl_xor_sync(0xffffffffu, dmax, o));
                dev = fmax(dev, __shfl_xor_sync(0xffffffffu, dev, o));
                bad |= __shfl_xor_sync(0xffffffffu, bad, o);
            }
            if (tid == 0) {
                s_dmax = dmax;
                s_dev = dev;
                s_fail = bad || !(dmax > 0.0);
            }
        }
        __syncthreads();
        int shifted = 0;
        if (!s_fail) {
            for (int attempt = 0; attempt < 2; ++attempt) {
                const double shift = attempt ? shift_rel * s_dmax : 0.0;
                const double thr = attempt ? 1e-300 : thr_chol;
                for (int e = tid; e < KC * KC; e += cholqr::NT) {
                    const int i = e % KC, l = e / KC;
                    R[e] = i < l ? G[e] : (i == l ? G[e] + shift : 0.0);
                }
                __syncthreads();
                if (tid == 0) s_fail = 0;
                __syncthreads();
                for (int j = 0; j < KC; ++j) {
                    if (tid == 0) {
                        const double d = R[j + KC * j];
                        if (!(d > thr * s_dmax)) s_fail = 1;
                        else R[j + KC * j] = sqrt(d);
                    }
                    __syncthreads();
                    if (s_fail) break;
                    const double rjj = R[j + KC * j];
                    if (tid > j && tid < KC) R[j + KC * tid] /= rjj;
                    __syncthreads();
                    const int m = KC - j - 1;
                    for (int e = tid; e < m * m; e += cholqr::NT) {
                        const int i = j + 1 + e % m, l = j + 1 + e / m;
                        if (i <= l) R[i + KC * l] -= R[j + KC * i] * R[j + KC * l];
                    }
                    __syncthreads();
                }
                if (!s_fail) { shifted = attempt; break; }
                __syncthreads();
            }
        }
        if (!s_fail) {
            for (int j = tid; j < KC; j += cholqr::NT) {
                for (int i = 0; i < KC; ++i) S[i + KC * j] = 0.0;
                S[j + KC * j] = 1.0 / R[j + KC * j];
                for (int i = j - 1; i >= 0; --i) {
                    double v = 0.0;
                    for (int t = i + 1; t <= j; ++t) v += R[i + KC * t] * S[t + KC * j];
                    S[i + KC * j] = -v / R[i + KC * i];
                }
            }
            __syncthreads();
            for (int e = tid; e < KC * KC; e += cholqr::NT) {
                out[e] = R[e];
                Sf[e] = (float)S[e];
            }
        }
        if (tid == 0) {
            out[KC * KC + 0] = s_fail ? 0.0 : 1.0;
            out[KC * KC + 1] = shifted;
            out[KC * KC + 2] = s_dev;
            out[KC * KC + 3] = s_dmax;
        }
    }
    grid.sync();

    // ---- phase 3: W ← W R⁻¹ from the shared-memory slice (skipped when the factorisation failed)
    if (out[KC * KC + 0] == 0.0) return;
    for (int e = tid; e < KC * KC; e += cholqr::NT) Ss[e] = Sf[e];
    __syncthreads();
    for (int r = tid; r < nr; r += cholqr::NT) {
        float x[KC];
#pragma unroll
        for (int a = 0; a < KC; ++a) x[a] = wsl[a * ldw + r];
#pragma unroll 1
        for (int b = 0; b < KC; ++b) {
            float acc = 0.f;
#pragma unroll
            for (int a = 0; a < KC; ++a)
                if (a <= b) acc = fmaf(x[a], Ss[a + KC * b], acc);
            W[r0 + r + ld * b] = acc;
        }
    }
}

// Launches the fused pass when the shape fits (kc = 32, W slices in shared memory, all CTAs
// co-resident); returns false otherwise.  `out` (device, kc·kc + 4 doubles) receives R and the
// flags; the caller copies it to the host and synchronises.  `ws`: device scratch of at least
// cholqr_ws_bytes(kc) bytes.
size_t cholqr_ws_bytes(int kc) {
    return sizeof(double) * ((size_t)1025 * kc * kc) + sizeof(float) * (size_t)kc * kc;
}
bool cholqr_fused(int64_t M, float *W, int64_t ld, int kc, double shift_rel, double thr_chol, double *ws, size_t ws_bytes,
                  double *out, cudaStream_t st) {
    // opt-in (SSA_CHOLQR_FUSED=1): measured slower than the separate path (c3 24.5 vs 23.0 ms, c2 9.9 vs
    // 9.1 ms): the fp64 CUDA-core slice Gram and three grid barriers cost more than the round trip saved
    static const int mode = [] { const char *e = std::getenv("SSA_CHOLQR_FUSED"); return e ? std::atoi(e) : 0; }();
    if (!mode || kc != 32 || M < 1) return false;
    const int nsm = num_sms();
    int grid = (int)std::min<int64_t>(nsm, cdiv(M, 64));
    const int rows_per = (int)((cdiv(M, grid) + 31) / 32 * 32);
    grid = (int)cdiv(M, rows_per);
    const size_t smem = sizeof(double) * 4 * kc * kc + sizeof(float) * (size_t)kc * kc +
                        sizeof(float) * (size_t)kc * (rows_per + 1);
    if (smem > (size_t)cholqr::SMEM_SLICE || grid > 1024 || ws_bytes < cholqr_ws_bytes(kc)) return false;
    void *fn = (void *)cholqr_fused_kernel<32>;
    set_max_smem_impl(fn);
    int per_sm = 0;
    SSA_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, cholqr::NT, smem));
    if (per_sm * nsm < grid) return false;
    int rp = rows_per;
    void *args[] = {&M, &W, &ld, &rp, &shift_rel, &thr_chol, &ws, &out};
    SSA_CUDA(cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(cholqr::NT), args, smem, st));
    after_launch("cholqr_fused");
    return true;
}

}  // namespace ssa
