// Tall-skinny dense helpers for the block Lanczos solver:
// Gram matrices Aᵀ B (fp64 accumulation across CTAs, deterministic), small
// right-multiplications A·C, column scaling, and a counter-based normal RNG.
// All are HBM-bound streaming kernels over M = L or K rows.
#include "common.h"
#include "kernels.h"

namespace ssa {

template <typename T> struct GramRows { static constexpr int value = sizeof(T) == 4 ? 64 : 32; };
constexpr int kGramPad = 4;

// One CTA = 256 threads, thread (ti, tj) owns G[4ti..4ti+3, 4tj..4tj+3].
template <typename T>
__global__ void __launch_bounds__(256)
gram_tn_kernel(int64_t M, const T *__restrict__ A, int64_t lda, int n1,
               const T *__restrict__ B, int64_t ldb, int n2, double *__restrict__ partials) {
    constexpr int kGramRows = GramRows<T>::value;   // rows staged per iteration (static smem < 48 KB)
    constexpr int P1 = 64 + kGramPad;
    __shared__ __align__(16) T AS[kGramRows * P1];
    __shared__ __align__(16) T BS[kGramRows * P1];
    const int tid = threadIdx.x;
    const int ti = tid % 16, tj = tid / 16;
    double accd[4][4];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) accd[a][b] = 0.0;
    // grid.y selects a 64-column chunk of A (one launch for up to 64*gridDim.y columns)
    A += lda * 64 * (int64_t)blockIdx.y;
    n1 = min(64, n1 - 64 * (int)blockIdx.y);
    const bool active = (4 * ti < n1) && (4 * tj < n2);
    for (int64_t r0 = (int64_t)blockIdx.x * kGramRows; r0 < M; r0 += (int64_t)gridDim.x * kGramRows) {
        __syncthreads();
        for (int idx = tid; idx < kGramRows * 64; idx += 256) {
            const int rl = idx % kGramRows, c = idx / kGramRows;
            const int64_t row = r0 + rl;
            T va = T(0), vb = T(0);
            if (row < M) {
                if (c < n1) va = A[row + lda * c];
                if (c < n2) vb = B[row + ldb * c];
            }
            AS[rl * P1 + c] = va;
            BS[rl * P1 + c] = vb;
        }
        __syncthreads();
        if (active) {
            T acc[4][4];
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
                for (int b = 0; b < 4; ++b) acc[a][b] = T(0);
#pragma unroll 4
            for (int rl = 0; rl < kGramRows; ++rl) {
                T av[4], bv[4];
#pragma unroll
                for (int a = 0; a < 4; ++a) { av[a] = AS[rl * P1 + 4 * ti + a]; bv[a] = BS[rl * P1 + 4 * tj + a]; }
#pragma unroll
                for (int a = 0; a < 4; ++a)
#pragma unroll
                    for (int b = 0; b < 4; ++b) acc[a][b] = fma(av[a], bv[b], acc[a][b]);
            }
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
                for (int b = 0; b < 4; ++b) accd[a][b] += (double)acc[a][b];
        }
    }
    if (!active) return;
    double *out = partials + ((int64_t)blockIdx.y * gridDim.x + blockIdx.x) * 64 * 64;
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) out[(4 * ti + a) + 64 * (4 * tj + b)] = accd[a][b];
}

// One warp per Gram entry: lanes sum strided partials, then a fixed shuffle tree
// (deterministic order).
__global__ void gram_reduce_kernel(const double *__restrict__ partials, int nparts, int n1, int n2,
                                   double *__restrict__ G) {
    const int e = (blockIdx.x * blockDim.x + threadIdx.x) / 32, lane = threadIdx.x % 32;
    if (e >= n1 * n2) return;
    const int a = e % n1, b = e / n1;
    const double *base = partials + (int64_t)(a / 64) * nparts * 4096;
    const int al = a % 64;
    double s = 0.0;
    for (int q = lane; q < nparts; q += 32) s += base[(int64_t)q * 4096 + al + 64 * b];
#pragma unroll
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) G[a + (int64_t)n1 * b] = s;
}

static int gram_ctas(int64_t M) {
    return (int)std::max<int64_t>(1, std::min<int64_t>(cdiv(M, 64), 2 * (int64_t)num_sms()));
}

size_t gram_partial_bytes(int64_t M, int n1, int) {
    return (size_t)gram_ctas(M) * 4096 * sizeof(double) * (size_t)cdiv(std::max(n1, 64), 64);
}

template <typename T>
void gram_tn(int64_t M, const T *A, int64_t lda, int n1, const T *B, int64_t ldb, int n2,
             double *G, double *partials, size_t partial_bytes, cudaStream_t st) {
    SSA_REQUIRE(n2 <= 64 && n1 <= 512, SSA_ERR_ARG, "gram_tn: at most 512 x 64 per call");
    const int ctas = gram_ctas(M);
    const int ych = (int)cdiv(n1, 64);
    SSA_REQUIRE((size_t)ctas * 4096 * sizeof(double) * ych <= partial_bytes, SSA_ERR_ARG, "gram_tn: workspace");
    gram_tn_kernel<T><<<dim3(ctas, ych), 256, 0, st>>>(M, A, lda, n1, B, ldb, n2, partials);
    after_launch("gram_tn");
    gram_reduce_kernel<<<(unsigned)cdiv((int64_t)n1 * n2 * 32, 256), 256, 0, st>>>(partials, ctas, n1, n2, G);
    after_launch("gram_reduce");
}
template void gram_tn<float>(int64_t, const float *, int64_t, int, const float *, int64_t, int, double *,
                             double *, size_t, cudaStream_t);
template void gram_tn<double>(int64_t, const double *, int64_t, int, const double *, int64_t, int,
                              double *, double *, size_t, cudaStream_t);

// Out = beta*Out + alpha*A*C.  Thread per row; the row of A is held in registers
// before any store, so Out == A (m == n) is safe.
template <typename T>
__global__ void __launch_bounds__(128)
gemm_small_kernel(int64_t M, const T *A, int64_t lda, int m, const double *__restrict__ C, int ldc,
                  int n, double alpha, double beta, T *Out, int64_t ldo, bool inplace) {
    __shared__ T CS[64 * 64];
    for (int idx = threadIdx.x; idx < m * n; idx += blockDim.x) {
        const int a = idx % m, b = idx / m;
        CS[a * 64 + b] = (T)(alpha * C[a + (int64_t)ldc * b]);
    }
    __syncthreads();
    const int64_t row = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (row >= M) return;
    T a[64];
#pragma unroll
    for (int c = 0; c < 64; ++c) a[c] = (c < m) ? A[row + lda * c] : T(0);
    // in-place (Out == A) needs one CTA column to own all outputs of its rows
    const int bstep = inplace ? 16 : 16 * gridDim.y;
    for (int b0 = inplace ? 0 : 16 * blockIdx.y; b0 < n; b0 += bstep) {
        T acc[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) acc[j] = T(0);
#pragma unroll
        for (int c = 0; c < 64; ++c) {
            if (c < m) {
#pragma unroll
                for (int j = 0; j < 16; ++j) acc[j] = fma(a[c], CS[c * 64 + b0 + j], acc[j]);
            }
        }
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            const int b = b0 + j;
            if (b < n) {
                T *o = Out + row + ldo * b;
                *o = (beta == 0.0) ? acc[j] : fma((T)beta, *o, acc[j]);
            }
        }
    }
}

template <typename T>
void gemm_small(int64_t M, const T *A, int64_t lda, int m, const double *C, int ldc, int n,
                double alpha, double beta, T *Out, int64_t ldo, cudaStream_t st) {
    SSA_REQUIRE(m <= 64 && n <= 64, SSA_ERR_ARG, "gemm_small: at most 64x64");
    if (M <= 0 || n <= 0) return;
    const bool inplace = (Out == A);
    // small M: spread the column chunks over more CTAs (not in place)
    const int gy = inplace ? 1 : (int)std::min<int64_t>(cdiv(n, 16), std::max<int64_t>(1, (2 * num_sms()) / cdiv(M, 128)));
    dim3 grid((unsigned)cdiv(M, 128), gy);
    gemm_small_kernel<T><<<grid, 128, 0, st>>>(M, A, lda, m, C, ldc, n, alpha, beta, Out, ldo, inplace);
    after_launch("gemm_small");
}
template void gemm_small<float>(int64_t, const float *, int64_t, int, const double *, int, int, double,
                                double, float *, int64_t, cudaStream_t);
template void gemm_small<double>(int64_t, const double *, int64_t, int, const double *, int, int, double,
                                 double, double *, int64_t, cudaStream_t);

// Out (M x n) = beta*Out + alpha * A (M x m) * C (m x n); m <= 512, n <= 64, Out != A.
// Thread per row: A streamed in 16-column chunks (one read of A), all n outputs in registers.
template <typename T, int NMAX>
__global__ void __launch_bounds__(128)
gemm_acc_kernel(int64_t M, const T *__restrict__ A, int64_t lda, int m, const double *__restrict__ C, int ldc,
                int n, double alpha, double beta, T *__restrict__ Out, int64_t ldo) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    T *CS = reinterpret_cast<T *>(smem_raw);   // [m][NMAX]
    for (int idx = threadIdx.x; idx < m * NMAX; idx += blockDim.x) {
        const int a = idx / NMAX, b = idx % NMAX;
        CS[idx] = (b < n) ? (T)(alpha * C[a + (int64_t)ldc * b]) : T(0);
    }
    __syncthreads();
    const int64_t row = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (row >= M) return;
    T acc[NMAX];
#pragma unroll
    for (int j = 0; j < NMAX; ++j) acc[j] = T(0);
    for (int c0 = 0; c0 < m; c0 += 16) {
        T a[16];
#pragma unroll
        for (int t = 0; t < 16; ++t) a[t] = (c0 + t < m) ? A[row + lda * (c0 + t)] : T(0);
#pragma unroll
        for (int t = 0; t < 16; ++t) {
            if (c0 + t >= m) break;
            const T *cr = CS + (c0 + t) * NMAX;
#pragma unroll
            for (int j = 0; j < NMAX; ++j) acc[j] = fma(a[t], cr[j], acc[j]);
        }
    }
#pragma unroll
    for (int j = 0; j < NMAX; ++j) {
        if (j < n) {
            T *o = Out + row + ldo * j;
            *o = (beta == 0.0) ? acc[j] : fma((T)beta, *o, acc[j]);
        }
    }
}

template <typename T>
void gemm_acc(int64_t M, const T *A, int64_t lda, int m, const double *C, int ldc, int n, double alpha,
              double beta, T *Out, int64_t ldo, cudaStream_t st) {
    SSA_REQUIRE(m <= 512 && n <= 64, SSA_ERR_ARG, "gemm_acc: at most 512 x 64");
    if (M <= 0 || n <= 0) return;
    const unsigned grid = (unsigned)cdiv(M, 128);
    if (n <= 32) {
        const size_t smem = sizeof(T) * (size_t)m * 32;
        SSA_CUDA(cudaFuncSetAttribute(gemm_acc_kernel<T, 32>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        gemm_acc_kernel<T, 32><<<grid, 128, smem, st>>>(M, A, lda, m, C, ldc, n, alpha, beta, Out, ldo);
    } else {
        const size_t smem = sizeof(T) * (size_t)m * 64;
        SSA_CUDA(cudaFuncSetAttribute(gemm_acc_kernel<T, 64>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        gemm_acc_kernel<T, 64><<<grid, 128, smem, st>>>(M, A, lda, m, C, ldc, n, alpha, beta, Out, ldo);
    }
    after_launch("gemm_acc");
}
template void gemm_acc<float>(int64_t, const float *, int64_t, int, const double *, int, int, double, double,
                              float *, int64_t, cudaStream_t);
template void gemm_acc<double>(int64_t, const double *, int64_t, int, const double *, int, int, double, double,
                               double *, int64_t, cudaStream_t);

// ---- counter-based normal generator (splitmix64 + Box-Muller) -------------
__device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

template <typename T>
__global__ void fill_normal_kernel(int64_t M, T *A, int64_t lda, int ncols, uint64_t seed, uint64_t sid) {
    const int64_t n = M * ncols;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t row = t % M, col = t / M;
        const uint64_t h = mix64(seed ^ mix64(sid * 0x100000001B3ull + (uint64_t)col) ^ (uint64_t)row * 0xD6E8FEB86659FD93ull);
        const double u1 = ((h >> 11) + 1.0) * (1.0 / 9007199254740993.0);
        const double u2 = (double)(mix64(h) >> 11) * (1.0 / 9007199254740992.0);
        A[row + lda * col] = (T)(sqrt(-2.0 * log(u1)) * cospi(2.0 * u2));
    }
}

template <typename T>
void fill_normal(int64_t M, T *A, int64_t lda, int ncols, uint64_t seed, uint64_t sid, cudaStream_t st) {
    const int64_t n = M * ncols;
    if (n <= 0) return;
    fill_normal_kernel<T><<<(unsigned)std::min<int64_t>(cdiv(n, 256), 16 * num_sms()), 256, 0, st>>>(
        M, A, lda, ncols, seed, sid);
    after_launch("fill_normal");
}
template void fill_normal<float>(int64_t, float *, int64_t, int, uint64_t, uint64_t, cudaStream_t);
template void fill_normal<double>(int64_t, double *, int64_t, int, uint64_t, uint64_t, cudaStream_t);

template <typename T>
__global__ void scale_columns_kernel(int64_t M, T *A, int64_t lda, int n, const double *__restrict__ s) {
    const int64_t tot = M * n;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < tot; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t row = t % M, col = t / M;
        A[row + lda * col] *= (T)s[col];
    }
}

template <typename T>
void scale_columns(int64_t M, T *A, int64_t lda, int n, const double *s, cudaStream_t st) {
    const int64_t tot = M * n;
    if (tot <= 0) return;
    scale_columns_kernel<T><<<(unsigned)std::min<int64_t>(cdiv(tot, 256), 16 * num_sms()), 256, 0, st>>>(
        M, A, lda, n, s);
    after_launch("scale_columns");
}
template void scale_columns<float>(int64_t, float *, int64_t, int, const double *, cudaStream_t);
template void scale_columns<double>(int64_t, double *, int64_t, int, const double *, cudaStream_t);

}  // namespace ssa

namespace ssa {
// Sign convention: flip each column so that its
// largest-|.| entry is positive.  One CTA per column; writes ±1 into sgn.
template <typename T>
__global__ void absmax_sign_kernel(int64_t M, const T *A, int64_t lda, double *sgn) {
    const int col = blockIdx.x;
    double best = -1.0; int64_t bi = 0;
    for (int64_t i = threadIdx.x; i < M; i += blockDim.x) {
        const double v = fabs((double)A[i + lda * col]);
        if (v > best) { best = v; bi = i; }
    }
    __shared__ double sb[256];
    __shared__ int64_t si[256];
    sb[threadIdx.x] = best; si[threadIdx.x] = bi;
    __syncthreads();
    for (int o = blockDim.x / 2; o; o >>= 1) {
        if ((int)threadIdx.x < o) {
            const double b2 = sb[threadIdx.x + o]; const int64_t i2 = si[threadIdx.x + o];
            if (b2 > sb[threadIdx.x] || (b2 == sb[threadIdx.x] && i2 < si[threadIdx.x])) {
                sb[threadIdx.x] = b2; si[threadIdx.x] = i2;
            }
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) sgn[col] = ((double)A[si[0] + lda * col] < 0.0) ? -1.0 : 1.0;
}
template <typename T>
void absmax_sign(int64_t M, const T *A, int64_t lda, int n, double *sgn, cudaStream_t st) {
    if (n <= 0) return;
    absmax_sign_kernel<T><<<n, 256, 0, st>>>(M, A, lda, sgn);
    after_launch("absmax_sign");
}
template void absmax_sign<float>(int64_t, const float *, int64_t, int, double *, cudaStream_t);
template void absmax_sign<double>(int64_t, const double *, int64_t, int, double *, cudaStream_t);
}  // namespace ssa

namespace ssa {

// ============================================================================
// Device-resident block orthonormalisation (one CGS + CholeskyQR pass per call
// pair orth_solve / apply_inplace; the solver runs two or three passes with a
// single host synchronisation).  For W (M x kc) following `na` orthonormal
// columns A in the same buffer ([A W] contiguous, ld M):
//   G = [A W]ᵀ W  (gram_tn)   C = G[0:na, :]   Gp = WᵀW − CᵀC  (= W'ᵀW', W' = W − A C)
//   Gp (+ shift) = RᵀR        S = R⁻¹          W ← W' S = [A W]·[−C S; S]
// Coefficients accumulate so that W_in = A·Ctot + W_out·Btot holds exactly:
//   pass 1: Ctot = C, Btot = R;   pass p > 1: Ctot += C·Btot, Btot = R·Btot.
// flags[0] trouble (non-finite Gram, a column numerically in span(A) or zero —
//          the host then redoes the block with the robust path),
// flags[1] pass 1 needed a shifted Cholesky, flags[2] another pass is needed
//          (shifted, or pass-p Gram far from identity), flags[3] = pass count.
// ============================================================================
__global__ void __launch_bounds__(256)
orth_solve_kernel(const double *__restrict__ G, int na, int kc, int pass, double zthr2, double shift_rel,
                  double thr_chol, int c_in_smem, double *__restrict__ Mout, double *__restrict__ Ctot,
                  double *__restrict__ Btot, int *__restrict__ flags) {
    extern __shared__ double sm[];
    double *Gp = sm;
    double *R = Gp + kc * kc;
    double *S = R + kc * kc;
    double *Bo = S + kc * kc;
    double *Cs = Bo + kc * kc;   // na x kc (only if c_in_smem)
    __shared__ int s_fail;
    __shared__ double s_dmax, s_dev;
    const int n1 = na + kc, tid = threadIdx.x, nt = blockDim.x;
    const double *C = G;
    int ldc = n1;
    if (c_in_smem) {   // odd leading dimension: column-parallel reads hit distinct banks
        ldc = na | 1;
        for (int e = tid; e < na * kc; e += nt) Cs[(e % na) + (size_t)ldc * (e / na)] = G[(e % na) + (size_t)n1 * (e / na)];
        C = Cs;
    }
    if (pass >= 2)
        for (int e = tid; e < kc * kc; e += nt) Bo[e] = Btot[e];
    __syncthreads();
    for (int e = tid; e < kc * kc; e += nt) {
        const int a = e % kc, b = e / kc;
        if (a > b) continue;
        double s = G[na + a + (size_t)n1 * b];
        const double *ca = C + (size_t)ldc * a, *cb = C + (size_t)ldc * b;
        for (int t = 0; t < na; ++t) s -= ca[t] * cb[t];
        Gp[a + kc * b] = s;
        Gp[b + kc * a] = s;
    }
    __syncthreads();
    if (tid == 0) {
        double dmax = 0.0, dev = 0.0;
        int bad = 0;
        for (int j = 0; j < kc; ++j) {
            const double d = Gp[j + kc * j];
            if (!isfinite(d)) bad = 1;
            dmax = fmax(dmax, d);
            if (pass == 1 && !(d > zthr2)) bad = 1;
        }
        for (int e = 0; e < kc * kc; ++e) {
            const double v = Gp[e] - ((e % kc) == (e / kc) ? 1.0 : 0.0);
            if (!isfinite(v)) bad = 1;
            dev = fmax(dev, fabs(v));
        }
        if (!(dmax > 0.0)) bad = 1;
        s_dmax = dmax;
        s_dev = dev;
        s_fail = bad;
    }
    __syncthreads();
    if (s_fail) {
        if (tid == 0) flags[0] = 1;
        return;
    }
    int shifted = 0;
    for (int attempt = 0; attempt < 2; ++attempt) {
        const double shift = attempt ? shift_rel * s_dmax : 0.0;
        const double thr = attempt ? 0.0 : thr_chol * s_dmax;
        for (int e = tid; e < kc * kc; e += nt) R[e] = Gp[e] + (((e % kc) == (e / kc)) ? shift : 0.0);
        __syncthreads();
        if (tid == 0) s_fail = 0;
        __syncthreads();
        for (int j = 0; j < kc; ++j) {
            if (tid == 0) {
                const double d = R[j + kc * j];
                if (!(d > thr)) s_fail = 1;
                else R[j + kc * j] = sqrt(d);
            }
            __syncthreads();
            if (s_fail) break;
            const double rjj = R[j + kc * j];
            for (int i = j + 1 + tid; i < kc; i += nt) R[j + kc * i] /= rjj;
            __syncthreads();
            const int m = kc - j - 1;
            for (int e = tid; e < m * m; e += nt) {
                const int a = j + 1 + e % m, b = j + 1 + e / m;
                if (a <= b) R[a + kc * b] -= R[j + kc * a] * R[j + kc * b];
            }
            __syncthreads();
        }
        if (!s_fail) { shifted = attempt; break; }
        __syncthreads();
    }
    if (s_fail) {
        if (tid == 0) flags[0] = 1;
        return;
    }
    for (int e = tid; e < kc * kc; e += nt)
        if ((e % kc) > (e / kc)) R[e] = 0.0;
    __syncthreads();
    // S = R^-1 (upper triangular), one column per thread
    for (int j = tid; j < kc; j += nt) {
        for (int i = 0; i < kc; ++i) S[i + kc * j] = 0.0;
        S[j + kc * j] = 1.0 / R[j + kc * j];
        for (int i = j - 1; i >= 0; --i) {
            double v = 0.0;
            for (int t = i + 1; t <= j; ++t) v += R[i + kc * t] * S[t + kc * j];
            S[i + kc * j] = -v / R[i + kc * i];
        }
    }
    __syncthreads();
    // Mout = [-C S ; S]
    for (int e = tid; e < n1 * kc; e += nt) {
        const int t = e % n1, b = e / n1;
        double v;
        if (t < na) {
            v = 0.0;
            for (int a = 0; a <= b; ++a) v -= C[t + (size_t)ldc * a] * S[a + kc * b];
        } else {
            v = S[(t - na) + kc * b];
        }
        Mout[e] = v;
    }
    // coefficient bookkeeping
    if (pass == 1) {
        for (int e = tid; e < na * kc; e += nt) Ctot[e] = C[(e % na) + (size_t)ldc * (e / na)];
        for (int e = tid; e < kc * kc; e += nt) Btot[e] = R[e];
    } else {
        for (int e = tid; e < na * kc; e += nt) {
            const int t = e % na, b = e / na;
            double v = Ctot[e];
            for (int a = 0; a < kc; ++a) v += C[t + (size_t)ldc * a] * Bo[a + kc * b];
            Ctot[e] = v;
        }
        for (int e = tid; e < kc * kc; e += nt) {
            const int a = e % kc, b = e / kc;
            double v = 0.0;
            for (int t = a; t < kc; ++t) v += R[a + kc * t] * Bo[t + kc * b];
            Btot[e] = v;
        }
    }
    if (tid == 0) {
        if (pass == 1) flags[1] = shifted;
        flags[2] = (shifted || (pass >= 2 && s_dev > 0.1)) ? 1 : 0;
        flags[3] = pass;
    }
}

// W[:, 0:kc] = A[:, 0:n1] · Mc (n1 x kc, device double) where W = A + lda·(n1 - kc):
// the block being orthonormalised is the last kc columns of its own input.  Thread
// per row; every input of a row is read before any of its outputs is written.
template <typename T, int NMAX>
__global__ void __launch_bounds__(128)
apply_inplace_kernel(int64_t M, T *A, int64_t lda, int n1, int kc, const double *Mc, const int *skip) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    if (skip && *skip != 0) return;   // the solve flagged trouble: leave W for the host's robust path
    T *CS = reinterpret_cast<T *>(smem_raw);   // [n1][NMAX]
    for (int idx = threadIdx.x; idx < n1 * NMAX; idx += blockDim.x) {
        const int c = idx / NMAX, b = idx % NMAX;
        CS[idx] = (b < kc) ? (T)Mc[c + (int64_t)n1 * b] : T(0);
    }
    __syncthreads();
    const int64_t row = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (row >= M) return;
    T acc[NMAX];
#pragma unroll
    for (int j = 0; j < NMAX; ++j) acc[j] = T(0);
    const T *ar = A + row;
    int c0 = 0;
    for (; c0 + 8 <= n1; c0 += 8) {
        T a[8];
#pragma unroll
        for (int t = 0; t < 8; ++t) a[t] = ar[lda * (c0 + t)];
#pragma unroll
        for (int t = 0; t < 8; ++t) {
            const T *cr = CS + (c0 + t) * NMAX;
#pragma unroll
            for (int j = 0; j < NMAX; ++j) acc[j] = fma(a[t], cr[j], acc[j]);
        }
    }
    for (; c0 < n1; ++c0) {
        const T a = ar[lda * c0];
        const T *cr = CS + c0 * NMAX;
#pragma unroll
        for (int j = 0; j < NMAX; ++j) acc[j] = fma(a, cr[j], acc[j]);
    }
    T *w = A + lda * (int64_t)(n1 - kc) + row;
#pragma unroll
    for (int j = 0; j < NMAX; ++j)
        if (j < kc) w[lda * j] = acc[j];
}

void orth_solve(const double *G, int na, int kc, int pass, double zthr2, double shift_rel, double thr_chol,
                double *Mout, double *Ctot, double *Btot, int *flags, cudaStream_t st) {
    SSA_REQUIRE(kc <= 64 && na + kc <= 512, SSA_ERR_ARG, "orth_solve: at most 64 new columns against 448");
    const size_t base = sizeof(double) * 4 * (size_t)kc * kc;
    const size_t cbytes = sizeof(double) * (size_t)(na | 1) * kc;
    const int c_in_smem = (base + cbytes <= 200 * 1024) ? 1 : 0;
    const size_t smem = base + (c_in_smem ? cbytes : 0);
    SSA_CUDA(cudaFuncSetAttribute(orth_solve_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    orth_solve_kernel<<<1, 256, smem, st>>>(G, na, kc, pass, zthr2, shift_rel, thr_chol, c_in_smem, Mout, Ctot, Btot,
                                            flags);
    after_launch("orth_solve");
}

template <typename T>
void apply_inplace(int64_t M, T *A, int64_t lda, int n1, int kc, const double *Mc, const int *skip, cudaStream_t st) {
    SSA_REQUIRE(kc <= 64 && n1 <= 512, SSA_ERR_ARG, "apply_inplace: at most 512 x 64");
    if (M <= 0) return;
    const unsigned grid = (unsigned)cdiv(M, 128);
    if (kc <= 32) {
        const size_t smem = sizeof(T) * (size_t)n1 * 32;
        SSA_CUDA(cudaFuncSetAttribute(apply_inplace_kernel<T, 32>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        apply_inplace_kernel<T, 32><<<grid, 128, smem, st>>>(M, A, lda, n1, kc, Mc, skip);
    } else {
        const size_t smem = sizeof(T) * (size_t)n1 * 64;
        SSA_CUDA(cudaFuncSetAttribute(apply_inplace_kernel<T, 64>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        apply_inplace_kernel<T, 64><<<grid, 128, smem, st>>>(M, A, lda, n1, kc, Mc, skip);
    }
    after_launch("apply_inplace");
}
template void apply_inplace<float>(int64_t, float *, int64_t, int, int, const double *, const int *, cudaStream_t);
template void apply_inplace<double>(int64_t, double *, int64_t, int, int, const double *, const int *, cudaStream_t);

}  // namespace ssa

namespace ssa {
// Out (M x n) = A (M x m) · C (m x n, device double), Out != A: thread per (row, group of
// 8 output columns), grid (ceil(M/128), ceil(n/8)) — enough CTAs for short bases (L side).
template <typename T>
__global__ void __launch_bounds__(128)
gemm_cols_kernel(int64_t M, const T *__restrict__ A, int64_t lda, int m, const double *__restrict__ C, int ldc, int n,
                 T *__restrict__ Out, int64_t ldo) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    T *CS = reinterpret_cast<T *>(smem_raw);   // [m][8]
    const int c0 = blockIdx.y * 8;
    for (int idx = threadIdx.x; idx < m * 8; idx += blockDim.x) {
        const int a = idx / 8, b = idx % 8;
        CS[idx] = (c0 + b < n) ? (T)C[a + (int64_t)ldc * (c0 + b)] : T(0);
    }
    __syncthreads();
    const int64_t row = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (row >= M) return;
    T acc[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[j] = T(0);
    const T *ar = A + row;
#pragma unroll 4
    for (int a = 0; a < m; ++a) {
        const T v = ar[lda * a];
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[j] = fma(v, CS[a * 8 + j], acc[j]);
    }
#pragma unroll
    for (int j = 0; j < 8; ++j)
        if (c0 + j < n) Out[row + ldo * (c0 + j)] = acc[j];
}

template <typename T>
void gemm_cols(int64_t M, const T *A, int64_t lda, int m, const double *C, int ldc, int n, T *Out, int64_t ldo,
               cudaStream_t st) {
    if (M <= 0 || n <= 0) return;
    const size_t smem = sizeof(T) * (size_t)m * 8;
    SSA_REQUIRE(smem <= 200 * 1024, SSA_ERR_ARG, "gemm_cols: too many input columns");
    SSA_CUDA(cudaFuncSetAttribute(gemm_cols_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    gemm_cols_kernel<T><<<dim3((unsigned)cdiv(M, 128), (unsigned)cdiv(n, 8)), 128, smem, st>>>(M, A, lda, m, C, ldc, n,
                                                                                            Out, ldo);
    after_launch("gemm_cols");
}
template void gemm_cols<float>(int64_t, const float *, int64_t, int, const double *, int, int, float *, int64_t,
                               cudaStream_t);
template void gemm_cols<double>(int64_t, const double *, int64_t, int, const double *, int, int, double *, int64_t,
                                cudaStream_t);
}  // namespace ssa
