// Tall-skinny dense helpers for the block Lanczos solver:
// Gram matrices Aᵀ B (fp64 accumulation across CTAs, deterministic), small
// right-multiplications A·C, column scaling, and a counter-based normal RNG.
// All are HBM-bound streaming kernels over M = L or K rows.
#include "common.h"
#include <cstdlib>
#include <cmath>
#include <vector>
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
                                   double *__restrict__ G, int ldg) {
    const int e = (blockIdx.x * blockDim.x + threadIdx.x) / 32, lane = threadIdx.x % 32;
    if (e >= n1 * n2) return;
    const int a = e % n1, b = e / n1;
    const double *base = partials + (int64_t)(a / 64) * nparts * 4096;
    const int al = a % 64;
    double s = 0.0;
    for (int q = lane; q < nparts; q += 32) s += base[(int64_t)q * 4096 + al + 64 * b];
#pragma unroll
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) G[a + (int64_t)ldg * b] = s;
}

void gram_reduce(const double *partials, int nparts, int n1, int n2, double *G, cudaStream_t st, int ldg) {
    gram_reduce_kernel<<<(unsigned)cdiv((int64_t)n1 * n2 * 32, 256), 256, 0, st>>>(partials, nparts, n1, n2, G,
                                                                                     ldg > 0 ? ldg : n1);
    after_launch("gram_reduce");
}

static int gram_ctas(int64_t M) {
    return (int)std::max<int64_t>(1, std::min<int64_t>(cdiv(M, 64), 2 * (int64_t)num_sms()));
}

size_t gram_partial_bytes(int64_t M, int n1, int) {
    return (size_t)gram_ctas(M) * 4096 * sizeof(double) * (size_t)cdiv(std::max(n1, 64), 64);
}

// ---------------------------------------------------------------------------
// Streaming fp32 Gram for tall-skinny column-major blocks (the K-side CGS / CholeskyQR
// Grams): G (n1 x n2) = AᵀB over M rows, 16-byte aligned columns (lda, ldb % 4 == 0).
// A CTA (256 threads, one per SM) walks 32-row chunks c, c + G, ... of all n1p (<= 256)
// columns of A and NB columns of B, staged by a 4-deep cp.async pipeline into
// column-major smem tiles (row pitch 36 floats: 16-byte rows of 4, pitch/4 odd).
// Thread tile: 8 A columns (ti + 8a) x 4 B columns (tj + NB/4·b) — strided so the 8
// threads of an LDS.128 phase hit distinct bank groups for A and broadcast B — each
// step consuming 4 rows (12 LDS.128, 128 FFMA).  fp32 partial sums per 32 rows are
// folded into fp64 accumulators; row groups (when n1 is small) are combined through
// shared memory; per-CTA partials go to gram_reduce (fixed order, deterministic).
// ---------------------------------------------------------------------------
namespace gram2 {
constexpr int R = 32, LDR = 36, STAGES = 4, NT = 256;
__device__ __forceinline__ void cp_async16(float *dst, const float *src, int src_bytes) {
    const uint32_t d = (uint32_t)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(src), "r"(src_bytes));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;"); }
template <int N> __device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N)); }
}  // namespace gram2

template <int NB>
__global__ void __launch_bounds__(256, 1)
gram_stream_kernel(int64_t M, const float *__restrict__ A, int64_t lda, int n1, const float *__restrict__ B,
                   int64_t ldb, int n2, int YG, double *__restrict__ partials) {
    using namespace gram2;
    extern __shared__ __align__(16) unsigned char gs_raw[];
    float *sm = reinterpret_cast<float *>(gs_raw);
    constexpr int TPT = 8 * (NB / 4);                  // threads per 64 x NB tile
    const int tid = threadIdx.x;
    const int RG = (NT / TPT) / YG;                     // row groups
    const int ncolA = 64 * YG;                          // A columns staged per CTA
    const int stage_f = (ncolA + NB) * LDR;             // floats per stage
    A += lda * (int64_t)(ncolA * blockIdx.y);
    const int n1c = min(ncolA, n1 - ncolA * (int)blockIdx.y);
    const int g = tid / TPT, yg = g % YG, rg = g / YG;
    const int ti = tid % 8, tj = (tid / 8) % (NB / 4);
    const int64_t nchunks = (M + R - 1) / R;
    // ---- loader: (n1c + n2) columns x R/4 float4 per stage
    auto load = [&](int64_t chunk, int buf) {
        float *As = sm + buf * stage_f, *Bs = As + ncolA * LDR;
        const int64_t r0 = chunk * R;
        const int tot = (n1c + n2) * (R / 4);
        for (int idx = tid; idx < tot; idx += NT) {
            const int col = idx / (R / 4), q = idx % (R / 4);
            const int64_t row = r0 + 4 * q;
            const int64_t rem = M - row;
            const int bytes = rem >= 4 ? 16 : (rem > 0 ? 4 * (int)rem : 0);
            if (col < n1c) cp_async16(As + col * LDR + 4 * q, A + lda * col + (bytes ? row : 0), bytes);
            else {
                const int cb = col - n1c;
                cp_async16(Bs + cb * LDR + 4 * q, B + ldb * cb + (bytes ? row : 0), bytes);
            }
        }
    };
    // zero the column padding once (columns n1c..ncolA-1 and n2..NB-1 stay zero)
    for (int idx = tid; idx < STAGES * stage_f; idx += NT) sm[idx] = 0.f;
    __syncthreads();
    // chunks of this CTA: a contiguous range
    const int64_t per = (nchunks + gridDim.x - 1) / gridDim.x;
    const int64_t c0 = blockIdx.x * per, cstep = 1;
    const int64_t my = max((int64_t)0, min(per, nchunks - c0));
#pragma unroll
    for (int s = 0; s < STAGES - 1; ++s) {
        if (s < my) load(c0 + (int64_t)s * cstep, s);
        cp_commit();
    }
    double accd[8][4];
#pragma unroll
    for (int a = 0; a < 8; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) accd[a][b] = 0.0;
    const int colA0 = 64 * yg + ti;
    for (int64_t i = 0; i < my; ++i) {
        cp_wait<STAGES - 2>();
        __syncthreads();
        {
            const int64_t nx = i + STAGES - 1;
            if (nx < my) load(c0 + nx * cstep, (int)(nx % STAGES));
            cp_commit();
        }
        const float *As = sm + (int)(i % STAGES) * stage_f, *Bs = As + ncolA * LDR;
        float acc[8][4];
#pragma unroll
        for (int a = 0; a < 8; ++a)
#pragma unroll
            for (int b = 0; b < 4; ++b) acc[a][b] = 0.f;
        for (int q = rg; q < R / 4; q += RG) {
            float4 av[8], bv[4];
#pragma unroll
            for (int a = 0; a < 8; ++a) av[a] = *reinterpret_cast<const float4 *>(As + (colA0 + 8 * a) * LDR + 4 * q);
#pragma unroll
            for (int b = 0; b < 4; ++b) bv[b] = *reinterpret_cast<const float4 *>(Bs + (tj + (NB / 4) * b) * LDR + 4 * q);
#pragma unroll
            for (int a = 0; a < 8; ++a)
#pragma unroll
                for (int b = 0; b < 4; ++b) {
                    acc[a][b] = fmaf(av[a].x, bv[b].x, acc[a][b]);
                    acc[a][b] = fmaf(av[a].y, bv[b].y, acc[a][b]);
                    acc[a][b] = fmaf(av[a].z, bv[b].z, acc[a][b]);
                    acc[a][b] = fmaf(av[a].w, bv[b].w, acc[a][b]);
                }
        }
#pragma unroll
        for (int a = 0; a < 8; ++a)
#pragma unroll
            for (int b = 0; b < 4; ++b) accd[a][b] += (double)acc[a][b];
    }
    cp_wait<0>();
    __syncthreads();
    // ---- combine row groups (fixed order) and write this CTA's partial tiles
    double *red = reinterpret_cast<double *>(sm);        // [RG][YG][64][NB]
    if (RG > 1) {
#pragma unroll
        for (int a = 0; a < 8; ++a)
#pragma unroll
            for (int b = 0; b < 4; ++b)
                red[((rg * YG + yg) * 64 + ti + 8 * a) * NB + tj + (NB / 4) * b] = accd[a][b];
        __syncthreads();
        if (rg == 0) {
#pragma unroll
            for (int a = 0; a < 8; ++a)
#pragma unroll
                for (int b = 0; b < 4; ++b) {
                    double s = accd[a][b];
                    for (int r2 = 1; r2 < RG; ++r2) s += red[((r2 * YG + yg) * 64 + ti + 8 * a) * NB + tj + (NB / 4) * b];
                    accd[a][b] = s;
                }
        }
    }
    if (rg != 0) return;
    const int ych = (int)blockIdx.y * YG + yg;          // global 64-column chunk of A
    if (64 * yg >= n1c) return;
    double *out = partials + ((int64_t)ych * gridDim.x + blockIdx.x) * 4096;
#pragma unroll
    for (int a = 0; a < 8; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            const int al = ti + 8 * a, bl = tj + (NB / 4) * b;
            if (bl < n2) out[al + 64 * bl] = accd[a][b];
        }
}

static bool gram_stream(int64_t M, const float *A, int64_t lda, int n1, const float *B, int64_t ldb, int n2,
                        double *G, double *partials, size_t partial_bytes, cudaStream_t st) {
    if (M < 4096 || (lda & 3) || (ldb & 3) || ((uintptr_t)A & 15) || ((uintptr_t)B & 15) || n2 > 64) return false;
    const int NB = n2 <= 32 ? 32 : 64;
    const int tiles = (NB == 32) ? 4 : 2;               // 64 x NB tiles computed in parallel per CTA
    const int ych = (int)cdiv(n1, 64);
    const int YG = std::min(ych, tiles);
    const int gy = (int)cdiv(ych, YG);
    const int ctas = (int)std::min<int64_t>(num_sms(), cdiv(M, gram2::R));
    if ((size_t)ctas * 4096 * sizeof(double) * (size_t)ych > partial_bytes) return false;
    // pipeline stages; reused at the end for the row-group combine ([RG][YG][64][NB] doubles)
    const size_t smem = std::max(sizeof(float) * (size_t)gram2::STAGES * (64 * YG + NB) * gram2::LDR,
                                 sizeof(double) * (size_t)tiles * 64 * NB);
    if (NB == 32) {
        set_max_smem(gram_stream_kernel<32>);
        gram_stream_kernel<32><<<dim3(ctas, gy), 256, smem, st>>>(M, A, lda, n1, B, ldb, n2, YG, partials);
    } else {
        set_max_smem(gram_stream_kernel<64>);
        gram_stream_kernel<64><<<dim3(ctas, gy), 256, smem, st>>>(M, A, lda, n1, B, ldb, n2, YG, partials);
    }
    after_launch("gram_stream");
    gram_reduce_kernel<<<(unsigned)cdiv((int64_t)n1 * n2 * 32, 256), 256, 0, st>>>(partials, ctas, n1, n2, G, n1);
    after_launch("gram_reduce");
    return true;
}

template <typename T>
void gram_tn(int64_t M, const T *A, int64_t lda, int n1, const T *B, int64_t ldb, int n2,
             double *G, double *partials, size_t partial_bytes, cudaStream_t st) {
    SSA_REQUIRE(n2 <= 64 && n1 <= 512, SSA_ERR_ARG, "gram_tn: at most 512 x 64 per call");
    if constexpr (sizeof(T) == 4) {
        if (gram_tc(M, A, lda, n1, B, ldb, n2, G, partials, partial_bytes, st)) return;
        if (gram_stream(M, A, lda, n1, B, ldb, n2, G, partials, partial_bytes, st)) return;
    }
    const int ctas = gram_ctas(M);
    const int ych = (int)cdiv(n1, 64);
    SSA_REQUIRE((size_t)ctas * 4096 * sizeof(double) * ych <= partial_bytes, SSA_ERR_ARG, "gram_tn: workspace");
    gram_tn_kernel<T><<<dim3(ctas, ych), 256, 0, st>>>(M, A, lda, n1, B, ldb, n2, partials);
    after_launch("gram_tn");
    gram_reduce_kernel<<<(unsigned)cdiv((int64_t)n1 * n2 * 32, 256), 256, 0, st>>>(partials, ctas, n1, n2, G, n1);
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
        if (beta != 0.0) {
            T old[16];
#pragma unroll
            for (int j = 0; j < 16; ++j) old[j] = (b0 + j < n) ? Out[row + ldo * (b0 + j)] : T(0);
#pragma unroll
            for (int j = 0; j < 16; ++j) acc[j] = fma((T)beta, old[j], acc[j]);
        }
#pragma unroll
        for (int j = 0; j < 16; ++j)
            if (b0 + j < n) Out[row + ldo * (b0 + j)] = acc[j];
    }
}

// ---------------------------------------------------------------------------
// Streaming fp32 update for tall-skinny blocks (CGS projections, recurrence terms,
// CholeskyQR applies): Out (M x n) = beta·Out + alpha·A (M x m)·C (m x n), n <= NC, Out may
// equal A (in place: every row tile is read completely before it is written).
// 128 threads per CTA, one CTA per SM walking 256-row tiles; each tile streams its m columns
// in 32-column chunks through a 3-deep cp.async pipeline ([32 cols][256 rows] smem tiles).
// Thread t owns rows 2t, 2t+1 of the tile and all NC outputs (2·NC fp32 accumulators):
// per column one LDS.64 of A and NC/4 broadcast LDS.128 of alpha·C (fp32, in smem).
// ---------------------------------------------------------------------------
namespace upd2 {
constexpr int ROWS = 256, KC = 32, STAGES = 3, NT = 128;
}

template <int NC>
__global__ void __launch_bounds__(128, 1)
tall_update_kernel(int64_t M, const float *A, int64_t lda, int m, const double *__restrict__ C, int ldc, int n,
                   double alpha, double beta, float *Out, int64_t ldo) {
    using namespace upd2;
    using gram2::cp_async16;
    using gram2::cp_commit;
    using gram2::cp_wait;
    extern __shared__ __align__(16) unsigned char us_raw[];
    float *Cs = reinterpret_cast<float *>(us_raw);                 // [m][NC] alpha·C
    float *St = Cs + (size_t)m * NC;                                 // [STAGES][KC][ROWS]
    const int tid = threadIdx.x;
    for (int idx = tid; idx < m * NC; idx += NT) {
        const int a = idx / NC, b = idx % NC;
        Cs[idx] = (b < n) ? (float)(alpha * C[a + (int64_t)ldc * b]) : 0.f;
    }
    const int nchk = (m + KC - 1) / KC;
    const int64_t ntiles = (M + ROWS - 1) / ROWS;
    // work items (tile, chunk) of this CTA, in order
    const int64_t my_tiles = (ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x;
    const int64_t nitems = my_tiles * nchk;
    auto load = [&](int64_t it, int buf) {
        const int64_t tile = blockIdx.x + (it / nchk) * gridDim.x;
        const int ch = (int)(it % nchk);
        const int64_t r0 = tile * ROWS;
        float *dst = St + (size_t)buf * KC * ROWS;
        const int ncol = min(KC, m - ch * KC);
        for (int idx = tid; idx < KC * (ROWS / 4); idx += NT) {
            const int c = idx / (ROWS / 4), q = idx % (ROWS / 4);
            const int64_t row = r0 + 4 * q;
            const int64_t rem = M - row;
            const int bytes = (c < ncol) ? (rem >= 4 ? 16 : (rem > 0 ? 4 * (int)rem : 0)) : 0;
            cp_async16(dst + c * ROWS + 4 * q, A + lda * (int64_t)(ch * KC + (c < ncol ? c : 0)) + (bytes ? row : 0), bytes);
        }
    };
#pragma unroll
    for (int st = 0; st < STAGES - 1; ++st) {
        if (st < nitems) load(st, st);
        cp_commit();
    }
    __syncthreads();   // Cs ready
    float acc0[NC], acc1[NC];
#pragma unroll
    for (int j = 0; j < NC; ++j) { acc0[j] = 0.f; acc1[j] = 0.f; }
    for (int64_t it = 0; it < nitems; ++it) {
        cp_wait<STAGES - 2>();
        __syncthreads();
        {
            const int64_t nx = it + STAGES - 1;
            if (nx < nitems) load(nx, (int)(nx % STAGES));
            cp_commit();
        }
        const int ch = (int)(it % nchk);
        const float *Sb = St + (size_t)(it % STAGES) * KC * ROWS;
        const int ncol = min(KC, m - ch * KC);
        for (int c = 0; c < ncol; ++c) {
            const float2 a = *reinterpret_cast<const float2 *>(Sb + c * ROWS + 2 * tid);
            const float4 *cr = reinterpret_cast<const float4 *>(Cs + (size_t)(ch * KC + c) * NC);
#pragma unroll
            for (int j4 = 0; j4 < NC / 4; ++j4) {
                const float4 cv = cr[j4];
                acc0[4 * j4 + 0] = fmaf(a.x, cv.x, acc0[4 * j4 + 0]);
                acc0[4 * j4 + 1] = fmaf(a.x, cv.y, acc0[4 * j4 + 1]);
                acc0[4 * j4 + 2] = fmaf(a.x, cv.z, acc0[4 * j4 + 2]);
                acc0[4 * j4 + 3] = fmaf(a.x, cv.w, acc0[4 * j4 + 3]);
                acc1[4 * j4 + 0] = fmaf(a.y, cv.x, acc1[4 * j4 + 0]);
                acc1[4 * j4 + 1] = fmaf(a.y, cv.y, acc1[4 * j4 + 1]);
                acc1[4 * j4 + 2] = fmaf(a.y, cv.z, acc1[4 * j4 + 2]);
                acc1[4 * j4 + 3] = fmaf(a.y, cv.w, acc1[4 * j4 + 3]);
            }
        }
        if (ch == nchk - 1) {
            // tile complete: every column of these rows has been read (cp.async data consumed
            // above); write the outputs, then reset the accumulators
            const int64_t tile = blockIdx.x + (it / nchk) * gridDim.x;
            const int64_t row = tile * ROWS + 2 * tid;
            const float fb = (float)beta;
            if (beta != 0.0) {   // old values first (independent loads in flight), then the stores
#pragma unroll
                for (int j = 0; j < NC; ++j) {
                    if (j < n && row + 1 < M) {
                        const float2 old = __ldcg(reinterpret_cast<const float2 *>(Out + row + ldo * (int64_t)j));
                        acc0[j] = fmaf(fb, old.x, acc0[j]);
                        acc1[j] = fmaf(fb, old.y, acc1[j]);
                    } else if (j < n && row < M) {
                        acc0[j] = fmaf(fb, __ldcg(Out + row + ldo * (int64_t)j), acc0[j]);
                    }
                }
            }
#pragma unroll
            for (int j = 0; j < NC; ++j) {
                if (j < n) {
                    float *o = Out + row + ldo * (int64_t)j;
                    if (row + 1 < M) *reinterpret_cast<float2 *>(o) = make_float2(acc0[j], acc1[j]);
                    else if (row < M) o[0] = acc0[j];
                }
                acc0[j] = 0.f;
                acc1[j] = 0.f;
            }
        }
    }
    cp_wait<0>();
}

// true when handled (fp32, aligned columns, M large); Out == A allowed
static bool tall_update(int64_t M, const float *A, int64_t lda, int m, const double *C, int ldc, int n, double alpha,
                        double beta, float *Out, int64_t ldo, cudaStream_t st) {
    // measured (scripts/bench_tall.py): faster than the thread-per-row kernel only for wide
    // blocks (m >= 256, n > 32: 4.2 vs 7.1 ms at M = 1.8M, m = 356, n = 64)
    if (!(m >= 256 && n > 32)) return false;
    if (M < 8192 || n > 64 || m > 512 || (lda & 3) || (ldo & 1) || ((uintptr_t)A & 15) || ((uintptr_t)Out & 7))
        return false;
    const int NC = n <= 32 ? 32 : 64;
    const size_t smem = sizeof(float) * ((size_t)m * NC + (size_t)upd2::STAGES * upd2::KC * upd2::ROWS);
    if (smem > 220 * 1024) return false;
    const int ctas = (int)std::min<int64_t>(num_sms(), cdiv(M, upd2::ROWS));
    if (NC == 32) {
        set_max_smem(tall_update_kernel<32>);
        tall_update_kernel<32><<<ctas, upd2::NT, smem, st>>>(M, A, lda, m, C, ldc, n, alpha, beta, Out, ldo);
    } else {
        set_max_smem(tall_update_kernel<64>);
        tall_update_kernel<64><<<ctas, upd2::NT, smem, st>>>(M, A, lda, m, C, ldc, n, alpha, beta, Out, ldo);
    }
    after_launch("tall_update");
    return true;
}

template <typename T>
static bool gemm_split(int64_t M, const T *A, int64_t lda, int m, const double *C, int ldc, int n, double alpha,
                       double beta, T *Out, int64_t ldo, cudaStream_t st);

template <typename T>
void gemm_small(int64_t M, const T *A, int64_t lda, int m, const double *C, int ldc, int n,
                double alpha, double beta, T *Out, int64_t ldo, cudaStream_t st) {
    SSA_REQUIRE(m <= 64 && n <= 64, SSA_ERR_ARG, "gemm_small: at most 64x64");
    if (M <= 0 || n <= 0) return;
    if constexpr (sizeof(T) == 4) {
        if (update_tc(M, A, lda, m, C, ldc, n, alpha, beta, Out, ldo, st)) return;
        if (tall_update(M, A, lda, m, C, ldc, n, alpha, beta, Out, ldo, st)) return;
    }
    if (gemm_split<T>(M, A, lda, m, C, ldc, n, alpha, beta, Out, ldo, st)) return;   // small M, in place ok
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
    // all old values first (independent loads in flight), then the stores
    if (beta != 0.0) {
        T old[NMAX];
#pragma unroll
        for (int j = 0; j < NMAX; ++j) old[j] = (j < n) ? Out[row + ldo * j] : T(0);
#pragma unroll
        for (int j = 0; j < NMAX; ++j) acc[j] = fma((T)beta, old[j], acc[j]);
    }
#pragma unroll
    for (int j = 0; j < NMAX; ++j)
        if (j < n) Out[row + ldo * j] = acc[j];
}

// Small-M variant (M < 16384, the L side): the m-long reduction of a row is split over the 8
// warps of a CTA (warp w: columns w, w+8, ...; lane = row), partial sums meet in shared memory.
// 4x the CTAs and 1/8 of the dependent loop of the thread-per-row kernel (33 µs -> see DESIGN).
// A CTA owns its 32 rows, so Out may be the trailing columns of A (all reads precede the
// reduction barrier, all writes follow it).
template <typename T, int NMAX>
__global__ void __launch_bounds__(256)
gemm_acc_split_kernel(int64_t M, const T *A, int64_t lda, int m, const double *__restrict__ C, int ldc, int n,
                      double alpha, double beta, T *Out, int64_t ldo) {
    extern __shared__ __align__(16) unsigned char ss_raw[];
    T *CS = reinterpret_cast<T *>(ss_raw);          // [m][NMAX] alpha·C
    T *red = CS + (size_t)m * NMAX;                   // [8][32][NMAX + 1] partial sums
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
#pragma unroll 4
    for (int idx = tid; idx < m * NMAX; idx += 256) {
        const int b = idx / m, a = idx - b * m;       // a (row of C) fastest: coalesced reads of C
        CS[a * NMAX + b] = (b < n) ? (T)(alpha * C[a + (int64_t)ldc * b]) : T(0);
    }
    __syncthreads();
    const int64_t row = (int64_t)blockIdx.x * 32 + lane;
    T acc[NMAX];
#pragma unroll
    for (int j = 0; j < NMAX; ++j) acc[j] = T(0);
    if (row < M) {
        int c = w;
        for (; c + 8 < m; c += 16) {                  // two columns per iteration: loads in flight
            const T a0 = A[row + lda * (int64_t)c], a1 = A[row + lda * (int64_t)(c + 8)];
            const T *c0 = CS + c * NMAX, *c1 = CS + (c + 8) * NMAX;
#pragma unroll
            for (int j = 0; j < NMAX; ++j) acc[j] = fma(a1, c1[j], fma(a0, c0[j], acc[j]));
        }
        if (c < m) {
            const T a0 = A[row + lda * (int64_t)c];
            const T *c0 = CS + c * NMAX;
#pragma unroll
            for (int j = 0; j < NMAX; ++j) acc[j] = fma(a0, c0[j], acc[j]);
        }
    }
#pragma unroll
    for (int j = 0; j < NMAX; ++j) red[(w * 32 + lane) * (NMAX + 1) + j] = acc[j];
    __syncthreads();
    // thread -> (row lane', outputs j = jg, jg + 8, ...): fixed summation order over the warps
    const int rl = tid & 31, jg = tid >> 5;
    const int64_t r = (int64_t)blockIdx.x * 32 + rl;
    if (r >= M) return;
    for (int j = jg; j < n; j += 8) {
        T s = T(0);
#pragma unroll
        for (int q = 0; q < 8; ++q) s += red[(q * 32 + rl) * (NMAX + 1) + j];
        T *o = Out + r + ldo * (int64_t)j;
        *o = (beta == 0.0) ? s : fma((T)beta, *o, s);
    }
}

template <typename T>
static bool gemm_split(int64_t M, const T *A, int64_t lda, int m, const double *C, int ldc, int n, double alpha,
                       double beta, T *Out, int64_t ldo, cudaStream_t st) {
    if (M >= 16384 || n > 64) return false;
    const unsigned g = (unsigned)cdiv(M, 32);
    if (n <= 32) {
        const size_t smem = sizeof(T) * ((size_t)m * 32 + 8 * 32 * 33);
        if (smem > 200 * 1024) return false;
        set_max_smem(gemm_acc_split_kernel<T, 32>);
        gemm_acc_split_kernel<T, 32><<<g, 256, smem, st>>>(M, A, lda, m, C, ldc, n, alpha, beta, Out, ldo);
    } else {
        const size_t smem = sizeof(T) * ((size_t)m * 64 + 8 * 32 * 65);
        if (smem > 200 * 1024) return false;
        set_max_smem(gemm_acc_split_kernel<T, 64>);
        gemm_acc_split_kernel<T, 64><<<g, 256, smem, st>>>(M, A, lda, m, C, ldc, n, alpha, beta, Out, ldo);
    }
    after_launch("gemm_acc_split");
    return true;
}

template <typename T>
void gemm_acc(int64_t M, const T *A, int64_t lda, int m, const double *C, int ldc, int n, double alpha,
              double beta, T *Out, int64_t ldo, cudaStream_t st) {
    SSA_REQUIRE(m <= 512 && n <= 64, SSA_ERR_ARG, "gemm_acc: at most 512 x 64");
    if (M <= 0 || n <= 0) return;
    if constexpr (sizeof(T) == 4) {
        if (update_tc(M, A, lda, m, C, ldc, n, alpha, beta, Out, ldo, st)) return;
        if (tall_update(M, A, lda, m, C, ldc, n, alpha, beta, Out, ldo, st)) return;
    }
    if (gemm_split<T>(M, A, lda, m, C, ldc, n, alpha, beta, Out, ldo, st)) return;
    const unsigned grid = (unsigned)cdiv(M, 128);
    if (n <= 32) {
        const size_t smem = sizeof(T) * (size_t)m * 32;
        set_max_smem(gemm_acc_kernel<T, 32>);
        gemm_acc_kernel<T, 32><<<grid, 128, smem, st>>>(M, A, lda, m, C, ldc, n, alpha, beta, Out, ldo);
    } else {
        const size_t smem = sizeof(T) * (size_t)m * 64;
        set_max_smem(gemm_acc_kernel<T, 64>);
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
    if constexpr (sizeof(T) == 4) {
        // fp32 plans: one hash per Box–Muller pair (rows 2i, 2i+1 get r·cos, r·sin), 24-bit uniforms
        // and fp32 transcendentals (c5's random refills of 14.75M-row columns were compute bound)
        const int64_t mp = (M + 1) / 2, n = mp * ncols;
        for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
            const int64_t pr = t % mp, col = t / mp;
            const uint64_t h = mix64(seed ^ mix64(sid * 0x100000001B3ull + (uint64_t)col) ^ (uint64_t)pr * 0xD6E8FEB86659FD93ull);
            const float u1 = (float)((uint32_t)(h >> 40) + 1u) * 0x1p-24f;              // (0, 1]
            const float u2 = (float)(uint32_t)((h >> 8) & 0xFFFFFFu) * 0x1p-24f;         // [0, 1)
            const float r = sqrtf(-2.0f * logf(u1));
            float sn, cs;
            sincospif(2.0f * u2, &sn, &cs);
            const int64_t row = 2 * pr;
            A[row + lda * col] = r * cs;
            if (row + 1 < M) A[row + 1 + lda * col] = r * sn;
        }
    } else {
        const int64_t n = M * ncols;
        for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
            const int64_t row = t % M, col = t / M;
            const uint64_t h = mix64(seed ^ mix64(sid * 0x100000001B3ull + (uint64_t)col) ^ (uint64_t)row * 0xD6E8FEB86659FD93ull);
            const double u1 = ((h >> 11) + 1.0) * (1.0 / 9007199254740993.0);
            const double u2 = (double)(mix64(h) >> 11) * (1.0 / 9007199254740992.0);
            A[row + lda * col] = (T)(sqrt(-2.0 * log(u1)) * cospi(2.0 * u2));
        }
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

// ---- ABI test hook: timing of the tall-skinny kernels on seeded device data
extern "C" ssa_status ssa_bench_tall(int32_t which, int64_t M, int32_t n1, int32_t n2, int32_t reps, double *ms,
                                     double *check) {
    using namespace ssa;
    try {
        // probe: n1 = columns + 1000 x L2-prefetch distance (stages), n2 = rows per box (32: swizzled)
        const int pd = which == 4 ? (n1 >= 0 ? n1 / 1000 : -((-n1) / 1000)) : 0, prow = std::abs(n2);
        if (which == 4 && n1 < 0) n1 = -n1;
        const bool pswz = n2 == 32;
        if (which == 4) {
            n1 %= 1000;
            n2 = std::min(prow, 64);
            if (n1 < 1 || n1 > 128 || prow < 8 || prow > 256) throw Error(SSA_ERR_ARG, "ssa_bench_tall: bad probe sizes");
        }
        if (M < 1 || n1 < 1 || n1 > 512 || n2 < 1 || n2 > 64 || reps < 1 || which < 0 || which > 5 || which == 2 ||
            (which == 5 && n2 > n1))
            throw Error(SSA_ERR_ARG, "ssa_bench_tall: bad sizes");
        const int64_t ld = (M + 31) / 32 * 32;
        DevBuf a, b, g, ws, c;
        a.alloc(sizeof(float) * ld * n1, nullptr);
        b.alloc(sizeof(float) * ld * n2, nullptr);
        g.alloc(sizeof(double) * 512 * 64, nullptr);
        c.alloc(sizeof(double) * 512 * 64, nullptr);
        const size_t wsb = gram_partial_bytes(M, 512, 64);
        ws.alloc(wsb, nullptr);
        SSA_CUDA(cudaMemset(a.p, 0, sizeof(float) * ld * n1));
        SSA_CUDA(cudaMemset(b.p, 0, sizeof(float) * ld * n2));
        fill_normal<float>(M, a.as<float>(), ld, n1, 7, 1, nullptr);
        fill_normal<float>(M, b.as<float>(), ld, n2, 7, 2, nullptr);
        std::vector<double> hc((size_t)n1 * n2);
        for (size_t t = 0; t < hc.size(); ++t) hc[t] = 0.1 * ((double)((t * 7919) % 1000) / 1000.0 - 0.5);
        SSA_CUDA(cudaMemcpy(c.p, hc.data(), sizeof(double) * hc.size(), cudaMemcpyHostToDevice));
        auto run = [&]() {
            if (which == 0) gram_tn<float>(M, a.as<float>(), ld, n1, b.as<float>(), ld, n2, g.as<double>(), ws.as<double>(), wsb, nullptr);
            else if (which == 3) gram_tn<float>(M, a.as<float>(), ld, n1, a.as<float>(), ld, n2, g.as<double>(), ws.as<double>(), wsb, nullptr);
            // projection Gram [A W]ᵀW of the solver: B = the last n2 columns of A (read from A's tiles)
            else if (which == 5) gram_tn<float>(M, a.as<float>(), ld, n1, a.as<float>() + ld * (n1 - n2), ld, n2, g.as<double>(), ws.as<double>(), wsb, nullptr);
            // probe: n1 columns, n2 = rows per box (32: 128-B swizzled boxes, else unswizzled), 128 rows per stage
            else if (which == 4) tma_stream_probe(M, a.as<float>(), ld, n1, prow, std::max(1, 128 / prow), pswz, pd, nullptr);
            else gemm_acc<float>(M, a.as<float>(), ld, n1, c.as<double>(), n1, n2, -1.0, 1.0, b.as<float>(), ld, nullptr);
        };
        run();
        cudaEvent_t e0, e1;
        SSA_CUDA(cudaEventCreate(&e0)); SSA_CUDA(cudaEventCreate(&e1));
        SSA_CUDA(cudaEventRecord(e0, nullptr));
        for (int i = 0; i < reps; ++i) run();
        SSA_CUDA(cudaEventRecord(e1, nullptr));
        SSA_CUDA(cudaEventSynchronize(e1));
        float t = 0.f;
        SSA_CUDA(cudaEventElapsedTime(&t, e0, e1));
        cudaEventDestroy(e0); cudaEventDestroy(e1);
        if (ms) *ms = t / reps;
        if (check && which == 1) {
            // max relative error of one update against an fp64 host evaluation on sampled rows
            fill_normal<float>(M, b.as<float>(), ld, n2, 7, 2, nullptr);
            std::vector<float> w0((size_t)ld * n2), w1((size_t)ld * n2), ha((size_t)ld * n1);
            SSA_CUDA(cudaMemcpy(w0.data(), b.p, sizeof(float) * w0.size(), cudaMemcpyDeviceToHost));
            SSA_CUDA(cudaMemcpy(ha.data(), a.p, sizeof(float) * ha.size(), cudaMemcpyDeviceToHost));
            run();
            SSA_CUDA(cudaMemcpy(w1.data(), b.p, sizeof(float) * w1.size(), cudaMemcpyDeviceToHost));
            double emax = 0.0, ref_max = 0.0;
            for (int64_t r = 0; r < M; r += std::max<int64_t>(1, M / 997)) {
                for (int j = 0; j < n2; ++j) {
                    double v = w0[r + ld * j];
                    for (int c = 0; c < n1; ++c) v -= (double)ha[r + ld * c] * hc[c + (size_t)n1 * j];
                    emax = std::max(emax, std::fabs(v - (double)w1[r + ld * j]));
                    ref_max = std::max(ref_max, std::fabs(v));
                }
            }
            *check = emax / std::max(ref_max, 1e-300);
        } else if (check) {
            double s = 0.0;
            if (which == 0 || which == 3 || which == 5) {
                std::vector<double> hg((size_t)n1 * n2);
                SSA_CUDA(cudaMemcpy(hg.data(), g.p, sizeof(double) * hg.size(), cudaMemcpyDeviceToHost));
                if ((double)M * n1 * n2 <= 5e8) {
                    // max relative error against an fp64 host Gram of the same fp32 data
                    std::vector<float> ha((size_t)ld * n1), hb((size_t)ld * n2);
                    SSA_CUDA(cudaMemcpy(ha.data(), a.p, sizeof(float) * ha.size(), cudaMemcpyDeviceToHost));
                    SSA_CUDA(cudaMemcpy(hb.data(), b.p, sizeof(float) * hb.size(), cudaMemcpyDeviceToHost));
                    const std::vector<float> &hB = (which == 3 || which == 5) ? ha : hb;
                    const int64_t bo = (which == 5) ? (int64_t)(n1 - n2) * ld : 0;
                    double emax = 0.0, gmax = 0.0;
                    for (int j = 0; j < n2; ++j)
                        for (int i = 0; i < n1; ++i) {
                            double v = 0.0;
                            for (int64_t r = 0; r < M; ++r) v += (double)ha[r + ld * i] * (double)hB[bo + r + ld * j];
                            emax = std::max(emax, std::fabs(v - hg[i + (size_t)n1 * j]));
                            gmax = std::max(gmax, std::fabs(v));
                        }
                    s = emax / std::max(gmax, 1e-300);
                } else {
                    for (double v : hg) s += std::fabs(v);
                }
            } else {
                std::vector<float> hw((size_t)ld * n2);
                SSA_CUDA(cudaMemcpy(hw.data(), b.p, sizeof(float) * hw.size(), cudaMemcpyDeviceToHost));
                for (float v : hw) s += std::fabs((double)v);
            }
            *check = s;
        }
        return SSA_OK;
    } catch (const Error &e) {
        ssa_set_error(e.what());
        return e.code;
    }
}
