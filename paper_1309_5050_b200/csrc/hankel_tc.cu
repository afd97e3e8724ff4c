// Tensor-core (tcgen05, sm_100a) implicit GEMM for the trajectory-operator
// products of arXiv 1309.5050, 3xTF32 split for fp32
// accuracy (SURVEY finding 3: 1xTF32 misses the 1e-5 product bar).
//
// Both products are one correlation of the image with k filters evaluated on an
// output box (direct.cu has the same definition on CUDA cores):
//
//     out[p, j] = Σ_{d ∈ in-box} x[p + d] · in[d, j]        (eq. P:3020-3028, 0-based)
//
//   X·V  : p ∈ 𝔏-box, d ∈ 𝔎-box, in = V      Xᵀ·U : p ∈ 𝔎-box, d ∈ 𝔏-box, in = U
//
// GEMM view per output column p_y: D[m, j] (M = 128 consecutive p_x) += A[m, kk] B[kk, j]
// with kk running over (d_y, d_x).  For fixed d_y, A[m, d_x] = x[p_x0 + m + d_x, p_y + d_y]
// is a Hankel block.  The Hankel structure is used twice:
//   * a chunk of NB k-blocks (32 d_x each) needs only the strip
//         S[i, jj] = x[p_x0 + d_x0 + i + jj, p_y + d_y],  i < 128 + 32(NB-1), jj < 32,
//     because A for k-block b is rows [32b, 32b + 128) of S — the UMMA shared-memory
//     descriptor of k-block b is the strip descriptor advanced by 4 core-matrix
//     groups.  Building the operand costs (128 + 32(NB-1))·32 instead of NB·128·32
//     shared-memory writes;
//   * the strip is built from a 1-D segment of one image column (staged once).
// B (the k filters) is split into tf32 hi/lo parts and packed into the UMMA
// core-matrix layout once per product by tc_pack_b; the main kernel streams its
// chunks into shared memory with bulk async copies (TMA engine, mbarrier tx count).
// One thread issues tcgen05.mma (kind::tf32, M = 128, N = 32/64, fp32 accumulator in
// TMEM): D += A_hi·B_hi + A_hi·B_lo + A_lo·B_hi.  Two pipeline stages: the builders
// fill stage s^1 while the tensor core consumes stage s; tcgen05.commit arrives on
// the stage's mbarrier when its MMAs have read shared memory.  The epilogue reads the
// accumulator with tcgen05.ld (32x32b: warp w owns TMEM lanes 32w..32w+31 = rows).
// Large reductions are split over CTAs along (d_y, d_x-chunks); partials are summed
// deterministically by reduce_splits_kernel (direct.cu layout).
#include "common.h"
#include "kernels.h"

namespace ssa {

namespace tc {

constexpr int kM = 128;          // UMMA M (one accumulator row per TMEM lane)
constexpr int kKB = 32;          // d_x per k-block (4 UMMA k-steps of 8 tf32)
constexpr int kBuilders = 256;   // warps 0-7 build the A strips; warp 8 issues TMA + MMA
constexpr int kThreads = kBuilders + 32;
constexpr int kSeg = 256;        // staged image segment per chunk (>= strip rows + 32)

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ uint32_t tf32_rna(float v) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(v));
    return r;
}

// UMMA shared-memory descriptor, K-major, 128-byte swizzle: one row of an operand
// tile is 32 tf32 (= one k-block, 128 B); 8 rows form a 1024-B swizzle atom in which
// the 16-B chunk c of row r sits at chunk position c ^ r.  SBO = 1024 (atom stride
// along M/N); LBO is unused for swizzled K-major layouts (encoded 1).  A k-step of 8
// tf32 inside the atom advances the start address by 32 B (the XOR is applied to the
// absolute address bits, so atoms must be 1024-B aligned).
__device__ __forceinline__ uint64_t make_desc(uint32_t addr) {
    uint64_t d = 0;
    d |= (uint64_t)((addr >> 4) & 0x3FFF);
    d |= (uint64_t)1 << 16;                 // LBO (unused)
    d |= (uint64_t)(1024 >> 4) << 32;       // SBO
    d |= (uint64_t)1 << 46;                 // descriptor version (sm_100)
    d |= (uint64_t)2 << 61;                 // SWIZZLE_128B
    return d;
}
// byte offset of the 16-B chunk c (0..7) of row i inside a swizzled K-major tile
__host__ __device__ __forceinline__ uint32_t sw128_off(int i, int c) {
    return (uint32_t)((i >> 3) * 1024 + (i & 7) * 128 + ((c ^ (i & 7)) << 4));
}

// Instruction descriptor, kind::tf32: D fp32, A/B tf32, both K-major, M x N.
__host__ __device__ constexpr uint32_t make_idesc(int M, int N) {
    return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    uint32_t done = 0;
    do {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(bar), "r"(parity)
            : "memory");
    } while (!done);
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void *src, uint32_t bytes, uint32_t bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(dst), "l"(src), "r"(bytes), "r"(bar)
                 : "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                         uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}"
        ::"r"(tmem_d), "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}
__device__ __forceinline__ void mma_commit(uint32_t bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
                 : "memory");
}

// 32 consecutive fp32 accumulator columns of this thread's TMEM lane
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float *v) {
    uint32_t r[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

}  // namespace tc

// ---------------------------------------------------------------------------
// B packing: in[d, j] (compact, column-major, ld ldi; imap: box -> compact or -1)
// -> Bpk[dy][kb][h] = an N x 32 swizzled K-major tile (h = tf32 hi / lo; row n = filter,
// 16-B chunk c = d_x 4c..4c+3 at sw128_off(n, c)), zero padded to nkb_pad k-blocks per
// d_y and N columns.  One k-block is 2·N·128 bytes.
// ---------------------------------------------------------------------------
template <int N>
__global__ void tc_pack_b_kernel(const float *__restrict__ in, int64_t ldi, const int *__restrict__ imap, int bx,
                                 int by, int k, int j0, int nkb_pad, float *__restrict__ bpk) {
    const int64_t total = (int64_t)by * nkb_pad * N * tc::kKB;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int kk = (int)(t % tc::kKB);
        const int64_t r = t / tc::kKB;
        const int n = (int)(r % N);
        const int64_t blk = r / N;                 // dy * nkb_pad + kb
        const int kb = (int)(blk % nkb_pad), dy = (int)(blk / nkb_pad);
        const int dx = kb * tc::kKB + kk;
        float v = 0.f;
        if (dx < bx && n + j0 < k) {
            const int64_t box = dx + (int64_t)bx * dy;
            const int64_t ci = imap ? (int64_t)imap[box] : box;
            if (ci >= 0) v = in[ci + ldi * (int64_t)(n + j0)];
        }
        const float hi = __uint_as_float(tc::tf32_rna(v));
        const float lo = v - hi;
        const int c = kk >> 2, q = kk & 3;
        const int64_t off = tc::sw128_off(n, c) / 4 + q;
        float *base = bpk + blk * (2 * N * tc::kKB);
        base[off] = hi;
        base[N * tc::kKB + off] = lo;
    }
}

// ---------------------------------------------------------------------------
// Main kernel.  grid.x = M-tiles (ceil(ox/128) per output column, times oy),
// grid.y = reduction splits (nsy along d_y times nsx along d_x chunks).
// Warp roles: warps 0-7 stage the image segment and build the hi/lo strip of
// each chunk; warp 8 (one lane) streams the packed B chunk with a bulk async
// copy and issues the MMAs.  Per stage s: full[s] (B landed, tx count),
// built[s] (8 builder-warp arrivals), empty[s] (tcgen05.commit: the MMAs that
// read stage s have completed).
// ---------------------------------------------------------------------------
struct TcArgs {
    const float *x; int64_t ldx; int nx;
    int ox, oy;                   // output box
    int bx, by;                   // reduction (input) box
    int nkb_pad;                  // packed k-blocks per d_y (multiple of NB)
    const float *bpk;             // packed B
    int k, j0;                    // columns j0 .. j0+N-1 of the k filters
    float *out; int64_t ldo; const int *omap;
    float *ws; int nsplit, nsx, dy_split, cx_split;
};

template <int N, int NB>
struct TcCfg {
    static constexpr int R = tc::kM + tc::kKB * (NB - 1);          // strip rows
    static constexpr uint32_t strip_bytes = R * 128;               // one of hi / lo
    static constexpr uint32_t bblock = 2 * N * 128;                // one packed k-block (hi + lo)
    static constexpr uint32_t bbytes = NB * bblock;
    static constexpr uint32_t stage = 2 * strip_bytes + bbytes;
    static constexpr size_t smem = 2 * (size_t)stage + 2 * tc::kSeg * sizeof(float) + 128;
    static_assert(R + tc::kKB <= tc::kSeg, "segment too short for the strip");
    static_assert(smem <= 227 * 1024, "shared memory budget");
};

template <int N, int NB>
__global__ void __launch_bounds__(tc::kThreads, 1) hankel_tc_kernel(TcArgs a) {
    using namespace tc;
    using C = TcCfg<N, NB>;
    constexpr int R = C::R;
    constexpr int kChunkDx = kKB * NB;
    extern __shared__ __align__(1024) unsigned char smem[];
    unsigned char *stage0 = smem;
    float *segs = reinterpret_cast<float *>(smem + 2 * C::stage);      // [2][kSeg]
    uint64_t *bars = reinterpret_cast<uint64_t *>(segs + 2 * kSeg);      // full[2], built[2], empty[2]
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bars + 6);
    const uint32_t bar0 = smem_u32(bars);
    auto full_bar = [&](int s) { return bar0 + 8u * s; };
    auto built_bar = [&](int s) { return bar0 + 16u + 8u * s; };
    auto empty_bar = [&](int s) { return bar0 + 32u + 8u * s; };

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int ntx = (a.ox + kM - 1) / kM;
    const int px0 = (blockIdx.x % ntx) * kM;
    const int py = blockIdx.x / ntx;
    const int split = blockIdx.y;
    const int zx = split % a.nsx, zy = split / a.nsx;
    const int dy_lo = zy * a.dy_split, dy_hi = min(a.by, dy_lo + a.dy_split);
    const int ncx_all = a.nkb_pad / NB;
    const int cx_lo = zx * a.cx_split, cx_hi = min(ncx_all, cx_lo + a.cx_split);
    const int ncx = cx_hi - cx_lo;
    const int n_it = (dy_hi > dy_lo && ncx > 0) ? (dy_hi - dy_lo) * ncx : 0;

    if (tid == 0) {
        for (int s = 0; s < 2; ++s) {
            mbar_init(full_bar(s), 1);
            mbar_init(built_bar(s), kBuilders / 32);
            mbar_init(empty_bar(s), 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    constexpr uint32_t kCols = N <= 32 ? 64 : 128;   // two accumulators (chunk parity)
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "n"(kCols)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    float racc[N];   // warps 0-3: running sum of the drained chunk accumulators (row = TMEM lane)
#pragma unroll
    for (int j = 0; j < N; ++j) racc[j] = 0.f;
    auto drain = [&](int buf) {
        tc_fence_after();
#pragma unroll
        for (int c0 = 0; c0 < N; c0 += 32) {
            float v[32];
            tmem_ld32(tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)(buf * N + c0), v);
#pragma unroll
            for (int j = 0; j < 32; ++j) racc[c0 + j] += v[j];
        }
        tc_fence_before();
    };
    if (warp == kBuilders / 32) {
        // ================= TMA + MMA issuer (one lane) =================
        if (lane == 0) {
            constexpr uint32_t idesc = make_idesc(kM, N);
            for (int it = 0; it < n_it; ++it) {
                const int s = it & 1;
                const int dy = dy_lo + it / ncx, cx = cx_lo + it % ncx;
                const uint32_t st_u = smem_u32(stage0 + s * C::stage);
                const uint32_t dacc = tmem + s * N;   // accumulator of this chunk (drained by warps 0-3)
                if (it >= 2) mbar_wait(empty_bar(s), ((it - 2) >> 1) & 1);   // B buffer of stage s free
                const float *src = a.bpk + ((int64_t)dy * a.nkb_pad + (int64_t)cx * NB) * (2 * N * kKB);
                mbar_expect_tx(full_bar(s), C::bbytes);
                bulk_g2s(st_u + 2 * C::strip_bytes, src, C::bbytes, full_bar(s));
                mbar_wait(built_bar(s), (it >> 1) & 1);
                mbar_wait(full_bar(s), (it >> 1) & 1);
                tc_fence_after();
#pragma unroll
                for (int b = 0; b < NB; ++b) {
#pragma unroll
                    for (int ks = 0; ks < kKB / 8; ++ks) {
                        // k-block b of the chunk = strip rows [32b, 32b + 128) = 4 atoms further
                        const uint32_t a_hi = st_u + b * 4096 + ks * 32;
                        const uint32_t b_hi = st_u + 2 * C::strip_bytes + b * C::bblock + ks * 32;
                        const uint64_t dAh = make_desc(a_hi);
                        const uint64_t dAl = make_desc(a_hi + C::strip_bytes);
                        const uint64_t dBh = make_desc(b_hi);
                        const uint64_t dBl = make_desc(b_hi + N * 128);
                        const uint32_t acc0 = (b > 0 || ks > 0) ? 1u : 0u;   // fresh accumulator per chunk
                        mma_tf32(dacc, dAh, dBl, idesc, acc0);
                        mma_tf32(dacc, dAl, dBh, idesc, 1u);
                        mma_tf32(dacc, dAh, dBh, idesc, 1u);
                    }
                }
                mma_commit(empty_bar(s));
            }
        }
        __syncwarp();
    } else {
        // ================= strip builders (warps 0-7) =================
        const float *xcol_base = a.x + px0;
        // image segment of column p_y + d_y from row p_x0 + d_x0 (zero past the edge), one
        // element per builder thread, prefetched one chunk ahead into a register
        auto seg_load = [&](int it2) -> float {
            const int dy2 = dy_lo + it2 / ncx, dx2 = (cx_lo + it2 % ncx) * kChunkDx;
            return (tid < a.nx - (px0 + dx2)) ? xcol_base[a.ldx * (int64_t)(py + dy2) + dx2 + tid] : 0.f;
        };
        float pre = n_it > 0 ? seg_load(0) : 0.f;
        for (int it = 0; it < n_it; ++it) {
            const int s = it & 1;
            unsigned char *st = stage0 + s * C::stage;
            float *seg = segs + s * kSeg;
            seg[tid] = pre;
            asm volatile("bar.sync 1, %0;" ::"n"(kBuilders) : "memory");   // builders only
            if (it + 1 < n_it) pre = seg_load(it + 1);
            // the strip of stage s is free once the MMAs of chunk it-2 have completed
            if (it >= 2) {
                mbar_wait(empty_bar(s), ((it - 2) >> 1) & 1);
                // drain chunk it-2's accumulator before the MMAs of chunk it overwrite it: the
                // tensor core accumulates with truncation, so partial sums are kept short
                // (NB·32 terms) and summed here in fp32 with round-to-nearest
                if (warp < 4) drain(s);
            }
            // strip S[i, jj] = seg[i + jj] -> hi / lo swizzled K-major tiles (row i, chunk jj/4)
            for (int item = tid; item < R * 8; item += kBuilders) {
                const int i = item % R, c = item / R;
                const float v0 = seg[i + 4 * c], v1 = seg[i + 4 * c + 1], v2 = seg[i + 4 * c + 2],
                            v3 = seg[i + 4 * c + 3];
                const uint32_t h0 = tf32_rna(v0), h1 = tf32_rna(v1), h2 = tf32_rna(v2), h3 = tf32_rna(v3);
                const uint32_t off = sw128_off(i, c);
                *reinterpret_cast<uint4 *>(st + off) = make_uint4(h0, h1, h2, h3);
                *reinterpret_cast<float4 *>(st + C::strip_bytes + off) =
                    make_float4(v0 - __uint_as_float(h0), v1 - __uint_as_float(h1), v2 - __uint_as_float(h2),
                                v3 - __uint_as_float(h3));
            }
            fence_proxy_async();
            __syncwarp();
            if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(built_bar(s)) : "memory");
        }
    }
    // ---- epilogue: drain the last (up to two) chunks, then rows -> output / split partials
    if (warp < 4) {
        for (int it = (n_it >= 2 ? n_it - 2 : 0); it < n_it; ++it) {
            mbar_wait(empty_bar(it & 1), (it >> 1) & 1);
            drain(it & 1);
        }
        const int m = warp * 32 + lane;
        const int px = px0 + m;
        const int64_t nbox = (int64_t)a.ox * a.oy;
        const int64_t pidx = px + (int64_t)a.ox * py;
        if (px < a.ox) {
            if (a.nsplit == 1) {
                const int64_t oi = a.omap ? (int64_t)a.omap[pidx] : pidx;
                if (oi >= 0)
#pragma unroll
                    for (int j = 0; j < N; ++j) {
                        const int jj = a.j0 + j;
                        if (jj < a.k) a.out[oi + a.ldo * (int64_t)jj] = racc[j];
                    }
            } else {
#pragma unroll
                for (int j = 0; j < N; ++j)
                    if (a.j0 + j < a.k) a.ws[((int64_t)split * N + j) * nbox + pidx] = racc[j];
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(kCols) : "memory");
}

// out[omap(p), j] = Σ_s ws[s][j][p]  (fixed summation order: deterministic)
__global__ void tc_reduce_kernel(const float *__restrict__ ws, int nsplit, int N, int64_t nbox, int kc,
                                 const int *__restrict__ omap, float *__restrict__ out, int64_t ldo) {
    const int64_t n = nbox * kc;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t p = t % nbox, j = t / nbox;
        const int64_t oi = omap ? (int64_t)omap[p] : p;
        if (oi < 0) continue;
        float s = 0.f;
        for (int q = 0; q < nsplit; ++q) s += ws[((int64_t)q * N + j) * nbox + p];
        out[oi + ldo * j] = s;
    }
}

static void reduce_splits_tc(const float *ws, int nsplit, int N, int64_t nbox, int kc, const int *omap, float *out,
                             int64_t ldo, cudaStream_t st) {
    const int64_t n = nbox * kc;
    tc_reduce_kernel<<<(unsigned)std::min<int64_t>(cdiv(n, 256), 8 * num_sms()), 256, 0, st>>>(ws, nsplit, N, nbox,
                                                                                              kc, omap, out, ldo);
    after_launch("tc_reduce");
}

bool tc_corr_supported(int ox, int oy, int bx, int by, int k) {
    (void)oy; (void)by; (void)k;
    return ox >= 96 && bx >= 32;
}

// k-blocks per chunk: 4 for long reductions, 2 when the reduction box is short (less padding)
static int tc_nb(int N, int bx) { return (N > 32 || cdiv(bx, tc::kKB) <= 2) ? 2 : 4; }

size_t tc_pack_bytes(int bx, int by, int k) {
    const int N = k <= 32 ? 32 : 64;
    const int64_t nkb_pad = rup(cdiv(bx, tc::kKB), tc_nb(N, bx));
    return sizeof(float) * (size_t)by * nkb_pad * 2 * N * tc::kKB;
}

template <int N, int NB>
static void tc_run(const TcCorrParams &P, int j0, cudaStream_t st) {
    const int nkb = (int)cdiv(P.bx, tc::kKB);
    const int nkb_pad = (int)rup(nkb, NB);
    const int64_t total = (int64_t)P.by * nkb_pad * N * tc::kKB;
    SSA_REQUIRE(sizeof(float) * (size_t)total * 2 <= P.bpk_bytes, SSA_ERR_ARG, "tc: packing buffer too small");
    tc_pack_b_kernel<N><<<(unsigned)std::min<int64_t>(cdiv(total, 256), 16 * num_sms()), 256, 0, st>>>(
        P.in, P.ldi, P.imap, P.bx, P.by, P.k, j0, nkb_pad, P.bpk);
    after_launch("tc_pack_b");

    TcArgs a{};
    a.x = P.x; a.ldx = P.ldx; a.nx = P.nx;
    a.ox = P.ox; a.oy = P.oy; a.bx = P.bx; a.by = P.by;
    a.nkb_pad = nkb_pad; a.bpk = P.bpk; a.k = P.k; a.j0 = j0;
    a.out = P.out; a.ldo = P.ldo; a.omap = P.omap;
    // split the reduction (d_y first, then d_x chunks) until ~one wave of CTAs
    const int64_t tiles = cdiv(P.ox, tc::kM) * P.oy;
    const int ncx_all = nkb_pad / NB;
    const int64_t nbox = (int64_t)P.ox * P.oy;
    const int64_t max_ws = std::max<int64_t>(1, (int64_t)(P.ws_bytes / ((size_t)N * nbox * sizeof(float))));
    int64_t want = std::max<int64_t>(1, num_sms() / tiles);
    want = std::min(want, max_ws);
    int64_t nsy = std::min<int64_t>(want, P.by);
    a.dy_split = (int)cdiv(P.by, nsy);
    nsy = cdiv(P.by, a.dy_split);
    int64_t nsx = std::max<int64_t>(1, std::min<int64_t>(want / nsy, ncx_all));
    a.cx_split = (int)cdiv(ncx_all, nsx);
    nsx = cdiv(ncx_all, a.cx_split);
    a.nsx = (int)nsx;
    a.nsplit = (int)(nsx * nsy);
    a.ws = P.ws;
    const size_t smem = TcCfg<N, NB>::smem;
    SSA_CUDA(cudaFuncSetAttribute(hankel_tc_kernel<N, NB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    hankel_tc_kernel<N, NB><<<dim3((unsigned)tiles, (unsigned)a.nsplit), tc::kThreads, smem, st>>>(a);
    after_launch("hankel_tc");
    if (a.nsplit > 1) {
        const int kc = std::min(N, P.k - j0);
        reduce_splits_tc(P.ws, a.nsplit, N, nbox, kc, P.omap, P.out + P.ldo * j0, P.ldo, st);
    }
}

void tc_corr(const TcCorrParams &P, cudaStream_t st) {
    if (P.k <= 0 || P.ox <= 0 || P.oy <= 0) return;
    for (int j0 = 0; j0 < P.k; j0 += 64) {
        if (P.k - j0 > 32) tc_run<64, 2>(P, j0, st);
        else if (tc_nb(32, P.bx) == 4) tc_run<32, 4>(P, j0, st);
        else tc_run<32, 2>(P, j0, st);
    }
}

}  // namespace ssa
