// Tensor-core (tcgen05 kind::tf32, 3xTF32) Gram of tall-skinny fp32 blocks for the
// block Lanczos solver (CGS / CholeskyQR Grams against the K-side
// basis, the largest HBM streams of the decomposition after the products):
//
//     G (n1 x n2, fp64) = Aᵀ B,   A: M x n1, B: M x n2, column-major, M ≫ n1, n2.
//
// The reduction runs over the M rows, which are contiguous in memory, so both UMMA
// operands are K-major straight from TMA: a 32-row chunk of 128 columns of A is one
// 128-B swizzled box [128 cols][32 rows] (A_op: M = columns of A, K = rows), a chunk of
// B likewise [N cols][32 rows] (B_op: N = columns of B).  Each CTA walks a contiguous
// range of chunks (one CTA per SM); per chunk:
//
//   TMA (warp 0) -> converter warps 2-7 split the raw fp32 tiles in place into
//   hi = rna_tf32(x) and lo = x − hi (same swizzled offsets) -> MMA thread (warp 1):
//   for each k-step kk (8 rows) and M-tile: D[kk] = A_lo·B_hi; D[kk] += A_hi·B_lo;
//   D[kk] += A_hi·B_hi (the large term last: one truncating accumulation at full
//   magnitude per 8-row partial) -> warps 8-15 drain the 4 k-step accumulators of the
//   chunk (tcgen05.ld), sum them in fp32 and fold them into compensated fp32 sums.
//
// TMEM holds two chunks of accumulators (ping-pong), so the tensor core works on chunk
// c+1 while chunk c drains.  Converters (warps 2-7) and drainers (warps 8-15) are separate
// warps so the split of chunk c+2, the MMAs of c+1 and the drain of c overlap.  Per-CTA fp64 partials are summed by gram_reduce_kernel in a
// fixed order (deterministic).  Accuracy: 3xTF32 products (~2^-21 relative per term)
// and one fp32 truncation per 8-row partial, comparable to the fp32 FFMA Gram.
#include <type_traits>
#include <map>
#include <tuple>

#include "common.h"
#include "kernels.h"
#include "tc_common.h"

namespace ssa {

namespace tallg {
constexpr int R = 32;                 // rows per chunk (128 B per column: one swizzled row)
constexpr int NTHR = 512;            // warps 0 TMA, 1 MMA, 2-7 convert, 8-15 drain

}  // namespace tallg

// ---------------------------------------------------------------------------
// Gram v3 (default): A operand in tensor memory.  Thin-N MMAs (N = k <= 64) with both operands in
// shared memory were bound by the shared-memory port and the chunk pipeline, not the tensor pipe:
// per 8-row k-step the three 3xTF32 MMAs read A three times plus B, and the in-smem hi/lo split
// read and wrote every element once more (v1 timeline: ~1 µs per 16 KB chunk with the TMA idle).
// Here a stage is RC 32-row sub-chunks; converter warps 4-7 (one per TMEM lane quarter) read a
// landed raw A row (one A column = one TMEM lane), split it and tcgen05.st hi / lo into TMEM (the
// A-from-TMEM `.kind::tf32` MMA: row m -> lane m, k -> column); then warps 2-7 split the thin B tile
// into shared memory, and the raw slot is released at once (the ring of raw slots takes the rest
// of shared memory).  Per accumulator (KG k-steps) the small terms A_lo·B_hi, A_hi·B_lo are
// accumulated first and the exact A_hi·B_hi products last: each truncating accumulation at full
// magnitude adds one large term.  TMEM: accumulators in columns [0, 256), A hi | lo buffers in
// [256, 512).
// ---------------------------------------------------------------------------
namespace tallg3 {
constexpr int MAXR = 24;
constexpr int SMEM = 226 * 1024;        // 227 KB opt-in − 1 KB reserved per CTA
template <int NM, int NN, int BA, int RC, int KG>
struct Cfg {
    static constexpr int OPB = 2;                           // operand buffers (TMEM A + shared B)
    static constexpr int KS = 4 * RC;                       // 8-row k-steps per stage
    static constexpr int KA = KS / KG;                      // accumulators per M-tile per stage
    static constexpr int a_raw = NM * BA * 128;             // A bytes per 32-row sub-chunk
    static constexpr int b_raw = NN * 128;
    static constexpr int bop = RC * 2 * b_raw;              // B [sub-chunk][hi | lo]
    static constexpr int acols = 64 * RC;                   // TMEM columns of one M-tile's A (hi | lo)
    static constexpr int off_raw = OPB * bop;
    static constexpr int off_bar = SMEM - 2048;             // 1 KB barriers + 1 KB alignment slack
    static constexpr int ring = off_bar - off_raw;
    static constexpr int acc_cols = NM * KA * NN;
    static constexpr int ACCB = 256 / acc_cols >= 4 ? 4 : 256 / acc_cols;
    static_assert(KS % KG == 0, "KG must divide the k-steps of a stage");
    static_assert(ACCB >= 2, "at least two accumulator buffers");
    static_assert(OPB * NM * acols <= 256, "A buffers exceed TMEM columns [256, 512)");
};
}  // namespace tallg3

template <int NM, int NN, int BA, int RC, int KG>
__global__ void __launch_bounds__(tallg::NTHR, 1)
gram_tc3_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, int64_t M,
                int n1, int n2, int b_col, double *__restrict__ partials, int per) {
    using namespace tc;
    using C = tallg3::Cfg<NM, NN, BA, RC, KG>;
    constexpr int KA = C::KA, OPB = C::OPB, AB = C::ACCB;
    extern __shared__ unsigned char smem_raw[];
    unsigned char *smem = smem_align1024(smem_raw);
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem + C::off_bar);
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bars + 64);
    const uint32_t bar0 = smem_u32(bars);
    auto full = [&](int r) { return bar0 + 8u * r; };             // raw stage landed        [24]
    auto rawe = [&](int r) { return bar0 + 8u * (24 + r); };      // raw slot consumed       [24]
    auto conv = [&](int o) { return bar0 + 8u * (48 + o); };      // operands split          [2]
    auto ope = [&](int o) { return bar0 + 8u * (52 + o); };       // operand MMAs done       [2]
    auto accf = [&](int b) { return bar0 + 8u * (56 + b); };      // accumulators ready      [4]
    auto acce = [&](int b) { return bar0 + 8u * (60 + b); };      // accumulators drained    [4]

    // B inside this CTA's A boxes (b_col = global A column where B starts, a multiple of 8 so that the
    // 128-B swizzle phase matches): the thin B tile is read from the A tile, no second TMA stream
    // (the projection Gram [Q W]ᵀW of the K side read W twice: 4.2 TB/s of traffic, 2.8 TB/s useful)
    const int col0_ = (int)blockIdx.y * NM * 128;
    const int boff = (b_col >= col0_ && b_col + NN <= col0_ + NM * BA) ? b_col - col0_ : -1;
    const bool self_b = boff >= 0;
    const int unit = C::a_raw + (self_b ? 0 : C::b_raw);          // raw bytes per sub-chunk
    const int raw_bytes = RC * unit;
    const int RS = min(tallg3::MAXR, C::ring / raw_bytes);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    // chunks interleaved over the CTAs (chunk = blockIdx.x + i·gridDim.x): the grid then streams one
    // contiguous run of ~148·32·RC rows of every column at a time; with a contiguous chunk range per
    // CTA the DRAM saw (CTAs x columns) separate 128-B streams (c5 K side: 1.8-2.8 TB/s, ncu)
    const int64_t nchunks = (M + 32 * RC - 1) / (32 * RC);
    const int nmy = (int)max((int64_t)0, (nchunks - (int64_t)blockIdx.x + gridDim.x - 1) / gridDim.x);
    const int col0 = (int)blockIdx.y * NM * 128;

    if (tid == 0) {
        for (int r = 0; r < RS; ++r) {
            mbar_init(full(r), 1);
            mbar_init(rawe(r), 6);
        }
        for (int o = 0; o < OPB; ++o) {
            mbar_init(conv(o), 6);
            mbar_init(ope(o), 1);
        }
        for (int b = 0; b < AB; ++b) {
            mbar_init(accf(b), 1);
            mbar_init(acce(b), 8);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "n"(512)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const uint32_t sm_u = smem_u32(smem);
    auto b_hi = [&](int o, int rc) { return sm_u + (uint32_t)(o * C::bop + rc * 2 * C::b_raw); };
    auto a_col = [&](int o, int mt) { return (uint32_t)(256 + (o * NM + mt) * C::acols); };   // hi; lo at +32·RC

    if (warp == 0) {
        if (lane == 0) {
            // ---------------- TMA producer: raw ring ----------------
            for (int i = 0; i < nmy; ++i) {
                const int r = i % RS;
                if (i >= RS) mbar_wait(rawe(r), ((i / RS) - 1) & 1);
                const uint32_t dst = sm_u + (uint32_t)(C::off_raw + r * raw_bytes);
                mbar_expect_tx(full(r), raw_bytes);
#pragma unroll
                for (int rc = 0; rc < RC; ++rc) {
                    const int r0 = (int)(((int64_t)blockIdx.x + (int64_t)i * gridDim.x) * 32 * RC + 32 * rc);
#pragma unroll
                    for (int mt = 0; mt < NM; ++mt)
                        tma_load_2d_true(dst + rc * unit + mt * BA * 128, &tmA, r0, col0 + 128 * mt, full(r));
                    if (!self_b) tma_load_2d_true(dst + rc * unit + C::a_raw, &tmB, r0, 0, full(r));
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            // ---------------- MMA issuer ----------------
            constexpr uint32_t idesc = make_idesc(128, NN);
            // accumulators live for `per` consecutive stages (one drain per period: the fp32 tensor-core
            // accumulation then spans per·32·RC rows before the Kahan sums)
            for (int i = 0; i < nmy; ++i) {
                const int pi = i / per, sp = i - pi * per;
                const int o = i % OPB, b = pi % AB;
                mbar_wait(conv(o), (i / OPB) & 1);
                if (sp == 0 && pi >= AB) mbar_wait(acce(b), ((pi / AB) - 1) & 1);
                tc_fence_after();
                const uint32_t dbase = tmem + (uint32_t)(b * C::acc_cols);
                const uint64_t bh0 = make_desc(b_hi(o, 0));
                {
                constexpr uint64_t b_lo_step = (uint64_t)(C::b_raw >> 4), rc_step = (uint64_t)((2 * C::b_raw) >> 4);
#pragma unroll
                for (int g = 0; g < KA; ++g) {
#pragma unroll
                    for (int mt = 0; mt < NM; ++mt) {
                        const uint32_t d = dbase + (uint32_t)((mt * KA + g) * NN);
                        const uint32_t ah = tmem + a_col(o, mt), al = ah + 32 * RC;
#pragma unroll
                        for (int q = 0; q < KG; ++q) {
                            const int kk = g * KG + q;
                            const uint64_t bh = bh0 + (uint64_t)(kk >> 2) * rc_step + (uint64_t)(2 * (kk & 3));
                            mma_tf32_ts(d, al + 8 * kk, bh, idesc, (q || sp) ? 1u : 0u);
                            mma_tf32_ts(d, ah + 8 * kk, bh + b_lo_step, idesc, 1u);
                        }
#pragma unroll
                        for (int q = 0; q < KG; ++q) {
                            const int kk = g * KG + q;
                            const uint64_t bh = bh0 + (uint64_t)(kk >> 2) * rc_step + (uint64_t)(2 * (kk & 3));
                            mma_tf32_ts(d, ah + 8 * kk, bh, idesc, 1u);
                        }
                    }
                }
                }
                mma_commit(ope(o));
                if (sp == per - 1 || i == nmy - 1) mma_commit(accf(b));
            }
        }
    } else if (warp < 8) {
        // ---------------- converters, warps 2-7 ----------------
        // warps 4-7 first move the A rows of their TMEM lane quarter (one A column per lane) into TMEM
        // as hi / lo; then all six warps split the thin B tile (or A's first NN rows) into shared memory
        const int q = warp & 3, m = 32 * q + lane;
        const bool a_warp = warp >= 4 && 32 * q < BA;
        const uint32_t lane_off = (uint32_t)(32 * q) << 16;
        const int ct = tid - 64;
        constexpr int nb4 = C::b_raw / 16;
        for (int i = 0; i < nmy; ++i) {
            const int r = i % RS, o = i % OPB;
            mbar_wait(full(r), (i / RS) & 1);
            if (i >= OPB) mbar_wait(ope(o), ((i / OPB) - 1) & 1);
            tc_fence_after();
            const unsigned char *rawp = smem + C::off_raw + (size_t)r * raw_bytes;
            if (a_warp) {
#pragma unroll
                for (int rc = 0; rc < RC; ++rc) {
#pragma unroll
                    for (int mt = 0; mt < NM; ++mt) {
                        const unsigned char *row = rawp + rc * unit + mt * BA * 128 + m * 128;
                        uint32_t hi[32], lo[32];
#pragma unroll
                        for (int c = 0; c < 8; ++c) {
                            const float4 x = *reinterpret_cast<const float4 *>(row + ((c ^ (m & 7)) << 4));
                            const float xs[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
                            for (int u = 0; u < 4; ++u) {
                                const uint32_t h = tf32_rna(xs[u]);
                                hi[4 * c + u] = h;
                                lo[4 * c + u] = __float_as_uint(xs[u] - __uint_as_float(h));
                            }
                        }
                        tmem_st32(tmem + lane_off + a_col(o, mt) + 32 * rc, hi);
                        tmem_st32(tmem + lane_off + a_col(o, mt) + 32 * RC + 32 * rc, lo);
                    }
                }
                tmem_wait_st();
            }
#pragma unroll
            for (int rc = 0; rc < RC; ++rc) {
                const float4 *src = reinterpret_cast<const float4 *>(rawp + rc * unit + (self_b ? boff * 128 : C::a_raw));
                float4 *dh = reinterpret_cast<float4 *>(smem + (size_t)o * C::bop + rc * 2 * C::b_raw);
#pragma unroll 2
                for (int e = ct; e < nb4; e += 192) {
                    const float4 x = src[e];
                    float4 hh, l;
                    hh.x = __uint_as_float(tf32_rna(x.x)); l.x = x.x - hh.x;
                    hh.y = __uint_as_float(tf32_rna(x.y)); l.y = x.y - hh.y;
                    hh.z = __uint_as_float(tf32_rna(x.z)); l.z = x.z - hh.z;
                    hh.w = __uint_as_float(tf32_rna(x.w)); l.w = x.w - hh.w;
                    dh[e] = hh;
                    dh[e + nb4] = l;
                }
            }
            fence_proxy_async();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) {
                asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(rawe(r)) : "memory");
                asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(conv(o)) : "memory");
            }
        }
    } else {
        // ---------------- drain (warps 8-15): KA accumulators summed in fp32, Kahan across stages ----------------
        constexpr int UNITS = NM * NN / 32;
        const int h = (warp - 8) >> 2;
        const int mt_u = (NM == 2) ? h : 0, n0_u = (NM == 2) ? 0 : 32 * h;
        const bool has_unit = h < UNITS;
        float ks[32], kc[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) { ks[j] = 0.f; kc[j] = 0.f; }
        const uint32_t lane_base = tmem + ((uint32_t)((warp & 3) * 32) << 16);
        const int nper = (nmy + per - 1) / per;
        for (int i = 0; i < nper; ++i) {
            const int b = i % AB;
            mbar_wait(accf(b), (i / AB) & 1);
            tc_fence_after();
            if (has_unit) {
#pragma unroll
                for (int hv = 0; hv < 2; ++hv) {
                    uint32_t rr[KA][16];
#pragma unroll
                    for (int g = 0; g < KA; ++g)
                        tmem_ld16_nowait(lane_base + (uint32_t)(b * C::acc_cols + (mt_u * KA + g) * NN + n0_u + 16 * hv), rr[g]);
                    tmem_wait_ld();
#pragma unroll
                    for (int j = 0; j < 16; ++j) {
                        float t = 0.f;
#pragma unroll
                        for (int g = 0; g < KA; ++g) t += __uint_as_float(rr[g][j]);
                        const int qq = 16 * hv + j;
                        const float y = t - kc[qq];
                        const float u = ks[qq] + y;
                        kc[qq] = (u - ks[qq]) - y;
                        ks[qq] = u;
                    }
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(acce(b)) : "memory");
        }
        if (has_unit) {
            const int nparts = gridDim.x;
            const int a = col0 + 128 * mt_u + (warp & 3) * 32 + lane;
            if (a < n1) {
                double *base = partials + ((int64_t)(a / 64) * nparts + blockIdx.x) * 4096 + (a % 64);
#pragma unroll
                for (int j = 0; j < 32; ++j)
                    if (n0_u + j < n2) base[64 * (n0_u + j)] = (double)ks[j] - (double)kc[j];
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(512) : "memory");
}

// ---------------------------------------------------------------------------
// Self Gram WᵀW (n <= 64 columns, the CholeskyQR Gram of the K-side blocks): hi and lo stacked on the
// M dimension.  With the truncating split h = x & ~0x1fff (exact tf32), l = x − h, the tensor core's
// own reading of the fp32 data as tf32 is h, so the data tile itself is the B operand (no split of B).
// One MMA per 8-row k-step, A = [h; l] (TMEM lanes 0..NC−1: h of column c, lanes NC..2NC−1: l of c):
//     D = [ hᵀh ; lᵀh ]   and   WᵀW = hᵀh + lᵀh + (lᵀh)ᵀ  (dropping lᵀl, as 3xTF32 does),
// combined by gram_reduce_stacked.  (The 3xTF32 form spent three 128-row MMAs per k-step on 64 useful
// rows and split every B element: ~2.6k cycles per 64-row stage, 1.9 TB/s on c5's K side, ncu.)
// Loads: TMA boxes of ROWS = 128 rows x NC columns, unswizzled (512 B per column: a probe streamed
// 128-B-wide boxes, the 128-B-swizzle limit, at 4.6 TB/s and >= 256-B-wide ones at 6.4 TB/s,
// scripts/probe_tma.py); warps 2-7 copy each landed stage into the canonical K-major 128-B-swizzled
// B tile (ROWS/32 sub-tiles of 32 rows), then warps 4-7 (one per TMEM lane quarter) read it back conflict-free and split A into
// TMEM (a separate 2-warp relayout stage was the bottleneck: 1.2 ms, ncu); warp 1 issues; warps 8-15 drain one accumulator per PAIR stages (64·PAIR rows:
// the accumulator read-back, 32 KB per drain, is the drain's cost) into Kahan-compensated fp32 sums.  Buffers: RS staging slots, OPB B tiles / TMEM A buffers, ACCB
// accumulators.
// ---------------------------------------------------------------------------
namespace tallgs {
constexpr int ACCB = 4, NTHR = 512;
constexpr int SMEM = 226 * 1024;
}  // namespace tallgs

template <int NC, int ROWS, int PAIR>
__global__ void __launch_bounds__(tallgs::NTHR, 1)
gram_self_kernel(const __grid_constant__ CUtensorMap tmA, int64_t M, double *__restrict__ partials) {
    using namespace tc;
    constexpr int STAGE = NC * ROWS * 4;              // bytes per stage (raw [c][ROWS] or B [ROWS/32][c][32])
    constexpr int OPB = 256 / ROWS < 4 ? 256 / ROWS : 4, AB = tallgs::ACCB;
    constexpr int RS = (128 * 1024) / STAGE < 8 ? (128 * 1024) / STAGE : 8;
    constexpr int NSUB = ROWS / 32;                   // 32-row sub-tiles per stage
    constexpr int CPC = ROWS / 4;                     // 16-B chunks per column and stage
    constexpr int SUB = NC * 128;                     // one 32-row sub-tile of B
    constexpr int off_b = RS * STAGE;
    constexpr int off_bar = off_b + OPB * STAGE;
    constexpr int NCONV = (2 * NC) / 32;              // converter warps (one per TMEM lane quarter)
    static_assert(off_bar + 1024 <= tallgs::SMEM - 1024, "shared memory budget");
    static_assert(AB * NC <= 256 && OPB * ROWS <= 256, "TMEM budget");
    extern __shared__ unsigned char smem_raw[];
    unsigned char *smem = smem_align1024(smem_raw);
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem + off_bar);
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bars + 64);
    const uint32_t bar0 = smem_u32(bars);
    auto full = [&](int r) { return bar0 + 8u * r; };             // raw stage landed       [8]
    auto rawe = [&](int r) { return bar0 + 8u * (8 + r); };       // raw stage copied       [8]
    auto bful = [&](int o) { return bar0 + 8u * (16 + o); };      // B tile o written       [4]
    auto conv = [&](int o) { return bar0 + 8u * (20 + o); };      // A buffer o split       [4]
    auto ope = [&](int o) { return bar0 + 8u * (24 + o); };       // MMAs of B / A o done   [4]
    auto accf = [&](int b) { return bar0 + 8u * (28 + b); };      // accumulator ready      [4]
    auto acce = [&](int b) { return bar0 + 8u * (32 + b); };      // accumulator drained    [4]

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int64_t nst = (M + ROWS - 1) / ROWS;
    const int nmy = (int)max((int64_t)0, (nst - (int64_t)blockIdx.x + gridDim.x - 1) / gridDim.x);

    if (tid == 0) {
        for (int r = 0; r < RS; ++r) {
            mbar_init(full(r), 1);
            mbar_init(rawe(r), 1);
        }
        for (int o = 0; o < OPB; ++o) {
            mbar_init(bful(o), 1);
            mbar_init(conv(o), NCONV);
            mbar_init(ope(o), 1);
        }
        for (int b = 0; b < AB; ++b) {
            mbar_init(accf(b), 1);
            mbar_init(acce(b), 8);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "n"(512)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const uint32_t sm_u = smem_u32(smem);
    auto a_col = [&](int o) { return (uint32_t)(256 + o * ROWS); };

    if (warp == 0) {
        if (lane == 0) {
            for (int i = 0; i < nmy; ++i) {
                const int r = i % RS;
                if (i >= RS) mbar_wait(rawe(r), ((i / RS) - 1) & 1);
                mbar_expect_tx(full(r), STAGE);
                const int r0 = (int)(((int64_t)blockIdx.x + (int64_t)i * gridDim.x) * ROWS);
                tma_load_2d_true(sm_u + r * STAGE, &tmA, r0, 0, full(r));
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            // accumulator g = i / PAIR collects PAIR stages (64·PAIR rows)
            constexpr uint32_t idesc = make_idesc(128, NC);
            for (int i = 0; i < nmy; ++i) {
                const int o = i % OPB, g = i / PAIR, b = g % AB, first = (i % PAIR) == 0;
                const bool last = (i % PAIR) == PAIR - 1 || i == nmy - 1;
                mbar_wait(bful(o), (i / OPB) & 1);
                mbar_wait(conv(o), (i / OPB) & 1);
                if (first && g >= AB) mbar_wait(acce(b), ((g / AB) - 1) & 1);
                tc_fence_after();
                const uint32_t d = tmem + (uint32_t)(b * NC), a = tmem + a_col(o);
#pragma unroll
                for (int rc = 0; rc < NSUB; ++rc) {
                    const uint64_t bd = make_desc(sm_u + off_b + o * STAGE + rc * SUB);
#pragma unroll
                    for (int q = 0; q < 4; ++q)
                        mma_tf32_ts(d, a + 32 * rc + 8 * q, bd + (uint64_t)(2 * q), idesc, (first && !(rc | q)) ? 0u : 1u);
                }
                mma_commit(ope(o));
                if (last) mma_commit(accf(b));
            }
        }
    } else if (warp < 8) {
        // warps 2-7: relayout raw [c][64 rows] (16 chunks of 16 B per column) -> B tile [rc][c][32 rows],
        // 128-B swizzle (all loads of a thread before its stores); named barrier; then warps 4-7 split
        // the A operand (lane m: column c = m mod NC, hi for m < NC, else lo) from the B tile into TMEM
        const int t = tid - 64;
        constexpr int PER = (NC * CPC + 191) / 192;
        const int q = warp & 3, m = 32 * q + lane, c = m % NC;
        const bool conv_warp = warp >= 4 && 32 * q < 2 * NC, lo_part = m >= NC;
        const uint32_t lane_off = (uint32_t)(32 * q) << 16;
        for (int i = 0; i < nmy; ++i) {
            const int r = i % RS, o = i % OPB;
            mbar_wait(full(r), (i / RS) & 1);
            if (i >= OPB) mbar_wait(ope(o), ((i / OPB) - 1) & 1);
            const float4 *src = reinterpret_cast<const float4 *>(smem + r * STAGE);
            unsigned char *dst = smem + off_b + o * STAGE;
            float4 x[PER];
#pragma unroll
            for (int k = 0; k < PER; ++k)
                if (t + 192 * k < NC * CPC) x[k] = src[t + 192 * k];
#pragma unroll
            for (int k = 0; k < PER; ++k) {
                const int e = t + 192 * k;
                if (e < NC * CPC) {
                    const int cc = e / CPC, j = e % CPC, rc = j >> 3, jj = j & 7;
                    *reinterpret_cast<float4 *>(dst + rc * SUB + cc * 128 + ((jj ^ (cc & 7)) << 4)) = x[k];
                }
            }
            fence_proxy_async();   // the MMAs read the tile through the async proxy
            asm volatile("bar.sync 1, 192;" ::: "memory");
            if (t == 0) {
                asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(rawe(r)) : "memory");
                asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bful(o)) : "memory");
            }
            if (conv_warp) {
                tc_fence_after();
                auto split = [&](auto lo_tag) {
#pragma unroll
                    for (int rc = 0; rc < NSUB; ++rc) {
                        const unsigned char *row = smem + off_b + o * STAGE + rc * SUB + c * 128;
                        uint32_t v[32];
#pragma unroll
                        for (int j = 0; j < 8; ++j) {
                            const float4 y = *reinterpret_cast<const float4 *>(row + ((j ^ (c & 7)) << 4));
                            const float ys[4] = {y.x, y.y, y.z, y.w};
#pragma unroll
                            for (int u = 0; u < 4; ++u) {
                                const uint32_t h = __float_as_uint(ys[u]) & 0xffffe000u;
                                v[4 * j + u] = decltype(lo_tag)::value ? __float_as_uint(ys[u] - __uint_as_float(h)) : h;
                            }
                        }
                        tmem_st32(tmem + lane_off + a_col(o) + 32 * rc, v);
                    }
                };
                if (lo_part) split(std::true_type{});
                else split(std::false_type{});
                tmem_wait_st();
                tc_fence_before();
                __syncwarp();
                if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(conv(o)) : "memory");
            }
        }
    } else if (warp >= 8) {
        // warp w: TMEM lanes 32·(w mod 4).., accumulator columns 32·((w − 8) / 4)..
        const int qd = warp & 3, h = (warp - 8) >> 2;
        const bool has = 32 * qd < 2 * NC && 32 * h < NC;
        float ks[32], kc[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) { ks[j] = 0.f; kc[j] = 0.f; }
        const uint32_t lane_base = tmem + ((uint32_t)(32 * qd) << 16) + (uint32_t)(32 * h);
        const int nacc = (nmy + PAIR - 1) / PAIR;
        for (int i = 0; i < nacc; ++i) {
            const int b = i % AB;
            mbar_wait(accf(b), (i / AB) & 1);
            tc_fence_after();
            float v[32];
            if (has) tmem_ld32(lane_base + (uint32_t)(b * NC), v);
            tc_fence_before();
            __syncwarp();
            if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(acce(b)) : "memory");
            if (has) {
#pragma unroll
                for (int j = 0; j < 32; ++j) {
                    const float y = v[j] - kc[j];
                    const float u = ks[j] + y;
                    kc[j] = (u - ks[j]) - y;
                    ks[j] = u;
                }
            }
        }
        if (has) {
            // partial rows a' = TMEM lane (0..2NC−1), columns b = 32h + j, 64 x 64 slabs as gram_reduce reads them
            const int a = 32 * qd + lane;
            double *base = partials + ((int64_t)(a / 64) * gridDim.x + blockIdx.x) * 4096 + (a % 64);
#pragma unroll
            for (int j = 0; j < 32; ++j) base[64 * (32 * h + j)] = (double)ks[j] - (double)kc[j];
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(512) : "memory");
}

// G (n x n) = S(a, b) + S(NC + a, b) + S(NC + b, a), S = the stacked partial sums [hᵀh; lᵀh] (2NC x NC)
__global__ void gram_reduce_stacked_kernel(const double *__restrict__ partials, int nparts, int nc, int n,
                                           double *__restrict__ G, int ldg) {
    const int e = (blockIdx.x * blockDim.x + threadIdx.x) / 32, lane = threadIdx.x % 32;
    if (e >= n * n) return;
    const int a = e % n, b = e / n;
    auto S = [&](int ap, int bp) {
        const double *base = partials + (int64_t)(ap / 64) * nparts * 4096 + (ap % 64) + 64 * bp;
        double s = 0.0;
        for (int q = lane; q < nparts; q += 32) s += base[(int64_t)q * 4096];
        return s;
    };
    double s = S(a, b) + (S(nc + a, b) + S(nc + b, a));
#pragma unroll
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) G[a + (int64_t)ldg * b] = s;
}

// ---------------------------------------------------------------------------
// Update v2 (default): Out = beta·Out + A·(alpha·C) with the A operand in tensor memory.  The
// contraction runs over A's columns, so an A row (one output row) is one TMEM lane: converter
// warps 4-7 read the landed raw tile [32 columns][128 rows] (plain TMA box, no swizzle: a warp
// reads 128 contiguous bytes per column), split it into tf32 hi / lo and tcgen05.st them as a
// K-major TMEM operand; the raw slot is released at once (ring of up to 12 raw tiles).  The
// pre-split coefficient tiles (B = (alpha·C)ᵀ chunk, K-major SW128 images) are bulk-copied from L2
// by warp 2 into OPB slots that the MMAs release.  Per (tile, chunk) one fresh accumulator: the
// small terms A_lo·B_hi, A_hi·B_lo of the 4 k-steps first, then the exact A_hi·B_hi products.
// Drain / epilogue: fp32 register sums across chunks; at the tile's end each drain warp stages its
// 32 x 32 piece in shared memory and one lane issues a tensor store of it (beta = 0) or an add-reduce
// at L2 (beta = 1: Out += A·C without reading Out into the SM).  The register read-modify-write with
// 32 scalar loads / stores per thread and tile (other beta) had put half of the kernel's instructions
// and its top stalls in the epilogue (c5 K side: 3.0 ms = 3.8 TB/s for Out −= A·C, ncu).
// ---------------------------------------------------------------------------
namespace tallu2 {
constexpr int ROWS = 128, KC = 64, OPB = 2, NBUF = 4, MAXR = 12, MAXB = 24, NTHR = 512;   // KC: A columns per item
constexpr int SMEM = 226 * 1024;
constexpr int BRES = 96 * 1024;      // coefficient tiles of all chunks kept resident up to this size
constexpr int BRING = 8;             // otherwise a ring of this many tiles, released by the MMAs
template <int NN>
struct Cfg {
    static constexpr int a_raw = ROWS * KC * 4;             // 32 KB
    static constexpr int b_bytes = 2 * NN * KC * 4;         // two packed 32-column chunks, each hi | lo
    static constexpr int off_bar = SMEM - 2048;
    static constexpr int off_stage = off_bar - 8 * 4096;    // epilogue staging: 32 x 32 fp32 per drain warp
    static_assert(NBUF * NN <= 256 && OPB * 2 * KC <= 256, "TMEM budget");
};
}  // namespace tallu2

template <int NN>
__global__ void __launch_bounds__(tallu2::NTHR, 1)
update_tc2_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmO, int omode, int64_t M,
                  int m, const float *__restrict__ Bpk, int n, double beta, float *Out, int64_t ldo) {
    using namespace tc;
    using Cf = tallu2::Cfg<NN>;
    constexpr int OPB = tallu2::OPB, NBUF = tallu2::NBUF, KC = tallu2::KC;
    extern __shared__ unsigned char smem_raw[];
    unsigned char *smem = smem_align1024(smem_raw);
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem + Cf::off_bar);
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bars + 96);   // after the 88 barriers
    const uint32_t bar0 = smem_u32(bars);
    auto fulla = [&](int r) { return bar0 + 8u * r; };            // raw A landed          [12]
    auto rawe = [&](int r) { return bar0 + 8u * (12 + r); };      // raw A converted       [12]
    auto conv = [&](int o) { return bar0 + 8u * (24 + o); };      // A in TMEM             [4]
    auto ope = [&](int o) { return bar0 + 8u * (28 + o); };       // MMAs of A buffer o done [4]
    auto accf = [&](int b) { return bar0 + 8u * (32 + b); };      // accumulator ready     [4]
    auto acce = [&](int b) { return bar0 + 8u * (36 + b); };      // accumulator drained   [4]
    auto fullb = [&](int q) { return bar0 + 8u * (40 + q); };     // coefficient slot landed [24]
    auto bemp = [&](int q) { return bar0 + 8u * (64 + q); };      // coefficient slot free   [24]

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int nchk = (m + KC - 1) / KC;
    // coefficient tiles: all nchk resident (loaded once, reused by every row tile) when they fit,
    // else a ring of BRING slots that runs ahead of the MMAs (a per-item reload from L2 tied to
    // the A buffers had put the L2 latency on the item cadence)
    const bool bres = nchk * Cf::b_bytes <= tallu2::BRES && nchk <= tallu2::MAXB;
    const int BS = bres ? nchk : max(2, min(tallu2::BRING, (Cf::off_stage - 3 * Cf::a_raw) / Cf::b_bytes));
    const int off_raw = BS * Cf::b_bytes;
    const int RS = min(tallu2::MAXR, (Cf::off_stage - off_raw) / Cf::a_raw);
    // tiles interleaved over the CTAs (tile = blockIdx.x + i·gridDim.x), as in the Gram: the grid
    // streams one contiguous run of rows of all m columns at a time (DRAM page locality)
    const int64_t ntiles = (M + tallu2::ROWS - 1) / tallu2::ROWS;
    const int64_t mytiles = max((int64_t)0, (ntiles - (int64_t)blockIdx.x + gridDim.x - 1) / gridDim.x);
    const int nitems = (int)(mytiles * nchk);

    if (tid == 0) {
        for (int r = 0; r < RS; ++r) {
            mbar_init(fulla(r), 1);
            mbar_init(rawe(r), 4);
        }
        for (int o = 0; o < OPB; ++o) {
            mbar_init(conv(o), 4);
            mbar_init(ope(o), 1);
        }
        for (int q = 0; q < BS; ++q) {
            mbar_init(fullb(q), 1);
            mbar_init(bemp(q), 1);
        }
        for (int b = 0; b < NBUF; ++b) {
            mbar_init(accf(b), 1);
            mbar_init(acce(b), 8);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
        if (omode) asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmO)) : "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "n"(512)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const uint32_t sm_u = smem_u32(smem);
    auto bslot = [&](int q) { return sm_u + (uint32_t)(q * Cf::b_bytes); };
    auto raw = [&](int r) { return sm_u + (uint32_t)(off_raw + r * Cf::a_raw); };
    auto a_col = [&](int o) { return (uint32_t)(256 + 2 * KC * o); };   // hi [KC] | lo [KC]

    if (warp == 0) {
        if (lane == 0) {
            for (int i = 0; i < nitems; ++i) {
                const int r = i % RS;
                if (i >= RS) mbar_wait(rawe(r), ((i / RS) - 1) & 1);
                const int64_t tile = (int64_t)blockIdx.x + (int64_t)(i / nchk) * gridDim.x;
                mbar_expect_tx(fulla(r), Cf::a_raw);
                tma_load_2d_true(raw(r), &tmA, (int)(tile * tallu2::ROWS), (i % nchk) * KC, fulla(r));
            }
        }
    } else if (warp == 2) {
        if (lane == 0) {
            if (bres) {
                for (int ch = 0; ch < nchk && nitems > 0; ++ch) {
                    mbar_expect_tx(fullb(ch), Cf::b_bytes);
                    bulk_g2s(bslot(ch), Bpk + (size_t)ch * (Cf::b_bytes / 4), Cf::b_bytes, fullb(ch));
                }
            } else {
                for (int i = 0; i < nitems; ++i) {
                    const int q = i % BS;
                    if (i >= BS) mbar_wait(bemp(q), ((i / BS) - 1) & 1);
                    mbar_expect_tx(fullb(q), Cf::b_bytes);
                    bulk_g2s(bslot(q), Bpk + (size_t)(i % nchk) * (Cf::b_bytes / 4), Cf::b_bytes, fullb(q));
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            constexpr uint32_t idesc = make_idesc(128, NN);
            for (int i = 0; i < nitems; ++i) {
                const int o = i % OPB, b = i % NBUF, q = bres ? i % nchk : i % BS;
                mbar_wait(conv(o), (i / OPB) & 1);
                mbar_wait(fullb(q), bres ? 0u : (uint32_t)((i / BS) & 1));
                if (i >= NBUF) mbar_wait(acce(b), ((i / NBUF) - 1) & 1);
                tc_fence_after();
                const uint32_t d = tmem + (uint32_t)(b * NN);
                const uint32_t ah = tmem + a_col(o), al = ah + KC;
                // B slot = two 32-column chunks [hi | lo] of NN x 32 each; k-step k: chunk k / 4, k % 4 within
                const uint64_t b0 = make_desc(bslot(q));
                constexpr uint64_t lo_step = (uint64_t)((NN * 32 * 4) >> 4), ch_step = 2 * lo_step;
                {
#pragma unroll
                for (int k = 0; k < KC / 8; ++k) {
                    const uint64_t bh = b0 + (uint64_t)(k >> 2) * ch_step + (uint64_t)(2 * (k & 3));
                    mma_tf32_ts(d, al + 8 * k, bh, idesc, k > 0 ? 1u : 0u);
                    mma_tf32_ts(d, ah + 8 * k, bh + lo_step, idesc, 1u);
                }
#pragma unroll
                for (int k = 0; k < KC / 8; ++k) {
                    const uint64_t bh = b0 + (uint64_t)(k >> 2) * ch_step + (uint64_t)(2 * (k & 3));
                    mma_tf32_ts(d, ah + 8 * k, bh, idesc, 1u);
                }
                }
                mma_commit(ope(o));
                mma_commit(accf(b));
                if (!bres) mma_commit(bemp(q));
            }
        }
    } else if (warp >= 4 && warp < 8) {
        // ---------------- converters: row r of the tile -> TMEM lane r (hi | lo) ----------------
        const int q = warp & 3, r_l = 32 * q + lane;
        const uint32_t lane_off = (uint32_t)(32 * q) << 16;
        for (int i = 0; i < nitems; ++i) {
            const int r = i % RS, o = i % OPB;
            mbar_wait(fulla(r), (i / RS) & 1);
            if (i >= OPB) mbar_wait(ope(o), ((i / OPB) - 1) & 1);
            tc_fence_after();
            const float *src = reinterpret_cast<const float *>(smem + off_raw + (size_t)r * Cf::a_raw) + r_l;
            {
#pragma unroll
            for (int hh = 0; hh < KC / 32; ++hh) {
                uint32_t hi[32], lo[32];
#pragma unroll
                for (int c = 0; c < 32; ++c) {
                    const float x = src[(32 * hh + c) * tallu2::ROWS];
                    const uint32_t h = tf32_rna(x);
                    hi[c] = h;
                    lo[c] = __float_as_uint(x - __uint_as_float(h));
                }
                tmem_st32(tmem + lane_off + a_col(o) + 32 * hh, hi);
                tmem_st32(tmem + lane_off + a_col(o) + KC + 32 * hh, lo);
            }
            tmem_wait_st();
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) {
                asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(rawe(r)) : "memory");
                asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(conv(o)) : "memory");
            }
        }
    } else if (warp >= 8) {
        // ---------------- drain + epilogue: warp w: rows 32·(w%4).., output columns 32·((w-8)/4).. ----------------
        const int h = (warp - 8) >> 2;
        const bool has = 32 * h < NN;
        float acc[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) acc[j] = 0.f;
        const uint32_t lane_base = tmem + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)(32 * h);
        const float fb = (float)beta;
        float old[32];
        float *stg = reinterpret_cast<float *>(smem + Cf::off_stage + (warp - 8) * 4096);   // [col][row], 32 x 32
        for (int i = 0; i < nitems; ++i) {
            const int b = i % NBUF;
            const int64_t row = ((int64_t)blockIdx.x + (int64_t)(i / nchk) * gridDim.x) * tallu2::ROWS + (warp & 3) * 32 + lane;
            if (i % nchk == 0 && !omode) {
                // the tile's old output values, loaded a whole tile ahead of the epilogue (their
                // latency used to stall the drain, and with it the MMAs, once per tile); in place
                // (Out = A) is safe: these rows are written only by this thread, at the tile's end
#pragma unroll
                for (int j = 0; j < 32; ++j) {
                    const int col = 32 * h + j;
                    old[j] = (has && row < M && beta != 0.0 && col < n) ? __ldcg(Out + row + ldo * (int64_t)col) : 0.f;
                }
            }
            mbar_wait(accf(b), (i / NBUF) & 1);
            tc_fence_after();
            if (has) {
                float v[32];
                tmem_ld32(lane_base + (uint32_t)(b * NN), v);
#pragma unroll
                for (int j = 0; j < 32; ++j) acc[j] += v[j];
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(acce(b)) : "memory");
            if (i % nchk == nchk - 1 && omode) {
                if (has) {
                    if (lane == 0) bulk_wait_read0();   // this warp's previous store has read the staging
                    __syncwarp();
#pragma unroll
                    for (int j = 0; j < 32; ++j) stg[32 * j + lane] = acc[j];
                    fence_proxy_async();
                    __syncwarp();
                    const int64_t row0 = row - lane;
                    if (lane == 0 && row0 < M) tma_store_2d(&tmO, smem_u32(stg), (int)row0, 32 * h, omode);
                }
#pragma unroll
                for (int j = 0; j < 32; ++j) acc[j] = 0.f;
            } else if (i % nchk == nchk - 1) {
                if (has && row < M) {
#pragma unroll
                    for (int j = 0; j < 32; ++j) {
                        const int col = 32 * h + j;
                        if (col < n) Out[row + ldo * (int64_t)col] = fmaf(fb, old[j], acc[j]);
                    }
                }
#pragma unroll
                for (int j = 0; j < 32; ++j) acc[j] = 0.f;
            }
        }
        if (omode && lane == 0) bulk_wait0();   // stores complete before the staging is released
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(512) : "memory");
}

// Streaming probe (measurement only, ssa_bench_tall which = 4): TMA loads of an M x n block in stages
// of `boxes` boxes of [brow rows x n columns] through a ring, released as soon as they land.  Separates
// the DRAM / TMA side of the tall kernels from their compute pipelines.
__global__ void __launch_bounds__(64, 1)
tma_stream_kernel(const __grid_constant__ CUtensorMap tm, const __grid_constant__ CUtensorMap tmp, int pd, int64_t M,
                  int brow, int boxes, int box_bytes, int ring) {
    using namespace tc;
    extern __shared__ unsigned char smem_raw[];
    unsigned char *smem = smem_align1024(smem_raw);
    const int stage = boxes * box_bytes;
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem + (size_t)ring * stage);
    const uint32_t bar0 = smem_u32(bars);
    auto full = [&](int r) { return bar0 + 8u * r; };
    auto emp = [&](int r) { return bar0 + 8u * (32 + r); };
    const int64_t rows = (int64_t)brow * boxes;
    const int64_t nst = (M + rows - 1) / rows;
    const int nmy = (int)max((int64_t)0, (nst - (int64_t)blockIdx.x + gridDim.x - 1) / gridDim.x);
    if (threadIdx.x == 0) {
        for (int r = 0; r < ring; ++r) { mbar_init(full(r), 1); mbar_init(emp(r), 1); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int i = 0; i < nmy; ++i) {
            const int r = i % ring;
            if (i >= ring) mbar_wait(emp(r), ((i / ring) - 1) & 1);
            mbar_expect_tx(full(r), stage);
            const int r0 = (int)(((int64_t)blockIdx.x + (int64_t)i * gridDim.x) * rows);
            if (pd > 0) {   // L2 prefetch of stage i + pd in one 128-row box per stage
                const int64_t rp = ((int64_t)blockIdx.x + (int64_t)(i + pd) * gridDim.x) * rows;
                if (rp < M)
                    asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];"
                                 ::"l"(reinterpret_cast<uint64_t>(&tmp)), "r"((int)rp), "r"(0) : "memory");
            }
            if (pd < 0) {   // 3D views: -1: box {32 rows, boxes row blocks, n cols}; -2: box {32 rows, n cols, boxes}
                for (int b = 0; b < boxes; b += 4) {
                    if (pd == -1) tma_load_2d(smem_u32(smem) + r * stage + b * box_bytes, &tm, 0, r0 / 32 + b, 0, full(r));
                    else tma_load_2d(smem_u32(smem) + r * stage + b * box_bytes, &tm, 0, 0, r0 / 32 + b, full(r));
                }
            } else {
                for (int b = 0; b < boxes; ++b)
                    tma_load_2d_true(smem_u32(smem) + r * stage + b * box_bytes, &tm, r0 + brow * b, 0, full(r));
            }
        }
    } else if (threadIdx.x == 32) {
        for (int i = 0; i < nmy; ++i) {
            const int r = i % ring;
            mbar_wait(full(r), (i / ring) & 1);
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(emp(r)) : "memory");
        }
    }
    __syncthreads();
}

void tma_stream_probe(int64_t M, const float *A, int64_t lda, int n, int brow, int boxes, bool swz, int pd, cudaStream_t st) {
    const CUtensorMap m =
        pd == -1 ? make_map3(A, 32, (uint64_t)(M / 32), (uint64_t)n, 128, (uint64_t)lda * 4, 32, 4, (uint32_t)n, true,
                             CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B)
        : pd == -2 ? make_map3(A, 32, (uint64_t)n, (uint64_t)(M / 32), (uint64_t)lda * 4, 128, 32, (uint32_t)n, 4, true,
                               CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B)
                   : make_map2(A, (uint64_t)M, (uint64_t)n, (uint64_t)lda * 4, (uint32_t)brow, (uint32_t)n, swz,
                               CU_TENSOR_MAP_L2_PROMOTION_L2_256B);
    const CUtensorMap mp = make_map2(A, (uint64_t)M, (uint64_t)n, (uint64_t)lda * 4, (uint32_t)(brow * boxes), (uint32_t)n,
                                     false, CU_TENSOR_MAP_L2_PROMOTION_L2_256B);
    const int box_bytes = brow * n * 4, stage = boxes * box_bytes;
    const int ring = std::min(32, (200 * 1024) / stage);
    set_max_smem(tma_stream_kernel);
    tma_stream_kernel<<<num_sms(), 64, ring * stage + 2048, st>>>(m, mp, pd, M, brow, boxes, box_bytes, ring);
    after_launch("tma_stream");
}

// tensor maps cached per (pointer, rows, columns, ld, box columns)
static const CUtensorMap &tall_map(const float *base, int64_t M, int ncols, int64_t ld, int boxc) {
    using Key = std::tuple<const float *, int64_t, int, int64_t, int>;
    static thread_local std::map<Key, CUtensorMap> cache;
    const Key key{base, M, ncols, ld, boxc};
    auto it = cache.find(key);
    if (it != cache.end()) return it->second;
    if (cache.size() > 256) cache.clear();
    return cache[key] = make_map2(base, (uint64_t)M, (uint64_t)ncols, (uint64_t)ld * 4, tallg::R, (uint32_t)boxc, true,
                                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B);
}

template <int NM, int NN, int BA, int RC, int KG>
static void launch_gram_tc3(int64_t M, const float *A, int64_t lda, int n1, const float *B, int64_t ldb, int n2,
                            double *partials, int ctas, cudaStream_t st) {
    // B = columns [b_col, b_col + n2) of A (same buffer and stride): taken from the A tiles where they lie
    int b_col = -1;
    if (ldb == lda && B >= A && (B - A) % lda == 0) {
        const int64_t c = (B - A) / lda;
        if (c % 8 == 0 && c + n2 <= n1) b_col = (int)c;
    }
    const CUtensorMap &ma = tall_map(A, M, n1, lda, BA);
    const CUtensorMap &mb = tall_map(B, M, n2, ldb, NN);
    auto kern = gram_tc3_kernel<NM, NN, BA, RC, KG>;
    set_max_smem(kern);
    const int gy = (int)cdiv(n1, NM * 128);
    // stages per accumulator drain: 1.  Four (256 rows of fp32 tensor-core accumulation per Kahan
    // step) was 0.3 ms faster per isolated c5 Gram (scripts/bench_tall_c5.py) but cost the c5
    // decomposition 9 ms (49.5 -> 58.6 ms, measured twice): the coarser accumulation changed the
    // orthonormalisation's decisions downstream.
    constexpr int per = 1;
    kern<<<dim3(ctas, gy), tallg::NTHR, tallg3::SMEM, st>>>(ma, mb, M, n1, n2, b_col, partials, per);
    after_launch("gram_tc3");
}

template <int NM, int NN, int BA>
static void launch_gram_tc(int64_t M, const float *A, int64_t lda, int n1, const float *B, int64_t ldb, int n2,
                           double *partials, int ctas, cudaStream_t st) {
    // RC = 2 (64-row stages) where the TMEM A buffers allow it; KG = 4 k-steps per accumulator
    if constexpr (NM == 1) launch_gram_tc3<NM, NN, BA, 2, 4>(M, A, lda, n1, B, ldb, n2, partials, ctas, st);
    else launch_gram_tc3<NM, NN, BA, 1, 2>(M, A, lda, n1, B, ldb, n2, partials, ctas, st);
}

// B tiles of all 32-column chunks, packed once per update as the exact shared-memory images
// (K-major, 128-B swizzle): Bpk[chunk][hi | lo][NN rows j][32 columns c] = split(alpha·C[c, j])
template <int NN>
__global__ void coef_pack_kernel(int m, const double *__restrict__ C, int ldc, int n, double alpha, float *Bpk) {
    const int ch = blockIdx.x;
    float *hi = Bpk + (size_t)ch * 2 * NN * 32, *lo = hi + NN * 32;
    for (int e = threadIdx.x; e < NN * 32; e += blockDim.x) {
        const int j = e / 32, cc = e % 32, c = ch * 32 + cc;
        const float v = (j < n && c < m) ? (float)(alpha * C[c + (int64_t)ldc * j]) : 0.f;
        const float hv = __uint_as_float(tc::tf32_rna(v));
        const uint32_t off = (tc::sw128_off(j, cc >> 2) + 4 * (cc & 3)) / 4;
        hi[off] = hv;
        lo[off] = v - hv;
    }
}

template <int NN>
static void launch_update_tc2(const float *A, int64_t lda, int64_t M, int m, const double *C, int ldc, int n,
                              double alpha, double beta, float *Out, int64_t ldo, cudaStream_t st) {
    using Key = std::tuple<const float *, int64_t, int, int64_t>;
    static thread_local std::map<Key, CUtensorMap> cache;
    const Key key{A, M, m, lda};
    auto it = cache.find(key);
    if (it == cache.end()) {
        if (cache.size() > 256) cache.clear();
        it = cache.emplace(key, make_map2(A, (uint64_t)M, (uint64_t)m, (uint64_t)lda * 4, tallu2::ROWS, tallu2::KC,
                                          false, CU_TENSOR_MAP_L2_PROMOTION_L2_256B)).first;
    }
    const int nchk = (m + tallu2::KC - 1) / tallu2::KC * (tallu2::KC / 32);   // 32-column chunks, zero padded
    static thread_local DevBuf bpk;
    const size_t need = sizeof(float) * (size_t)nchk * 2 * NN * 32;
    if (bpk.bytes < need) bpk.alloc(need, st);
    coef_pack_kernel<NN><<<nchk, 256, 0, st>>>(m, C, ldc, n, alpha, bpk.as<float>());
    after_launch("coef_pack");
    // epilogue: tensor store (beta = 0) / add-reduce (beta = 1) when Out's layout allows a tensor map
    const int omode = ((beta == 0.0 || beta == 1.0) && !(ldo & 3) && !((uintptr_t)Out & 15) && ldo >= M && M <= INT32_MAX)
                          ? (beta == 0.0 ? 1 : 2) : 0;
    const CUtensorMap *mo = &it->second;
    if (omode) {
        static thread_local std::map<Key, CUtensorMap> ocache;
        const Key okey{Out, M, n, ldo};
        auto jt = ocache.find(okey);
        if (jt == ocache.end()) {
            if (ocache.size() > 256) ocache.clear();
            jt = ocache.emplace(okey, make_map2(Out, (uint64_t)M, (uint64_t)n, (uint64_t)ldo * 4, 32, 32, false,
                                               CU_TENSOR_MAP_L2_PROMOTION_L2_256B)).first;
        }
        mo = &jt->second;
    }
    auto kern = update_tc2_kernel<NN>;
    set_max_smem(kern);
    const int ctas = (int)std::min<int64_t>(num_sms(), cdiv(M, tallu2::ROWS));
    kern<<<ctas, tallu2::NTHR, tallu2::SMEM, st>>>(it->second, *mo, omode, M, m, bpk.as<float>(), n, beta, Out, ldo);
    after_launch("update_tc2");
}

// Out = beta·Out + alpha·A·C on the tensor cores; false when unsupported (caller: CUDA cores).
// Needs lda a multiple of 32 with lda >= M rounded up to 32 (the solver's padded bases), 16-B
// aligned A, M < 2^31 · 32.
bool update_tc(int64_t M, const float *A, int64_t lda, int m, const double *C, int ldc, int n, double alpha,
               double beta, float *Out, int64_t ldo, cudaStream_t st) {
    static const int mode = [] { const char *e = std::getenv("SSA_UPD_TC"); return e ? std::atoi(e) : 1; }();
    // measured (scripts/bench_tall.py, M = 201,601): 85 µs vs 171 µs (FFMA) at m = 224, 60 vs 81 at m = 96,
    // but 40 vs 29 at m = 32 — narrow updates stay on the CUDA cores
    if (!mode || M < 8192 || n > 64 || m > 4096 || (mode == 1 && m < 64) || (lda & 31) || lda < (M + 31) / 32 * 32 ||
        ((uintptr_t)A & 127))
        return false;
    if (n <= 32) launch_update_tc2<32>(A, lda, M, m, C, ldc, n, alpha, beta, Out, ldo, st);
    else launch_update_tc2<64>(A, lda, M, m, C, ldc, n, alpha, beta, Out, ldo, st);
    return true;
}

// Returns false when the shape / layout is not supported (the caller uses the CUDA-core path).
bool gram_tc(int64_t M, const float *A, int64_t lda, int n1, const float *B, int64_t ldb, int n2, double *G,
             double *partials, size_t partial_bytes, cudaStream_t st) {
    if (M < 8192 || n2 > 64 || n1 > 512 || (lda & 3) || (ldb & 3) || ((uintptr_t)A & 15) ||
        ((uintptr_t)B & 15) || M > INT32_MAX)
        return false;
    const int ctas = (int)std::min<int64_t>(num_sms(), cdiv(M, tallg::R));
    auto self_ok = [&](const float *X, int n) {
        return n <= 64 && !(lda & 31) && !((uintptr_t)X & 127) &&
               (size_t)ctas * 4096 * sizeof(double) * 2 <= partial_bytes;
    };
    // self Gram XᵀX (n <= 64 columns): hi / lo stacked on M, one MMA per k-step (gram_self_kernel);
    // result into G with leading dimension ldg
    auto self_gram = [&](const float *X, int n, double *Gout, int ldg) {
        const int nc = n <= 32 ? 32 : 64;
        constexpr int self_rows = 128;
        // unswizzled boxes of self_rows rows x nc columns (the kernel relayouts them for the MMA)
        using Key = std::tuple<const float *, int64_t, int, int64_t, int>;
        static thread_local std::map<Key, CUtensorMap> cache;
        const Key key{X, M, n, lda, nc * 1000 + self_rows};
        auto it = cache.find(key);
        if (it == cache.end()) {
            if (cache.size() > 256) cache.clear();
            it = cache.emplace(key, make_map2(X, (uint64_t)M, (uint64_t)n, (uint64_t)lda * 4, self_rows, (uint32_t)nc,
                                              false, CU_TENSOR_MAP_L2_PROMOTION_L2_256B)).first;
        }
        auto go = [&](auto kern) {
            set_max_smem(kern);
            kern<<<ctas, tallgs::NTHR, tallgs::SMEM, st>>>(it->second, M, partials);
        };
        // one accumulator per 256 rows (32 k-steps of fp32 tensor-core accumulation, then Kahan sums)
        // (64-row stages with 4 per accumulator: 882 µs vs 806 µs at c5's K side)
        if (nc == 32) go(gram_self_kernel<32, self_rows, 2>);
        else go(gram_self_kernel<64, self_rows, 2>);
        after_launch("gram_self");
        gram_reduce_stacked_kernel<<<(unsigned)cdiv((int64_t)n * n * 32, 256), 256, 0, st>>>(partials, ctas, nc, n, Gout,
                                                                                             ldg);
        after_launch("gram_reduce_stacked");
    };
    if (B == A && ldb == lda && n2 == n1 && self_ok(A, n1)) {
        self_gram(A, n1, G, n1);
        return true;
    }
    // [A W]ᵀW with W = the last n2 = 64 columns of A, more than one 128-column block: AᵀW over the first
    // n1 − n2 columns (W loaded beside them) plus WᵀW by the self-Gram kernel — one full wave each,
    // instead of a second, nearly empty wave of CTAs that re-reads W (c5 K side, n1 = 192: 4.6 ms, ncu)
    if (n2 == 64 && n1 > 128 && ldb == lda && B == A + (int64_t)(n1 - n2) * lda && self_ok(B, n2) &&
        (size_t)ctas * 4096 * sizeof(double) * (size_t)cdiv(n1 - n2, 64) <= partial_bytes) {
        const int na = n1 - n2;
        launch_gram_tc<1, 64, 128>(M, A, lda, na, B, ldb, n2, partials, ctas, st);
        gram_reduce(partials, ctas, na, n2, G, st, n1);
        self_gram(B, n2, G + na, n1);
        return true;
    }
    if ((size_t)ctas * 4096 * sizeof(double) * (size_t)cdiv(n1, 64) > partial_bytes) return false;
    // narrow blocks (n1 <= 64, e.g. the CholeskyQR Gram WᵀW): a 64-column A box, B read from the A tile
    if (n2 <= 32) {
        if (n1 <= 64) launch_gram_tc<1, 32, 64>(M, A, lda, n1, B, ldb, n2, partials, ctas, st);
        // two M-tiles per CTA (B read once per 256 columns) up to 256 columns; above that a second
        // nearly empty y-block made it slower than 128-column CTAs (n1 = 288: 136 vs 107 µs)
        else if (n1 <= 128 || n1 > 256) launch_gram_tc<1, 32, 128>(M, A, lda, n1, B, ldb, n2, partials, ctas, st);
        else launch_gram_tc<2, 32, 128>(M, A, lda, n1, B, ldb, n2, partials, ctas, st);
    } else {
        if (n1 <= 64) launch_gram_tc<1, 64, 64>(M, A, lda, n1, B, ldb, n2, partials, ctas, st);
        else launch_gram_tc<1, 64, 128>(M, A, lda, n1, B, ldb, n2, partials, ctas, st);
    }
    gram_reduce(partials, ctas, n1, n2, G, st);
    return true;
}

}  // namespace ssa
