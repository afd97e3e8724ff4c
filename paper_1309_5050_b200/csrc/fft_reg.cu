// Register-resident radix-16 FFT passes of the FFT correlation path (SURVEY §8(a) a4-a6, a10:
// the method of Alg. 1/3/5, re-derived for the device).
//
// The round-1 passes ran every radix-8 Stockham stage through shared memory (load 8, twiddle,
// butterfly, store 8 per thread and stage) and were instruction / latency bound (c5 pass B: 3.8 G
// warp instructions per launch at ~50% issue efficiency; c3: 50-60% of shared-memory wavefronts
// were bank conflicts).  Here a 2^LG-point transform (LG = 8..12) is owned by NT = 2^LG / 16
// threads that each hold 16 elements in registers for the whole transform:
//
//   stage 0   radix R0 = 2^(LG mod 4) (16 if LG mod 4 = 0), span 1, no twiddles; a thread does
//             16/R0 butterflies in registers;
//   stage s   radix 16, span Ns = R0·16^(s-1): one shared-memory exchange (Stockham output
//             index (j − k)·16 + k + Ns·r, k = j mod Ns, read back strided), twiddles
//             e^{∓2πi r k/(16 Ns)} from a per-stage table in shared memory (15 per k read as 16-B pairs,
//             at a 144-B stride: conflict-free), then a 16-point DFT in registers (4 x 4, 32 real
//             multiplies, 144 adds).
//
// Thread t holds x[t + NT·e] (e < 16) before the transform and X[t + NT·e] after it, so global
// loads and stores are coalesced along t, and the inverse transform of pass B starts from the
// registers the forward one ended in (the spectrum product needs no exchange).  Shared-memory
// indices are padded by one element per 16 (i + i/16), which makes every exchange pattern above
// conflict-free for 8-byte accesses.  4096 points: 2 exchanges per transform instead of 4 stages
// through shared memory, ~45 instructions per point instead of ~60.
//
// Intermediate layouts are the ones of fft.cu (A[(j*H + fx)*by + col], B[(j*H + fx)*oy + y]), so a
// pass can run either implementation.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <map>
#include <mutex>
#include <vector>

#include "common.h"
#include "fft_reg.h"
#include "tc_common.h"

namespace ssa {
namespace rfft {

__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) { return make_float2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
    return make_float2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
// a * conj(b)
__device__ __forceinline__ float2 cmulc(float2 a, float2 b) {
    return make_float2(a.x * b.x + a.y * b.y, a.y * b.x - a.x * b.y);
}
// DIR·i·a (DIR = −1 forward, +1 inverse)
template <int DIR> __device__ __forceinline__ float2 mul_i(float2 a) {
    return DIR > 0 ? make_float2(-a.y, a.x) : make_float2(a.y, -a.x);
}

template <int DIR> __device__ __forceinline__ void dft2(float2 &a0, float2 &a1) {
    const float2 t = a0;
    a0 = cadd(t, a1);
    a1 = csub(t, a1);
}
// X[k] = Σ_n x[n] ω^{nk}, ω = DIR·i; natural order in and out
template <int DIR> __device__ __forceinline__ void dft4(float2 &a0, float2 &a1, float2 &a2, float2 &a3) {
    const float2 t0 = cadd(a0, a2), t1 = csub(a0, a2);
    const float2 t2 = cadd(a1, a3), t3 = mul_i<DIR>(csub(a1, a3));
    a0 = cadd(t0, t2);
    a2 = csub(t0, t2);
    a1 = cadd(t1, t3);
    a3 = csub(t1, t3);
}
template <int DIR> __device__ __forceinline__ void dft8(float2 *v, int s) {   // elements v[i*s]
    float2 e0 = v[0], e1 = v[2 * s], e2 = v[4 * s], e3 = v[6 * s];
    float2 o0 = v[s], o1 = v[3 * s], o2 = v[5 * s], o3 = v[7 * s];
    dft4<DIR>(e0, e1, e2, e3);
    dft4<DIR>(o0, o1, o2, o3);
    const float h = 0.70710678118654752440f;
    o1 = make_float2(h * (o1.x - (float)DIR * o1.y), h * (o1.y + (float)DIR * o1.x));
    o2 = mul_i<DIR>(o2);
    o3 = make_float2(h * (-o3.x - (float)DIR * o3.y), h * (-o3.y + (float)DIR * o3.x));
    v[0] = cadd(e0, o0); v[4 * s] = csub(e0, o0);
    v[s] = cadd(e1, o1); v[5 * s] = csub(e1, o1);
    v[2 * s] = cadd(e2, o2); v[6 * s] = csub(e2, o2);
    v[3 * s] = cadd(e3, o3); v[7 * s] = csub(e3, o3);
}

// 16-point DFT in natural order: n = n1 + 4 n2, k = k2 + 4 k1:
// X[k2 + 4k1] = Σ_{n1} ω4^{n1 k1} ω16^{n1 k2} Σ_{n2} x[n1 + 4n2] ω4^{n2 k2}
template <int DIR> __device__ __forceinline__ void dft16(float2 *v) {
#pragma unroll
    for (int n1 = 0; n1 < 4; ++n1) dft4<DIR>(v[n1], v[n1 + 4], v[n1 + 8], v[n1 + 12]);   // Y[n1][k2] at v[n1 + 4k2]
    const float c1 = 0.92387953251128675613f, s1 = 0.38268343236508977173f, h = 0.70710678118654752440f;
    const float d = (float)DIR;
    auto rot = [](float2 a, float c, float s) { return make_float2(a.x * c - a.y * s, a.x * s + a.y * c); };
    // ω16^m = cos(2πm/16) + DIR·i·sin(2πm/16)
    v[1 + 4] = rot(v[1 + 4], c1, d * s1);                                                    // ω^1
    v[1 + 8] = make_float2(h * (v[1 + 8].x - d * v[1 + 8].y), h * (v[1 + 8].y + d * v[1 + 8].x));   // ω^2
    v[1 + 12] = rot(v[1 + 12], s1, d * c1);                                                  // ω^3
    v[2 + 4] = make_float2(h * (v[2 + 4].x - d * v[2 + 4].y), h * (v[2 + 4].y + d * v[2 + 4].x));   // ω^2
    v[2 + 8] = mul_i<DIR>(v[2 + 8]);                                                         // ω^4
    v[2 + 12] = make_float2(h * (-v[2 + 12].x - d * v[2 + 12].y), h * (-v[2 + 12].y + d * v[2 + 12].x));   // ω^6
    v[3 + 4] = rot(v[3 + 4], s1, d * c1);                                                    // ω^3
    v[3 + 8] = make_float2(h * (-v[3 + 8].x - d * v[3 + 8].y), h * (-v[3 + 8].y + d * v[3 + 8].x));   // ω^6
    v[3 + 12] = rot(v[3 + 12], -c1, -d * s1);                                                // ω^9
#pragma unroll
    for (int k2 = 0; k2 < 4; ++k2) dft4<DIR>(v[4 * k2], v[4 * k2 + 1], v[4 * k2 + 2], v[4 * k2 + 3]);   // X[k2+4k1] at v[4k2+k1]
    float2 o[16];
#pragma unroll
    for (int k2 = 0; k2 < 4; ++k2)
#pragma unroll
        for (int k1 = 0; k1 < 4; ++k1) o[k2 + 4 * k1] = v[4 * k2 + k1];
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = o[i];
}

__device__ __forceinline__ int pad(int i) { return i + (i >> 4); }
__host__ __device__ constexpr int pad_size(int n) { return n + n / 16 + 1; }
__host__ __device__ constexpr int r0_of(int lg) { return (lg & 3) ? (1 << (lg & 3)) : 16; }
// twiddle-table entries of all radix-16 stages: Σ spans · 15 = N − R0
// Twiddle table: per radix-16 stage of span NS, for each k < NS the 15 factors e^{∓2πi r k/(16 NS)},
// r = 1..15, plus one pad entry, at a stride of TWS = 18 complex values (144 B): the factors are read as
// 8 16-B pairs, and the 144-B stride puts the 8 threads of a quarter-warp on disjoint banks.  The stage
// of span NS starts at TWS·(NS − R0)/15 (= TWS·Σ of the earlier spans).
constexpr int TWS = 18;
__host__ __device__ constexpr int tw_off(int lg, int ns) { return TWS * ((ns - r0_of(lg)) / 15); }
__host__ __device__ constexpr int tw_count_c(int lg) { return tw_off(lg, 1 << lg); }
__host__ __device__ constexpr int H_of(int lg) { return (1 << lg) / 2 + 1; }

template <int NT> __device__ __forceinline__ void xsync() {
    if constexpr (NT <= 32) __syncwarp();
    else __syncthreads();
}

// stage-0 butterflies: radix R0, 16/R0 per thread, inputs v[b + B·r]
template <int DIR, int R> __device__ __forceinline__ void stage0(float2 *v) {
    constexpr int B = 16 / R;
    if constexpr (R == 16) {
        dft16<DIR>(v);
    } else {
#pragma unroll
        for (int b = 0; b < B; ++b) {
            if constexpr (R == 2) dft2<DIR>(v[b], v[b + B]);
            else if constexpr (R == 4) dft4<DIR>(v[b], v[b + B], v[b + 2 * B], v[b + 3 * B]);
            else dft8<DIR>(v + b, B);
        }
    }
}

// Stockham exchange after a stage of radix RP and span NSP: outputs to shared memory, read back
// x[t + NT·e] for the next stage
template <int NT, int RP, int NSP> __device__ __forceinline__ void exchange(float2 *v, float2 *S, int t) {
    constexpr int B = 16 / RP;
#pragma unroll
    for (int b = 0; b < B; ++b) {
        const int j = t + NT * b;
        const int k = j & (NSP - 1);
        const int base = (j - k) * RP + k;
        if constexpr (NSP % 16 == 0 || (NSP == 1 && RP == 16)) {
            // pad(base + NSP·r) = pad(base) + (NSP + NSP/16)·r (NSP·r a multiple of 16, or r < 16 = RP with
            // base a multiple of 16)
            const unsigned pb = (unsigned)base + ((unsigned)base >> 4);
#pragma unroll
            for (int r = 0; r < RP; ++r) S[pb + (NSP + NSP / 16) * r] = v[b + B * r];
        } else {
#pragma unroll
            for (int r = 0; r < RP; ++r) S[pad(base + NSP * r)] = v[b + B * r];
        }
    }
    xsync<NT>();
    // pad(t + NT·e) = (t + t/16) + (NT + NT/16)·e for NT % 16 == 0: one base register and immediate
    // offsets (the signed form cost two address instructions per element, ncu SASS of pass B)
    const float2 *Sr = S + ((unsigned)t + ((unsigned)t >> 4));
#pragma unroll
    for (int e = 0; e < 16; ++e) v[e] = Sr[(NT + NT / 16) * e];
    xsync<NT>();
}

// KEEP1: only the outputs X[t] (e = 0) are needed (pass B of X·V keeps the first Ly <= NT rows):
// the last stage then forms just the r = 0 output of its 16-point DFT, Σ_r twiddled inputs
template <int LG, int DIR, int RP, int NSP, bool KEEP1, bool SKIPX = false>
__device__ __forceinline__ void stages16(float2 *v, float2 *S, const float2 *__restrict__ tw, int t) {
    constexpr int N = 1 << LG, NT = N >> 4, NS = NSP * RP;
    if constexpr (NS < N) {
        if constexpr (!SKIPX) exchange<NT, RP, NSP>(v, S, t);
        const int k = t & (NS - 1);
        const float4 *w = reinterpret_cast<const float4 *>(tw + tw_off(LG, NS) + TWS * k);
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const float4 c4 = w[q];
            float2 ca = make_float2(c4.x, c4.y), cb = make_float2(c4.z, c4.w);
            if (DIR > 0) { ca.y = -ca.y; cb.y = -cb.y; }
            v[2 * q + 1] = cmul(v[2 * q + 1], ca);
            if (q < 7) v[2 * q + 2] = cmul(v[2 * q + 2], cb);
        }
        if constexpr (KEEP1 && NS * 16 == N) {
            float2 s0 = v[0], s1 = v[1];
#pragma unroll
            for (int r = 2; r < 16; r += 2) { s0 = cadd(s0, v[r]); s1 = cadd(s1, v[r + 1]); }
            v[0] = cadd(s0, s1);
        } else {
            dft16<DIR>(v);
            stages16<LG, DIR, 16, NS, KEEP1>(v, S, tw, t);
        }
    }
}

// Full 2^LG-point DFT of the data held as v[e] = x[t + NT·e]; on return v[e] = X[t + NT·e] (KEEP1:
// only v[0] = X[t] is valid).  triv0: only the r = 0 inputs of every stage-0 butterfly are nonzero
// (x[i] = 0 for i >= NT·16/R0), so stage 0 just replicates them.  All NT threads of the transform
// (and, for NT > 32, all threads of the CTA) must call it together.
template <int LG, int DIR, bool KEEP1 = false>
__device__ __forceinline__ void fft(float2 *v, float2 *S, const float2 *__restrict__ tw, int t, bool triv0) {
    constexpr int R0 = r0_of(LG), B0 = 16 / R0;
    if (triv0) {
#pragma unroll
        for (int b = 0; b < B0; ++b)
#pragma unroll
            for (int r = 1; r < R0; ++r) v[b + B0 * r] = v[b];
    } else {
        stage0<DIR, R0>(v);
    }
    stages16<LG, DIR, R0, 1, KEEP1>(v, S, tw, t);
}

// Launch shapes.  Passes A and C (HBM-bound, transposed column access) run TPC = 2 transforms
// (4 real columns: 32-byte segments per fx) per CTA at 2^12 points and 256-thread CTAs below,
// with 64 registers per thread.  Pass B (compute-bound: two transforms and the spectrum product per
// row) runs 256-thread CTAs with up to 85 registers (3 CTAs / SM), which avoids the local-memory
// spills a 64-register budget causes; the grouped averaging keeps a running sum and needs 128.
template <int LG, bool ROWPASS = false> struct Cfg {
    static constexpr int N = 1 << LG, NT = N / 16, H = N / 2 + 1;
    static constexpr int TPC = ROWPASS ? (NT >= 256 ? 1 : 256 / NT) : (NT >= 256 ? 2 : 256 / NT);
    static constexpr int THREADS = NT * TPC;
    static constexpr int MINB = ROWPASS ? (LG == 12 ? 3 : 2) : 65536 / (THREADS * 64);
    static constexpr int TW = tw_count_c(LG);
    static constexpr int TWP = (TW + 1) & ~1;               // keep the buffers 16-B aligned
    static constexpr int XB = (pad_size(N) + 1) & ~1;       // one exchange buffer
    static constexpr size_t smem = sizeof(float2) * ((size_t)TWP + (size_t)TPC * XB);
};

template <int LG> __device__ __forceinline__ float2 *stage_tw(float2 *sm, const float2 *__restrict__ twg) {
    for (int i = threadIdx.x; i < Cfg<LG>::TW; i += blockDim.x) sm[i] = twg[i];
    return sm;
}
template <int LG> __device__ __forceinline__ float2 *xbuf(float2 *sm, int q) {
    return sm + Cfg<LG>::TWP + (size_t)q * Cfg<LG>::XB;
}

// All passes are persistent: a grid of (resident CTAs per SM) x (SMs) CTAs loops over the work items,
// so the twiddle table is staged into shared memory once per CTA rather than once per item (one
// 32 KB table per 32 KB row of pass B was half of its L2 traffic, ncu), and launch tails vanish.

// Address of element (row fx, column y) of vector / group j in the intermediate B between pass B and
// pass C: row layout (cbc = 0: B[(j*H + fx)*ldb + y]) or blocked by pass C's column blocks
// (cbc = its CB: B[((j*nyb + y/cbc)*H + fx)*cbc + y%cbc]), in which pass C's item — all H rows of
// cbc columns — is one contiguous block: its reads stream instead of gathering a 32-B sector per row
// (the row layout left c5's Xᵀ·U pass C at 1.5 TB/s, ncu); pass B's writes take the scatter instead.
__device__ __forceinline__ int64_t boff(int j, int fx, int y, int H, int ldb, int cbc, int nyb) {
    if (cbc == 0) return ((int64_t)j * H + fx) * ldb + y;
    const int yb = y / cbc;
    return (((int64_t)j * nyb + yb) * H + fx) * cbc + (y - yb * cbc);
}

// ------------------------------------------------------------------------------------ pass A
// item = (vector jo, block of CB = 2·TPC input columns); consecutive CTAs take consecutive column
// blocks of one vector (contiguous reads)
template <int LG>
__global__ void __launch_bounds__(Cfg<LG>::THREADS, Cfg<LG>::MINB)
rpass_a(const float *__restrict__ in, int64_t ld, const int *__restrict__ map, int bx, int by, int k,
        const int *__restrict__ jsel, const double *__restrict__ scale, float2 *__restrict__ A, int lda,
        const float2 *__restrict__ twg) {
    using C = Cfg<LG>;
    constexpr int N = C::N, NT = C::NT, H = C::H, TPC = C::TPC, CB = 2 * TPC;
    extern __shared__ float2 sm[];
    const float2 *tw = stage_tw<LG>(sm, twg);
    const int q = threadIdx.x / NT, t = threadIdx.x % NT;
    float2 *S = xbuf<LG>(sm, q);
    const int nb = (by + CB - 1) / CB, items = nb * k;
    __syncthreads();   // twiddle table staged
    for (int it = blockIdx.x; it < items; it += gridDim.x) {
        const int jo = it / nb, col0 = (it - jo * nb) * CB;
        const int j = jsel ? jsel[jo] : jo;
        const int ca = col0 + 2 * q, cb = ca + 1;
        const float *src = in + ld * j;
        float2 v[16];
        if (!map) {
            // all 32 loads issued before any use (the round-1 form with a per-element map test and scale
            // serialised load -> use -> next load: 5.4 ms of latency-bound pass A on c5, ncu)
            const float *pa = src + (int64_t)bx * min(ca, by - 1), *pb = src + (int64_t)bx * min(cb, by - 1);
#pragma unroll
            for (int e = 0; e < 16; ++e) {
                const int ix = t + NT * e;
                v[e].x = ix < bx ? __ldg(pa + ix) : 0.f;
                v[e].y = ix < bx ? __ldg(pb + ix) : 0.f;
            }
            if (ca >= by)
#pragma unroll
                for (int e = 0; e < 16; ++e) v[e].x = 0.f;
            if (cb >= by)
#pragma unroll
                for (int e = 0; e < 16; ++e) v[e].y = 0.f;
        } else {
            int ia[16], ib[16];
#pragma unroll
            for (int e = 0; e < 16; ++e) {
                const int ix = t + NT * e;
                ia[e] = (ix < bx && ca < by) ? map[ix + (int64_t)bx * ca] : -1;
                ib[e] = (ix < bx && cb < by) ? map[ix + (int64_t)bx * cb] : -1;
            }
#pragma unroll
            for (int e = 0; e < 16; ++e) {
                v[e].x = ia[e] >= 0 ? __ldg(src + ia[e]) : 0.f;
                v[e].y = ib[e] >= 0 ? __ldg(src + ib[e]) : 0.f;
            }
        }
        fft<LG, -1>(v, S, tw, t, false);
        // Hermitian split of the two packed real columns: X_a[f] = (Z[f] + conj Z[−f]) / 2,
        // X_b[f] = (Z[f] − conj Z[−f]) / (2i); needs Z[f] and Z[N − f] (held by other threads).  The
        // per-vector scale (σ_i of the averaging) is linear and applied here.
#pragma unroll
        for (int e = 0; e < 16; ++e) S[pad(t + NT * e)] = v[e];
        __syncthreads();
        const float hs = 0.5f * (scale ? (float)scale[j] : 1.f);
        // transposed write: one 16-B store of the column pair (2q2, 2q2 + 1) per (fx, q2);
        // consecutive threads -> consecutive pairs of one fx (32-B aligned rows of stride lda)
        float2 *arow = A + (int64_t)jo * H * lda + col0;
        for (int idx = threadIdx.x; idx < H * TPC; idx += blockDim.x) {
            const int fx = idx / TPC, q2 = idx - fx * TPC;
            const int col = col0 + 2 * q2;
            if (col >= by) continue;
            const float2 *Sq = xbuf<LG>(sm, q2);
            const float2 z = Sq[pad(fx)], zm = Sq[pad((N - fx) & (N - 1))];
            const float4 o = make_float4(hs * (z.x + zm.x), hs * (z.y - zm.y), hs * (z.y + zm.y), hs * (zm.x - z.x));
            float2 *dst = arow + (int64_t)fx * lda + 2 * q2;
            if (col + 1 < by) *reinterpret_cast<float4 *>(dst) = o;
            else *dst = make_float2(o.x, o.y);
        }
        __syncthreads();   // the buffers are rewritten by the next item
    }
}

// ------------------------------------------------------------------------------ pipelined A / C
// Passes A and C alternate a memory phase (a block of columns in, a block out) with a compute phase
// (the transforms); run as above, one CTA's loads wait for its own transforms and the two phases add
// up (c5: X·V pass A and Xᵀ·U pass C at ~2.9 TB/s, with the 4096-point transforms costing about as
// long as the block's transfer).  Here the CTA owns two buffer sets of TPC exchange buffers: while
// the transforms of item n run in set n&1 — first as the staging area its input arrived in, then as
// the exchange buffers — one bulk asynchronous copy (cp.async.bulk, mbarrier completion) brings item
// n+1's input into the other set, so the HBM stream never waits for the ALUs.  Both inputs are
// contiguous per item: pass A's CB input columns of the box (x fastest), pass C's H x CB block of the
// blocked B layout (boff).  Shared memory: twiddles + 2·TPC exchange buffers (172 KB at 2^12 points,
// one 512-thread CTA per SM).
template <int LG> struct CfgP {
    static constexpr int THREADS = Cfg<LG>::THREADS;
    static constexpr size_t set_elems = (size_t)Cfg<LG>::TPC * Cfg<LG>::XB;   // float2 per buffer set
    static constexpr size_t smem = sizeof(float2) * ((size_t)Cfg<LG>::TWP + 2 * set_elems) + 16;
};
__device__ __forceinline__ void mbar_arrive1(uint32_t bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
// bytes (multiple of 16, 16-B aligned ends) from global to shared, completing on `bar`: chunks of
// at most 32 KB (expect_tx counts per instruction are limited), then the producer's arrival
__device__ __forceinline__ void bulk_in(float2 *dst, const void *src, uint32_t bytes, uint32_t bar) {
    const uint32_t d = tc::smem_u32(dst);
    for (uint32_t o = 0; o < bytes; o += 32768u) {
        const uint32_t n = min(32768u, bytes - o);
        tc::mbar_expect_tx_noarrive(bar, n);
        tc::bulk_g2s(d + o, static_cast<const char *>(src) + o, n, bar);
    }
    mbar_arrive1(bar);
}
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// pass A, pipelined: same items and outputs as rpass_a (identity map: rectangular box).  Staged input
// of item (jo, col0): the CB columns in[ld·j + bx·col0 ...], bx floats each, from the 16-B boundary at
// or below their start; the part beyond their last 16-B boundary is read directly from global memory.
template <int LG>
__global__ void __launch_bounds__(CfgP<LG>::THREADS, 1)
rpass_a2(const float *__restrict__ in, int64_t ld, int bx, int by, int k, const int *__restrict__ jsel,
         const double *__restrict__ scale, float2 *__restrict__ A, int lda, const float2 *__restrict__ twg) {
    using C = Cfg<LG>;
    constexpr int N = C::N, NT = C::NT, H = C::H, TPC = C::TPC, CB = 2 * TPC;
    extern __shared__ float2 sm[];
    const float2 *tw = stage_tw<LG>(sm, twg);
    float2 *set0 = sm + C::TWP;
    uint64_t *bars = reinterpret_cast<uint64_t *>(set0 + 2 * CfgP<LG>::set_elems);
    const uint32_t bar0 = tc::smem_u32(bars), bar1 = tc::smem_u32(bars + 1);
    const int q = threadIdx.x / NT, t = threadIdx.x % NT;
    const int nb = (by + CB - 1) / CB, items = nb * k;
    auto src_of = [&](int it, int &ncol) {
        const int jo = it / nb, col0 = (it - jo * nb) * CB;
        const int j = jsel ? jsel[jo] : jo;
        ncol = min(CB, by - col0);
        return in + ld * j + (int64_t)bx * col0;
    };
    // staged range: from src rounded down to 16 B (off < 4 floats before it, inside the allocation
    // since `in` itself is 16-B aligned) to the last 16-B boundary inside the item's columns
    auto staged = [&](const float *src, int ncol, int &off) {
        off = (int)((reinterpret_cast<uintptr_t>(src) & 15) >> 2);
        const int64_t end = (int64_t)off + (int64_t)bx * ncol;
        return (int)(end & ~int64_t(3));   // staged floats, counted from src - off
    };
    auto issue = [&](int it, int s) {
        int ncol, off;
        const float *src = src_of(it, ncol);
        const int nst = staged(src, ncol, off);
        bulk_in(set0 + s * CfgP<LG>::set_elems, src - off, (uint32_t)nst * 4u, s ? bar1 : bar0);
    };
    if (threadIdx.x == 0) {
        tc::mbar_init(bar0, 1);
        tc::mbar_init(bar1, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();   // twiddle table staged, barriers initialised
    if (threadIdx.x == 0 && (int)blockIdx.x < items) issue(blockIdx.x, 0);
    int n = 0;
    for (int it = blockIdx.x; it < items; it += gridDim.x, ++n) {
        const int s = n & 1;
        if (threadIdx.x == 0 && it + (int)gridDim.x < items) issue(it + gridDim.x, s ^ 1);
        const int jo = it / nb, col0 = (it - jo * nb) * CB;
        const int j = jsel ? jsel[jo] : jo;
        int ncol;
        const float *src = src_of(it, ncol);
        int off;
        const int nflt = staged(src, ncol, off) - off;   // staged floats from src on
        float2 *base = set0 + s * CfgP<LG>::set_elems;
        const float *raw = reinterpret_cast<const float *>(base) + off;
        tc::mbar_wait(s ? bar1 : bar0, (n >> 1) & 1);
        const int ca = 2 * q, cb = ca + 1;
        float2 v[16];
#pragma unroll
        for (int e = 0; e < 16; ++e) {
            const int ix = t + NT * e;
            const int ia = ca * bx + ix, ib = cb * bx + ix;
            v[e].x = (ix < bx && ca < ncol) ? (ia < nflt ? raw[ia] : __ldg(src + ia)) : 0.f;
            v[e].y = (ix < bx && cb < ncol) ? (ib < nflt ? raw[ib] : __ldg(src + ib)) : 0.f;
        }
        __syncthreads();   // every staged value is in registers: the set becomes the exchange buffers
        float2 *S = base + (size_t)q * C::XB;
        fft<LG, -1>(v, S, tw, t, false);
#pragma unroll
        for (int e = 0; e < 16; ++e) S[pad(t + NT * e)] = v[e];
        __syncthreads();
        const float hs = 0.5f * (scale ? (float)scale[j] : 1.f);
        float2 *arow = A + (int64_t)jo * H * lda + col0;
        // unrolled: all shared-memory reads of the thread's (fx, pair) outputs before the first store
        // (the rolled loop exposed the read latency once per output, ncu source page)
        constexpr int PER = (H * TPC + C::THREADS - 1) / C::THREADS;
        float2 zz[PER], zzm[PER];
#pragma unroll
        for (int u = 0; u < PER; ++u) {
            const int idx = threadIdx.x + C::THREADS * u;
            const int fx = idx / TPC, q2 = idx - fx * TPC;
            const float2 *Sq = base + (size_t)q2 * C::XB;
            if (idx < H * TPC) { zz[u] = Sq[pad(fx)]; zzm[u] = Sq[pad((N - fx) & (N - 1))]; }
        }
#pragma unroll
        for (int u = 0; u < PER; ++u) {
            const int idx = threadIdx.x + C::THREADS * u;
            const int fx = idx / TPC, q2 = idx - fx * TPC;
            const int col = col0 + 2 * q2;
            if (idx >= H * TPC || col >= by) continue;
            const float2 z = zz[u], zm = zzm[u];
            const float4 o = make_float4(hs * (z.x + zm.x), hs * (z.y - zm.y), hs * (z.y + zm.y), hs * (zm.x - z.x));
            float2 *dst = arow + (int64_t)fx * lda + 2 * q2;
            if (col + 1 < by) *reinterpret_cast<float4 *>(dst) = o;
            else *dst = make_float2(o.x, o.y);
        }
        fence_async_smem();   // generic accesses of this set ordered before the next bulk copy into it
        __syncthreads();
    }
}

// ------------------------------------------------------------------------------------ pass B
// item = (vector j, block of TPC rows fx); the k items that use the same X̂ rows are consecutive
// (X̂ stays in L2 while the much larger A stream passes).
// TRIVL (R0 = 16 and ny_in <= NT: Xᵀ·U, whose input rows hold only Ly nonzero entries): stage 0 of
// every butterfly would just replicate its one nonzero input, so the row is loaded directly in the
// layout the first exchange produces, v[e] = x[t/16 + (NT/16)·e], and the transform starts at the
// span-16 stage (one exchange and one stage less).  The B stores use per-thread base addresses and
// a constant stride per e (the per-element index arithmetic with a division by the block width was
// ~35% of the Xᵀ·U pass-B instructions, ncu SASS, profiles/r02).
template <int LG, bool KEEP1, bool TRIVL>
__global__ void __launch_bounds__(Cfg<LG, true>::THREADS, Cfg<LG, true>::MINB)
rpass_b(const float2 *__restrict__ A, int ny_in, int lda, int H, int k, const float2 *__restrict__ Xh,
        float2 *__restrict__ B, int ny_out, int ldb, int cbc, const float2 *__restrict__ twg) {
    using C = Cfg<LG, true>;
    constexpr int N = C::N, NT = C::NT, TPC = C::TPC, B0 = 16 / r0_of(LG);
    static_assert(!TRIVL || r0_of(LG) == 16, "direct exchanged-layout load needs a radix-16 stage 0");
    extern __shared__ float2 sm[];
    const float2 *tw = stage_tw<LG>(sm, twg);
    const int q = threadIdx.x / NT, t = threadIdx.x % NT;
    float2 *S = xbuf<LG>(sm, q);
    const int items = k * ((H + TPC - 1) / TPC);
    const bool triv = ny_in <= NT * B0;
    const bool full_in = t + NT * 15 < ny_in;
    // B addressing, y = t + NT·e: fixed base per (j, fx) and a constant stride es per e
    const int nyb = cbc ? (ny_out + cbc - 1) / cbc : 0;
    const bool fastst = cbc == 0 || NT % cbc == 0;
    const int tq = cbc ? t / cbc : 0, tr = cbc ? t - tq * cbc : t;
    const int64_t es = cbc ? (int64_t)(NT / max(cbc, 1)) * H * cbc : NT;
    const int ne = t < ny_out ? min(16, (ny_out - t + NT - 1) / NT) : 0;
    __syncthreads();
    for (int it = blockIdx.x; it < items; it += gridDim.x) {
        const int j = it % k;
        const int fx = (it / k) * TPC + q;
        const bool ok = fx < H;
        const float2 *arow = A + ((int64_t)j * H + (ok ? fx : 0)) * lda;
        float2 v[16];
        if constexpr (TRIVL) {
            const int t16 = t >> 4;
#pragma unroll
            for (int e = 0; e < 16; ++e) {
                const int y = t16 + (NT / 16) * e;
                v[e] = (ok && y < ny_in) ? arow[y] : make_float2(0.f, 0.f);
            }
            stages16<LG, -1, 16, 1, false, true>(v, S, tw, t);
        } else {
            if (ok && full_in) {
#pragma unroll
                for (int e = 0; e < 16; ++e) v[e] = arow[t + NT * e];
            } else {
#pragma unroll
                for (int e = 0; e < 16; ++e) {
                    const int y = t + NT * e;
                    v[e] = (ok && y < ny_in) ? arow[y] : make_float2(0.f, 0.f);
                }
            }
            fft<LG, -1>(v, S, tw, t, triv);
        }
        const float2 *xr = Xh + (int64_t)(ok ? fx : 0) * N;
#pragma unroll
        for (int e = 0; e < 16; ++e) v[e] = cmulc(__ldg(xr + t + NT * e), v[e]);   // X̂ ⊙ conj(Â)
        if constexpr (KEEP1) {   // X·V: only the first Ly <= NT rows of the inverse are kept
            fft<LG, +1, true>(v, S, tw, t, false);
            if (ok && t < ny_out) B[boff(j, fx, t, H, ldb, cbc, nyb)] = v[0];
        } else {
            fft<LG, +1>(v, S, tw, t, false);
            if (ok && fastst) {
                float2 *bp = B + (cbc ? ((((int64_t)j * nyb + tq) * H + fx) * cbc + tr)
                                      : (((int64_t)j * H + fx) * ldb + t));
#pragma unroll
                for (int e = 0; e < 16; ++e)
                    if (e < ne) bp[e * es] = v[e];
            } else if (ok) {
#pragma unroll
                for (int e = 0; e < 16; ++e) {
                    const int y = t + NT * e;
                    if (y < ny_out) B[boff(j, fx, y, H, ldb, cbc, nyb)] = v[e];
                }
            }
        }
    }
}

// Pass B, X̂-resident form (work unit = one row fx and a chunk of JC vectors): the X̂ row is copied
// into shared memory once per unit (cp.async, overlapped with the unit's first forward transform)
// instead of 16 dependent L2 loads per thread and item after the forward transform (the top stall
// of rpass_b on c5's Xᵀ·U: long scoreboard, ncu); A rows of the next item are loaded into registers
// while the current item's inverse transform runs.  Shared memory per CTA: twiddles + exchange
// buffer + X̂ row (~100 KB at 2^12 points: 2 CTAs / SM, up to 128 registers per thread).
template <int LG> struct CfgB2 {
    static constexpr int N = 1 << LG, NT = N / 16, THREADS = NT;
    // X̂ row held per thread: element t + NT·e at Xs[t·TWS + e] (16-B pairs, 144-B thread stride)
    static constexpr size_t smem = Cfg<LG, true>::smem + sizeof(float2) * (size_t)NT * TWS;
};
__device__ __forceinline__ void cp_async8(void *sdst, const void *gsrc) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(sdst);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sa), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

template <int LG, bool KEEP1, bool TRIVL, int JC>
__global__ void __launch_bounds__(CfgB2<LG>::THREADS, 2)
rpass_b2(const float2 *__restrict__ A, int ny_in, int lda, int H, int k, const float2 *__restrict__ Xh,
         float2 *__restrict__ B, int ny_out, int ldb, int cbc, const float2 *__restrict__ twg) {
    using C = Cfg<LG, true>;
    constexpr int N = C::N, NT = C::NT, B0 = 16 / r0_of(LG);
    static_assert(C::TPC == 1, "one transform per CTA");
    static_assert(!TRIVL || r0_of(LG) == 16, "direct exchanged-layout load needs a radix-16 stage 0");
    extern __shared__ float2 sm[];
    const float2 *tw = stage_tw<LG>(sm, twg);
    float2 *S = xbuf<LG>(sm, 0);
    float2 *Xs = sm + C::TWP + C::XB;                    // X̂ row of the current unit
    const int t = threadIdx.x;
    const int nch = (k + JC - 1) / JC, units = H * nch;
    const bool triv = ny_in <= NT * B0;
    const bool full_in = t + NT * 15 < ny_in;
    const int nyb = cbc ? (ny_out + cbc - 1) / cbc : 0;
    const bool fastst = cbc == 0 || NT % cbc == 0;
    const int tq = cbc ? t / cbc : 0, tr = cbc ? t - tq * cbc : t;
    const int64_t es = cbc ? (int64_t)(NT / max(cbc, 1)) * H * cbc : NT;
    const int ne = t < ny_out ? min(16, (ny_out - t + NT - 1) / NT) : 0;
    auto load_row = [&](float2 *v, int j, int fx) {
        const float2 *arow = A + ((int64_t)j * H + fx) * lda;
        if constexpr (TRIVL) {
            const int t16 = t >> 4;
#pragma unroll
            for (int e = 0; e < 16; ++e) {
                const int y = t16 + (NT / 16) * e;
                v[e] = y < ny_in ? __ldg(arow + y) : make_float2(0.f, 0.f);
            }
        } else if (full_in) {
#pragma unroll
            for (int e = 0; e < 16; ++e) v[e] = __ldg(arow + t + NT * e);
        } else {
#pragma unroll
            for (int e = 0; e < 16; ++e) {
                const int y = t + NT * e;
                v[e] = y < ny_in ? __ldg(arow + y) : make_float2(0.f, 0.f);
            }
        }
    };
    __syncthreads();   // twiddle table staged
    for (int u = blockIdx.x; u < units; u += gridDim.x) {
        const int fx = u / nch, j0 = (u - fx * nch) * JC, j1 = min(k, j0 + JC);
        // X̂ row -> shared memory in the thread-major layout (8 B per copy, coalesced global reads; the
        // previous unit's readers are past a barrier); read back as 8 16-B pairs per thread and item
        {
            const float2 *xr = Xh + (int64_t)fx * N + t;
#pragma unroll
            for (int e = 0; e < 16; ++e) cp_async8(Xs + TWS * t + e, xr + NT * e);
            asm volatile("cp.async.commit_group;" ::: "memory");
        }
        float2 v[16];
        load_row(v, j0, fx);
        bool xs_ready = false;
        for (int j = j0; j < j1; ++j) {
            if constexpr (TRIVL) stages16<LG, -1, 16, 1, false, true>(v, S, tw, t);
            else fft<LG, -1>(v, S, tw, t, triv);
            if (!xs_ready) {   // the first forward transform covered the copy's latency
                cp_async_wait_all();
                __syncthreads();
                xs_ready = true;
            }
            {   // X̂ ⊙ conj(Â)
                const float4 *xp = reinterpret_cast<const float4 *>(Xs + TWS * t);
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    const float4 x4 = xp[q];
                    v[2 * q] = cmulc(make_float2(x4.x, x4.y), v[2 * q]);
                    v[2 * q + 1] = cmulc(make_float2(x4.z, x4.w), v[2 * q + 1]);
                }
            }
            float2 vn[16];
            if (j + 1 < j1) load_row(vn, j + 1, fx);   // in flight during the inverse transform
            if constexpr (KEEP1) {
                fft<LG, +1, true>(v, S, tw, t, false);
                if (t < ny_out) B[boff(j, fx, t, H, ldb, cbc, nyb)] = v[0];
            } else {
                fft<LG, +1>(v, S, tw, t, false);
                if (fastst) {
                    float2 *bp = B + (cbc ? ((((int64_t)j * nyb + tq) * H + fx) * cbc + tr)
                                          : (((int64_t)j * H + fx) * ldb + t));
#pragma unroll
                    for (int e = 0; e < 16; ++e)
                        if (e < ne) bp[e * es] = v[e];
                } else {
#pragma unroll
                    for (int e = 0; e < 16; ++e) {
                        const int y = t + NT * e;
                        if (y < ny_out) B[boff(j, fx, y, H, ldb, cbc, nyb)] = v[e];
                    }
                }
            }
#pragma unroll
            for (int e = 0; e < 16; ++e) v[e] = vn[e];
        }
        __syncthreads();   // all reads of Xs done before the next unit's copy
    }
}

// averaging: per (g, fx) Σ_{i∈I_g} DFT_y(AU_i) ⊙ DFT_y(AV_i), inverse; the AU transform of a member
// waits in a thread-private shared-memory slot while the AV transform runs
// (2^12 points: two CTAs per SM within 128 registers — c5's averaging was latency-bound at one;
// smaller transforms spill at that budget and keep one)
template <int LG>
__global__ void __launch_bounds__(Cfg<LG, true>::THREADS, LG == 12 ? 2 : 1)
rpass_bconv(const float2 *__restrict__ AU, int ly, int ldu, const float2 *__restrict__ AV, int ky, int ldv,
            const int *__restrict__ grp_off, const int *__restrict__ grp_idx, const int *__restrict__ slot, int H, int ng,
            float2 *__restrict__ B, int ny_out, int ldb, int cbc, const float2 *__restrict__ twg) {
    using C = Cfg<LG, true>;
    constexpr int NT = C::NT, TPC = C::TPC, B0 = 16 / r0_of(LG);
    extern __shared__ float2 sm[];
    const float2 *tw = stage_tw<LG>(sm, twg);
    const int q = threadIdx.x / NT, t = threadIdx.x % NT;
    float2 *S = xbuf<LG>(sm, q);
    float2 *P = xbuf<LG>(sm, TPC + q);      // private slots of this transform
    const int nfb = (H + TPC - 1) / TPC, items = ng * nfb;
    __syncthreads();
    for (int it = blockIdx.x; it < items; it += gridDim.x) {
        const int g = it / nfb;
        const int fx = (it - g * nfb) * TPC + q;
        const bool ok = fx < H;
        float2 acc[16];
#pragma unroll
        for (int e = 0; e < 16; ++e) acc[e] = make_float2(0.f, 0.f);
        for (int m = grp_off[g]; m < grp_off[g + 1]; ++m) {
            const int s = slot[grp_idx[m]];
            float2 v[16];
            const float2 *ur = AU + ((int64_t)s * H + (ok ? fx : 0)) * ldu;
#pragma unroll
            for (int e = 0; e < 16; ++e) {
                const int y = t + NT * e;
                v[e] = (ok && y < ly) ? ur[y] : make_float2(0.f, 0.f);
            }
            fft<LG, -1>(v, S, tw, t, ly <= NT * B0);
#pragma unroll
            for (int e = 0; e < 16; ++e) P[pad(t + NT * e)] = v[e];
            const float2 *vr = AV + ((int64_t)s * H + (ok ? fx : 0)) * ldv;
#pragma unroll
            for (int e = 0; e < 16; ++e) {
                const int y = t + NT * e;
                v[e] = (ok && y < ky) ? vr[y] : make_float2(0.f, 0.f);
            }
            fft<LG, -1>(v, S, tw, t, ky <= NT * B0);
#pragma unroll
            for (int e = 0; e < 16; ++e) {
                const float2 u = P[pad(t + NT * e)];
                acc[e] = cadd(acc[e], cmul(u, v[e]));
            }
        }
        fft<LG, +1>(acc, S, tw, t, false);
        const int nyb = cbc ? (ny_out + cbc - 1) / cbc : 0;
#pragma unroll
        for (int e = 0; e < 16; ++e) {
            const int y = t + NT * e;
            if (ok && y < ny_out) B[boff(g, fx, y, H, ldb, cbc, nyb)] = acc[e];
        }
    }
}

// ------------------------------------------------------------------------------------ pass C
// item = (vector j, block of CB = 2·TPC output columns)
template <int LG>
__global__ void __launch_bounds__(Cfg<LG>::THREADS, Cfg<LG>::MINB)
rpass_c(const float2 *__restrict__ B, int oy, int ldb, int cblk, int H, int k, int ox, float inv,
        float *__restrict__ out, int64_t ldo, const int *__restrict__ omap, const int *__restrict__ w, int64_t stride,
        const float2 *__restrict__ twg, const double *__restrict__ cs) {
    using C = Cfg<LG>;
    constexpr int N = C::N, NT = C::NT, TPC = C::TPC, CB = 2 * TPC, THR = C::THREADS;
    constexpr int PER = (H_of(LG) * TPC + THR - 1) / THR;   // gathered column pairs per thread
    extern __shared__ float2 sm[];
    const float2 *tw = stage_tw<LG>(sm, twg);
    const int q = threadIdx.x / NT, t = threadIdx.x % NT;
    float2 *S = xbuf<LG>(sm, q);
    const int H0 = C::H;
    const int nb = (oy + CB - 1) / CB, items = nb * k;
    __syncthreads();
    for (int it = blockIdx.x; it < items; it += gridDim.x) {
        const int j = it / nb, y0 = (it - j * nb) * CB;
        const int ncol = min(CB, oy - y0);
        // gather the CB half-spectrum columns: transform q's buffer holds columns 2q (at [0, H)) and
        // 2q + 1 (at [H, 2H)); one 16-B load per (fx, column pair), consecutive threads -> consecutive
        // pairs of one fx; all of a thread's loads are issued before the shared-memory stores (the
        // per-element form was latency-bound: 5.3 ms for c5's Xᵀ·U pass C, ncu)
        // row layout: rows of stride ldb; blocked layout: this item's CB columns inside the H x cblk
        // block that holds them (rows of stride cblk; the cblk/CB consecutive items of a block read
        // the 32-B sectors of the same 128-B lines together)
        const float2 *bj;
        int64_t rs;
        if (cblk) {
            const int nyb = (oy + cblk - 1) / cblk, yb = y0 / cblk;
            bj = B + ((int64_t)j * nyb + yb) * H0 * cblk + (y0 - yb * cblk);
            rs = cblk;
        } else {
            bj = B + (int64_t)j * H0 * ldb + y0;
            rs = ldb;
        }
        float4 tmp[PER];
#pragma unroll
        for (int u = 0; u < PER; ++u) {
            const int idx = threadIdx.x + THR * u;
            const int fx = idx / TPC, q2 = idx - fx * TPC;
            tmp[u] = (idx < H0 * TPC && 2 * q2 < ncol)
                         ? __ldg(reinterpret_cast<const float4 *>(bj + (int64_t)fx * rs + 2 * q2))
                         : make_float4(0.f, 0.f, 0.f, 0.f);
            if (2 * q2 + 1 >= ncol) { tmp[u].z = 0.f; tmp[u].w = 0.f; }   // padding column: never written
        }
#pragma unroll
        for (int u = 0; u < PER; ++u) {
            const int idx = threadIdx.x + THR * u;
            const int fx = idx / TPC, q2 = idx - fx * TPC;
            if (idx < H0 * TPC) {
                float2 *Sq = xbuf<LG>(sm, q2);
                Sq[fx] = make_float2(tmp[u].x, tmp[u].y);
                Sq[H0 + fx] = make_float2(tmp[u].z, tmp[u].w);
            }
        }
        __syncthreads();
        // Z[f] = Y_a[f] + i·Y_b[f] over the full spectrum (Y[N − f] = conj Y[f] for real columns;
        // the bins 0 and N/2 of a real column are real)
        float2 v[16];
#pragma unroll
        for (int e = 0; e < 16; ++e) {
            const int f = t + NT * e;
            const bool lo = f <= N / 2;
            const int fs = lo ? f : N - f;
            float2 ya = S[fs], yb = S[H0 + fs];
            if (!lo) { ya.y = -ya.y; yb.y = -yb.y; }
            if (f == 0 || f == N / 2) { ya.y = 0.f; yb.y = 0.f; }
            v[e] = make_float2(ya.x - yb.y, ya.y + yb.x);
        }
        __syncthreads();   // the buffers are reused by the exchanges
        fft<LG, +1>(v, S, tw, t, false);
        const int ya_col = y0 + 2 * q;
        const float sc = cs ? (float)((double)inv * cs[j]) : inv;
        if (!w && !omap) {
            // products on a full box: out[x + ox·y + ldo·j] with x = t + NT·e — one base pointer and
            // immediate offsets (the generic path below spent ~20 instructions per element)
            float *o0 = out + ldo * j + (int64_t)ox * ya_col + t;
            const bool c0 = ya_col - y0 < ncol, c1 = ya_col + 1 - y0 < ncol;
#pragma unroll
            for (int e = 0; e < 16; ++e) {
                if (t + NT * e >= ox) break;
                if (c0) o0[NT * e] = v[e].x * sc;
                if (c1) o0[ox + NT * e] = v[e].y * sc;
            }
            __syncthreads();
            continue;
        }
#pragma unroll
        for (int e = 0; e < 16; ++e) {
            const int x = t + NT * e;
            if (x >= ox) continue;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int y = ya_col + h;
                if (y - y0 >= ncol) continue;
                const float val = (h ? v[e].y : v[e].x) * sc;
                if (w) {
                    const int wn = w[x + (int64_t)ox * y];
                    out[(int64_t)j * stride + x + ldo * y] = wn > 0 ? val / (float)wn : __int_as_float(0x7fc00000);
                } else {
                    const int64_t box = x + (int64_t)ox * y;
                    const int64_t oi = omap ? (int64_t)omap[box] : box;
                    if (oi >= 0) out[oi + ldo * j] = val;
                }
            }
        }
        __syncthreads();
    }
}

// pass C, pipelined (blocked B layout with cbc = CB only): same items and outputs as rpass_c.  The
// item's H x CB block is one contiguous bulk copy; transform q reads its column pair (2q, 2q + 1) as
// one 16-B value per frequency.
template <int LG>
__global__ void __launch_bounds__(CfgP<LG>::THREADS, 1)
rpass_c2(const float2 *__restrict__ B, int oy, int H, int k, int ox, float inv, float *__restrict__ out,
         int64_t ldo, const int *__restrict__ omap, const int *__restrict__ w, int64_t stride,
         const float2 *__restrict__ twg, const double *__restrict__ cs) {
    using C = Cfg<LG>;
    constexpr int N = C::N, NT = C::NT, TPC = C::TPC, CB = 2 * TPC;
    extern __shared__ float2 sm[];
    const float2 *tw = stage_tw<LG>(sm, twg);
    float2 *set0 = sm + C::TWP;
    uint64_t *bars = reinterpret_cast<uint64_t *>(set0 + 2 * CfgP<LG>::set_elems);
    const uint32_t bar0 = tc::smem_u32(bars), bar1 = tc::smem_u32(bars + 1);
    const int q = threadIdx.x / NT, t = threadIdx.x % NT;
    const int H0 = C::H;
    const int nb = (oy + CB - 1) / CB, items = nb * k;
    const uint32_t bytes = (uint32_t)H0 * CB * sizeof(float2);
    auto issue = [&](int it, int s) {
        // item it = (j, block yb) is block j·nb + yb of the blocked layout: blocks are consecutive
        bulk_in(set0 + s * CfgP<LG>::set_elems, B + (int64_t)it * H0 * CB, bytes, s ? bar1 : bar0);
    };
    if (threadIdx.x == 0) {
        tc::mbar_init(bar0, 1);
        tc::mbar_init(bar1, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0 && (int)blockIdx.x < items) issue(blockIdx.x, 0);
    int n = 0;
    for (int it = blockIdx.x; it < items; it += gridDim.x, ++n) {
        const int s = n & 1;
        if (threadIdx.x == 0 && it + (int)gridDim.x < items) issue(it + gridDim.x, s ^ 1);
        const int j = it / nb, y0 = (it - j * nb) * CB;
        const int ncol = min(CB, oy - y0);
        float2 *base = set0 + s * CfgP<LG>::set_elems;
        const float4 *raw = reinterpret_cast<const float4 *>(base) + q;   // (fx, pair q) at raw[fx·TPC]
        tc::mbar_wait(s ? bar1 : bar0, (n >> 1) & 1);
        // Z[f] = Y_a[f] + i·Y_b[f] over the full spectrum (as rpass_c); never-written padding columns
        // of a ragged last block are zeroed
        const bool za = 2 * q >= ncol, zb = 2 * q + 1 >= ncol;
        float2 v[16];
#pragma unroll
        for (int e = 0; e < 16; ++e) {
            const int f = t + NT * e;
            const bool lo = f <= N / 2;
            const int fs = lo ? f : N - f;
            const float4 z = raw[fs * TPC];
            float2 ya = make_float2(z.x, z.y), yb = make_float2(z.z, z.w);
            if (!lo) { ya.y = -ya.y; yb.y = -yb.y; }
            if (f == 0 || f == N / 2) { ya.y = 0.f; yb.y = 0.f; }
            if (za) ya = make_float2(0.f, 0.f);
            if (zb) yb = make_float2(0.f, 0.f);
            v[e] = make_float2(ya.x - yb.y, ya.y + yb.x);
        }
        __syncthreads();   // the staged block is in registers: the set becomes the exchange buffers
        float2 *S = base + (size_t)q * C::XB;
        fft<LG, +1>(v, S, tw, t, false);
        const int ya_col = y0 + 2 * q;
        const float sc = cs ? (float)((double)inv * cs[j]) : inv;
        if (!w && !omap) {
            float *o0 = out + ldo * j + (int64_t)ox * ya_col + t;
            const bool c0 = !za, c1 = !zb;
#pragma unroll
            for (int e = 0; e < 16; ++e) {
                if (t + NT * e >= ox) break;
                if (c0) o0[NT * e] = v[e].x * sc;
                if (c1) o0[ox + NT * e] = v[e].y * sc;
            }
        } else {
#pragma unroll
            for (int e = 0; e < 16; ++e) {
                const int x = t + NT * e;
                if (x >= ox) continue;
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int y = ya_col + h;
                    if (y - y0 >= ncol) continue;
                    const float val = (h ? v[e].y : v[e].x) * sc;
                    if (w) {
                        const int wn = w[x + (int64_t)ox * y];
                        out[(int64_t)j * stride + x + ldo * y] = wn > 0 ? val / (float)wn : __int_as_float(0x7fc00000);
                    } else {
                        const int64_t box = x + (int64_t)ox * y;
                        const int64_t oi = omap ? (int64_t)omap[box] : box;
                        if (oi >= 0) out[oi + ldo * j] = val;
                    }
                }
            }
        }
        fence_async_smem();
        __syncthreads();
    }
}


// ------------------------------------------------------------------------------------ host side
int tw_count(int lg) { return tw_count_c(lg); }

void build_table(int lg, std::vector<float2> &h) {
    const int N = 1 << lg, R0 = r0_of(lg);
    h.assign((size_t)tw_count_c(lg), make_float2(0.f, 0.f));
    for (int ns = R0; ns < N; ns *= 16)
        for (int k = 0; k < ns; ++k)
            for (int r = 1; r < 16; ++r) {
                const double a = -2.0 * M_PI * (double)(r * k) / (16.0 * ns);
                h[(size_t)tw_off(lg, ns) + (size_t)TWS * k + (r - 1)] = make_float2((float)std::cos(a), (float)std::sin(a));
            }
}

// the kernel's dynamic shared memory exceeds the 48 KB default: raise the cap once per kernel;
// persistent grid = resident CTAs per SM (occupancy query, cached per kernel) x SMs, capped by the items
template <typename F> static int prep(F *kern, int threads, size_t smem, int64_t items) {
    set_max_smem(kern);
    static std::mutex mu;
    static std::map<const void *, int> occ;
    int per = 0;
    {
        std::lock_guard<std::mutex> lk(mu);
        auto itc = occ.find((const void *)kern);
        if (itc != occ.end()) {
            per = itc->second;
        } else {
            SSA_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, threads, smem));
            per = std::max(per, 1);
            occ[(const void *)kern] = per;
        }
    }
    return (int)std::min<int64_t>(items, (int64_t)per * num_sms());
}

#define RFFT_DISPATCH(lg, ...)                       \
    switch (lg) {                                     \
    case 8: { constexpr int LG = 8; __VA_ARGS__; } break;    \
    case 9: { constexpr int LG = 9; __VA_ARGS__; } break;    \
    case 10: { constexpr int LG = 10; __VA_ARGS__; } break;  \
    case 11: { constexpr int LG = 11; __VA_ARGS__; } break;  \
    case 12: { constexpr int LG = 12; __VA_ARGS__; } break;  \
    default: throw Error(SSA_ERR_ARG, "rfft: unsupported transform size"); \
    }

void pass_a(int lg, const float *in, int64_t ld, const int *map, int bx, int by, int k, const int *jsel,
            const double *scale, float2 *A, int lda, const float2 *tw, cudaStream_t st) {
    SSA_REQUIRE(lda % 2 == 0 && ((uintptr_t)A & 15) == 0, SSA_ERR_ARG, "rfft pass A: rows must be 16-B aligned");
    RFFT_DISPATCH(lg, {
        using Cf = Cfg<LG>;
        // (a 16-B aligned base keeps the staged ranges, which start at the 16-B boundary at or below each
        // item, inside the input)
        if (!map && ((uintptr_t)in & 15) == 0) {
            const int grid = prep(rpass_a2<LG>, Cf::THREADS, CfgP<LG>::smem, cdiv(by, 2 * Cf::TPC) * (int64_t)k);
            rpass_a2<LG><<<grid, Cf::THREADS, CfgP<LG>::smem, st>>>(in, ld, bx, by, k, jsel, scale, A, lda, tw);
            break;
        }
        const int grid = prep(rpass_a<LG>, Cf::THREADS, Cf::smem, cdiv(by, 2 * Cf::TPC) * (int64_t)k);
        rpass_a<LG><<<grid, Cf::THREADS, Cf::smem, st>>>(in, ld, map, bx, by, k, jsel, scale, A, lda, tw);
    });
    after_launch("rfft_pass_a");
}

// block width of the blocked B layout for a 2^lg-point pass C: its column group CB = 2·TPC.  (Blocks of
// 16 columns — whole 128-B lines for pass B's writes, read as 32-B sectors by 4 consecutive pass-C
// items — measured worse on c5's Xᵀ·U: pass B 3.8 ms / pass C 4.6 ms, against 4.0 / 3.1 ms here and
// 2.9 / 5.3 ms for the row layout; ncu launch lists.)
int cb_of(int lg) {
    int cb = 0;
    switch (lg) {
    case 8: cb = 2 * Cfg<8>::TPC; break;
    case 9: cb = 2 * Cfg<9>::TPC; break;
    case 10: cb = 2 * Cfg<10>::TPC; break;
    case 11: cb = 2 * Cfg<11>::TPC; break;
    default: cb = 2 * Cfg<12>::TPC; break;
    }
    return cb;
}

template <int LG>
static void pass_b_lg(const float2 *A, int ny_in, int lda, int H, int k, const float2 *Xh, float2 *B, int ny_out,
                      int ldb, int cbc, const float2 *tw, cudaStream_t st) {
    using Cf = Cfg<LG, true>;
    // X̂-resident form by default (c5: Xᵀ·U 5.59 -> 5.42 ms, X·V 5.45 -> 5.39 ms per block product);
    // (k = 1: the item-per-row form above)
    if constexpr (Cf::TPC == 1) {
        if (k > 1) {
            constexpr int JC = 16;
            const int64_t units = (int64_t)H * cdiv(k, JC);
            auto launch2 = [&](auto kern) {
                const int grid = prep(kern, CfgB2<LG>::THREADS, CfgB2<LG>::smem, units);
                kern<<<grid, CfgB2<LG>::THREADS, CfgB2<LG>::smem, st>>>(A, ny_in, lda, H, k, Xh, B, ny_out, ldb, cbc,
                                                                          tw);
            };
            const bool keep1 = ny_out <= Cf::NT;
            if constexpr (r0_of(LG) == 16) {
                if (ny_in <= Cf::NT) {
                    if (keep1) launch2(rpass_b2<LG, true, true, JC>);
                    else launch2(rpass_b2<LG, false, true, JC>);
                    return;
                }
            }
            if (keep1) launch2(rpass_b2<LG, true, false, JC>);
            else launch2(rpass_b2<LG, false, false, JC>);
            return;
        }
    }
    const int64_t items = cdiv(H, Cf::TPC) * (int64_t)k;
    auto launch = [&](auto kern) {
        const int grid = prep(kern, Cf::THREADS, Cf::smem, items);
        kern<<<grid, Cf::THREADS, Cf::smem, st>>>(A, ny_in, lda, H, k, Xh, B, ny_out, ldb, cbc, tw);
    };
    const bool keep1 = ny_out <= Cf::NT;
    if constexpr (r0_of(LG) == 16) {
        if (ny_in <= Cf::NT) {
            if (keep1) launch(rpass_b<LG, true, true>);
            else launch(rpass_b<LG, false, true>);
            return;
        }
    }
    if (keep1) launch(rpass_b<LG, true, false>);
    else launch(rpass_b<LG, false, false>);
}

void pass_b(int lg, const float2 *A, int ny_in, int lda, int H, int k, const float2 *Xh, float2 *B, int ny_out,
            int ldb, int cbc, const float2 *tw, cudaStream_t st) {
    RFFT_DISPATCH(lg, pass_b_lg<LG>(A, ny_in, lda, H, k, Xh, B, ny_out, ldb, cbc, tw, st));
    after_launch("rfft_pass_b");
}

void pass_bconv(int lg, const float2 *AU, int ly, int ldu, const float2 *AV, int ky, int ldv, const int *grp_off,
                const int *grp_idx, const int *slot, int H, int ng, float2 *B, int ny_out, int ldb, int cbc,
                const float2 *tw, cudaStream_t st) {
    RFFT_DISPATCH(lg, {
        using Cf = Cfg<LG, true>;
        const size_t smem = Cf::smem + sizeof(float2) * (size_t)Cf::TPC * Cf::XB;
        const int grid = prep(rpass_bconv<LG>, Cf::THREADS, smem, cdiv(H, Cf::TPC) * (int64_t)ng);
        rpass_bconv<LG><<<grid, Cf::THREADS, smem, st>>>(AU, ly, ldu, AV, ky, ldv, grp_off, grp_idx, slot, H, ng, B,
                                                          ny_out, ldb, cbc, tw);
    });
    after_launch("rfft_pass_bconv");
}

void pass_c(int lg, const float2 *B, int oy, int ldb, int cblk, int H, int k, int ox, float inv, float *out,
            int64_t ldo, const int *omap, const int *w, int64_t stride, const float2 *tw, cudaStream_t st,
            const double *cs) {
    SSA_REQUIRE(ldb % 2 == 0 && ((uintptr_t)B & 15) == 0, SSA_ERR_ARG, "rfft pass C: rows must be 16-B aligned");
    RFFT_DISPATCH(lg, {
        using Cf = Cfg<LG>;
        static_assert(2 * Cfg<LG>::H <= Cfg<LG>::XB, "column pair fits the exchange buffer");
        const int grid = prep(rpass_c<LG>, Cf::THREADS, Cf::smem, cdiv(oy, 2 * Cf::TPC) * (int64_t)k);
        SSA_REQUIRE(cblk == 0 || cblk % (2 * Cf::TPC) == 0, SSA_ERR_ARG, "rfft pass C: block width");
        if (cblk == 2 * Cf::TPC && H == Cf::H) {
            const int g2 = prep(rpass_c2<LG>, Cf::THREADS, CfgP<LG>::smem, cdiv(oy, 2 * Cf::TPC) * (int64_t)k);
            rpass_c2<LG><<<g2, Cf::THREADS, CfgP<LG>::smem, st>>>(B, oy, H, k, ox, inv, out, ldo, omap, w, stride, tw, cs);
            break;
        }
        rpass_c<LG><<<grid, Cf::THREADS, Cf::smem, st>>>(B, oy, ldb, cblk, H, k, ox, inv, out, ldo, omap, w, stride,
                                                         tw, cs);
    });
    after_launch("rfft_pass_c");
}

}  // namespace rfft
}  // namespace ssa
