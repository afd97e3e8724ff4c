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
#include <cstdlib>

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

// ---------------------------------------------------------------------------
// Cluster variant (n <= 32·BW): the nb/2 CTAs of ONE thread-block cluster keep the
// column blocks in shared memory for the whole factorisation.  With the circle
// method, the transition from round t to t+1 is a systolic shift: CTA c's "+c" block
// goes to CTA c-1, its "-c" block to CTA c+1 (CTA 0 keeps block nb-1; the last CTA
// turns its "-c" block into its "+c" block).  Blocks are pushed into the neighbours'
// next-round buffers through distributed shared memory and a cluster barrier replaces
// the grid synchronisation (no global-memory round trip per round).
// ---------------------------------------------------------------------------
template <int MR, int BW>
__global__ void __launch_bounds__(32 * BW, 1)
jacobi_cluster_kernel(int m, int n, int nb, double *__restrict__ A, float tol, int max_sweeps,
                      int *__restrict__ sweeps_out) {
    namespace cg = cooperative_groups;
    cg::cluster_group cluster = cg::this_cluster();
    extern __shared__ __align__(16) double SM[];
    __shared__ int flags[2];
    const int ldc = m | 1;
    const int blk = ldc * BW;                          // doubles per column block
    double *buf[2] = {SM, SM + 2 * blk};                // [2 buffers][slot A | slot B]
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int c = (int)cluster.block_rank(), ncta = nb / 2;
    constexpr int NP = 2 * BW;
    // initial blocks (round 0): CTA 0 -> (0, nb-1); CTA c -> (c, (nb-1-c) mod (nb-1))
    {
        const int ba = (c == 0) ? 0 : c % (nb - 1);
        const int bb = (c == 0) ? nb - 1 : (nb - 1 - c) % (nb - 1);
        for (int h = 0; h < 2; ++h) {
            const int b = h ? bb : ba;
            for (int idx = tid; idx < BW * m; idx += blockDim.x) {
                const int jl = idx / m, i = idx - jl * m;
                const int col = b * BW + jl;
                buf[0][h * blk + i + ldc * jl] = col < n ? A[i + (int64_t)m * col] : 0.0;
            }
        }
    }
    if (tid == 0) { flags[0] = 0; flags[1] = 0; }
    cluster.sync();
    int cur = 0, t = 0, sweep = 0;
    for (; sweep < max_sweeps; ++sweep) {
        int rot = 0;
        for (int round = 0; round < nb - 1; ++round, ++t) {
            double *C = buf[cur];
            // one inner sweep over the 2·BW columns held by this CTA
            for (int ir = 0; ir < NP - 1; ++ir) {
                int p, q;
                if (warp == 0) { p = ir; q = NP - 1; }
                else { p = (ir + warp) % (NP - 1); q = (ir - warp + (NP - 1)) % (NP - 1); }
                if (jacobi_pair<MR>(C + ldc * p, C + ldc * q, m, lane, tol)) rot = 1;
                __syncthreads();
            }
            // systolic shift into the neighbours' next buffers
            double *nxt_local = buf[cur ^ 1];
            if (ncta == 1) {
                // single CTA: nothing moves
                for (int idx = tid; idx < 2 * blk; idx += blockDim.x) nxt_local[idx] = C[idx];
            } else {
                double *dstA = nullptr, *dstB = nullptr;   // where my slot A / slot B go
                int offA = 0, offB = 0;
                if (c == 0) {
                    dstA = cluster.map_shared_rank(buf[cur ^ 1], 1); offA = blk;    // -> CTA 1 slot B
                    dstB = nxt_local; offB = blk;                                    // stays in slot B
                } else {
                    dstA = cluster.map_shared_rank(buf[cur ^ 1], c - 1); offA = 0;   // -> CTA c-1 slot A
                    if (c + 1 < ncta) { dstB = cluster.map_shared_rank(buf[cur ^ 1], c + 1); offB = blk; }
                    else { dstB = nxt_local; offB = 0; }                            // last CTA: B -> own A
                }
                for (int idx = tid; idx < blk; idx += blockDim.x) {
                    dstA[offA + idx] = C[idx];
                    dstB[offB + idx] = C[blk + idx];
                }
            }
            cluster.sync();
            cur ^= 1;
        }
        // sweep convergence: any CTA rotated?  (flags alternate with sweep parity)
        if (__syncthreads_or(rot) && tid == 0) atomicOr(cluster.map_shared_rank(&flags[sweep & 1], 0), 1);
        cluster.sync();
        const int any = *cluster.map_shared_rank(&flags[sweep & 1], 0);
        if (c == 0 && tid == 0) flags[(sweep + 1) & 1] = 0;
        cluster.sync();
        if (!any) break;
    }
    // write back: blocks held at round t
    {
        const int tt = t % (nb - 1);
        const int ba = (c == 0) ? tt : (tt + c) % (nb - 1);
        const int bb = (c == 0) ? nb - 1 : (tt - c + (nb - 1)) % (nb - 1);
        for (int h = 0; h < 2; ++h) {
            const int b = h ? bb : ba;
            for (int idx = tid; idx < BW * m; idx += blockDim.x) {
                const int jl = idx / m, i = idx - jl * m;
                const int col = b * BW + jl;
                if (col < n) A[i + (int64_t)m * col] = buf[cur][h * blk + i + ldc * jl];
            }
        }
    }
    if (c == 0 && tid == 0 && sweeps_out) *sweeps_out = sweep + 1;
}

// ---------------------------------------------------------------------------
// Gram-based cluster variant (the default).  Same block circle schedule and systolic
// DSMEM shift as jacobi_cluster_kernel, but one inner sweep over the NC = 2·BW columns
// a CTA holds is run on their NC x NC Gram matrix instead of on the m-long columns:
//   1. G = CᵀC on the fp64 tensor cores (DMMA m8n8k4, fp64 accumulate);
//   2. one cyclic two-sided Jacobi sweep on G (NC-1 steps of NC/2 disjoint rotations,
//      the same fp32-angle / fp64-rotation rule and skip test as jacobi_pair, applied to
//      the current G) accumulating V = J_1 J_2 ... (exactly orthogonal up to rounding);
//   3. C ← C·V on the tensor cores, the result tiles stored straight into the
//      neighbours' next-round buffers (the systolic shift fused into the epilogue).
// The rotations are those the column-wise inner sweep would apply (G carries the same
// inner products), but each step costs O(NC) instead of an m-long dot product plus a
// warp reduction.  Gram rounding only perturbs the angles at ε·|c_p||c_q| (a pair may
// need another visit); σ_j are still the column norms of the rotated T.  Column buffers
// use ld ≡ 4 (mod 16) doubles with zero padding rows (conflict-free fragment loads).
// ---------------------------------------------------------------------------
__device__ __forceinline__ void dmma884(double &d0, double &d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

template <int NC>
struct GramCfg {
    static constexpr int BW = NC / 2;
    static constexpr int NT = 256;                        // threads per CTA
    static constexpr int TILES = (NC / 8) * (NC / 8);     // 8x8 Gram tiles
    static constexpr int KSPLIT = TILES >= 8 ? 1 : 8 / TILES;
    static constexpr int LDG = NC + 1;
    __host__ __device__ static int ldc(int m) { return (m + 15) / 16 * 16 + 4; }
    static size_t smem(int m) {
        return sizeof(double) * ((size_t)2 * NC * ldc(m) + 4 * (size_t)NC * LDG + (size_t)KSPLIT * NC * NC);
    }
};

// Rotation of the pair (p, q) from al = |C_p|², be = |C_q|², ga = C_pᵀC_q (the rule of
// jacobi_pair: skip unless ga² > tol²·al·be, ζ = (be−al)/(2ga), t = sign(ζ)/(|ζ|+√(1+ζ²)),
// c = 1/√(1+t²), s = c·t).  The test is in fp64; the angle in fp32 on operands scaled
// by an exact power of two (no fp32 overflow for any fp64 input); c, s in fp64.
__device__ __forceinline__ float rcp_approx(float x) { float r; asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x)); return r; }
__device__ __forceinline__ float sqrt_approx(float x) { float r; asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x)); return r; }

__device__ __forceinline__ bool pair_rotation(double al, double be, double ga, double tol2, double &c, double &s,
                                              float &mrel) {
    c = 1.0; s = 0.0;
    // 2^-e with e the exponent of max(al, be): scaled operands are <= 1 in magnitude, so the skip
    // test and the angle run in fp32 without overflow (fewer dependent fp64 ops per step)
    const int hi = __double2hiint(fmax(al, be));
    const double scale = __hiloint2double(((2046 - ((hi >> 20) & 2047)) & 2047) << 20, 0);
    const float fa = (float)(al * scale), fb = (float)(be * scale), fg = (float)(ga * scale);
    if (!(fg * fg > (float)tol2 * fa * fb)) return false;
    mrel = fmaxf(mrel, fabsf(fg) * rsqrtf(fa * fb));   // relative off-diagonal (early stop)
    const float zeta = (fb - fa) * 0.5f * rcp_approx(fg);
    float tf = copysignf(1.0f, zeta) * rcp_approx(fabsf(zeta) + sqrt_approx(fmaf(zeta, zeta, 1.0f)));
    if (!isfinite(zeta)) tf = 0.0f;
    const double t = (double)tf;
    c = rsqrt(fma(t, t, 1.0));
    s = c * t;
    return true;
}

template <int NC>
__global__ void __launch_bounds__(256, 1)
jacobi_gram_kernel(int m, int n, int nb, double *__restrict__ A, float tol, float early, int max_sweeps,
                   int *__restrict__ sweeps_out) {
    using Cfg = GramCfg<NC>;
    constexpr int BW = Cfg::BW, LDG = Cfg::LDG;
    namespace cg = cooperative_groups;
    cg::cluster_group cluster = cg::this_cluster();
    extern __shared__ __align__(16) double SM[];
    __shared__ int flags[2];
    __shared__ int rot_sh, mrel_sh, mflags[2];
    const int ldc = Cfg::ldc(m);
    const int blk = ldc * BW;                               // doubles per column block (slot)
    double *const bufs = SM;                                // [2][NC][ldc]
    double *const Gs = SM + 2 * NC * ldc;                   // [2][NC][LDG] ping-pong Gram
    double *const Vs = Gs + 2 * NC * LDG;                   // [2][NC][LDG] ping-pong V (row-major V[x][y])
    double *const Gp = Vs + 2 * NC * LDG;                   // [KSPLIT][NC][NC] partial Grams
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int c = (int)cluster.block_rank(), ncta = nb / 2;
    const int m4 = (m + 3) & ~3, m8 = (m + 7) & ~7;
    for (int idx = tid; idx < 2 * NC * ldc; idx += Cfg::NT) bufs[idx] = 0.0;
    // step schedule.  A round pairs slot A (columns 0..BW-1) with slot B (BW..NC-1): BW "cross"
    // steps s with pairs (i, BW + (i+s) mod BW).  The first round of a sweep is preceded by BW-1
    // "intra" steps (circle method inside each slot), so every column pair is visited exactly
    // once per sweep, as in the cyclic ordering.  Steps 0..BW-2: intra, BW-1..NC-2: cross.
    //   tab[step][x] = partner | pair index << 8 | (x is the 'p' of its pair) << 16
    //   ptab[step][w] = p | q << 8
    __shared__ int tab[(NC - 1) * NC];
    __shared__ int ptab[(NC - 1) * (NC / 2)];
    for (int idx = tid; idx < (NC - 1) * (NC / 2); idx += Cfg::NT) {
        const int st = idx / (NC / 2), w = idx - st * (NC / 2);
        int p, q;
        if (st < BW - 1) {                       // intra: circle over BW players in slot w / (BW/2)
            constexpr int M1 = BW - 1;
            const int h = w / (BW / 2), v = w - h * (BW / 2);
            p = (v == 0) ? st : (st + v) % M1;
            q = (v == 0) ? M1 : (st - v + M1) % M1;
            p += h * BW; q += h * BW;
        } else {                                 // cross
            const int sx = st - (BW - 1);
            p = w;
            q = BW + (w + sx) % BW;
        }
        ptab[idx] = p | (q << 8);
        tab[st * NC + p] = q | (w << 8) | (1 << 16);
        tab[st * NC + q] = p | (w << 8);
    }
    const double tol2 = (double)tol * (double)tol;
    __syncthreads();
    {
        const int ba = (c == 0) ? 0 : c % (nb - 1);
        const int bb = (c == 0) ? nb - 1 : (nb - 1 - c) % (nb - 1);
        for (int h = 0; h < 2; ++h) {
            const int b = h ? bb : ba;
            for (int idx = tid; idx < BW * m; idx += Cfg::NT) {
                const int jl = idx / m, i = idx - jl * m;
                const int col = b * BW + jl;
                bufs[h * blk + i + ldc * jl] = col < n ? A[i + (int64_t)m * col] : 0.0;
            }
        }
    }
    if (tid == 0) { flags[0] = 0; flags[1] = 0; mflags[0] = 0; mflags[1] = 0; }
    cluster.sync();
    int cur = 0, t = 0, sweep = 0;
    for (; sweep < max_sweeps; ++sweep) {
        if (tid == 0) { rot_sh = 0; mrel_sh = 0; }
        for (int round = 0; round < nb - 1; ++round, ++t) {
            const double *C = bufs + cur * NC * ldc;
            // ---- 1. Gram G = CᵀC (tensor cores), k split over warps when there are few tiles
            {
                const int ks = warp % Cfg::KSPLIT;
                for (int tile = warp / Cfg::KSPLIT; tile < Cfg::TILES; tile += 8 / Cfg::KSPLIT) {
                    const int ta = tile / (NC / 8), tb = tile % (NC / 8);
                    const double *ca = C + ldc * (8 * ta + (lane >> 2)) + (lane & 3);
                    const double *cb = C + ldc * (8 * tb + (lane >> 2)) + (lane & 3);
                    double d[4][2] = {{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}};   // four accumulator chains
                    constexpr int KS4 = 4 * Cfg::KSPLIT;
                    for (int k0 = 4 * ks; k0 < m4; k0 += 4 * KS4) {
#pragma unroll
                        for (int q = 0; q < 4; ++q)   // warp-uniform guard, constant chain index
                            if (k0 + q * KS4 < m4) dmma884(d[q][0], d[q][1], ca[k0 + q * KS4], cb[k0 + q * KS4]);
                    }
                    const double d0 = (d[0][0] + d[1][0]) + (d[2][0] + d[3][0]);
                    const double d1 = (d[0][1] + d[1][1]) + (d[2][1] + d[3][1]);
                    double *gp = Gp + ks * NC * NC + NC * (8 * ta + (lane >> 2)) + 8 * tb + 2 * (lane & 3);
                    gp[0] = d0;
                    gp[1] = d1;
                }
            }
            __syncthreads();
            for (int e = tid; e < NC * NC; e += Cfg::NT) {
                double s = 0.0;
#pragma unroll
                for (int ks = 0; ks < Cfg::KSPLIT; ++ks) s += Gp[ks * NC * NC + e];
                const int x = e / NC, y = e - x * NC;
                Gs[x * LDG + y] = s;
                Vs[x * LDG + y] = (x == y) ? 1.0 : 0.0;
            }
            __syncthreads();
            // ---- 2. Jacobi steps on G, V accumulated: G_new = Jᵀ G J, V_new = V J (ping-pong
            // buffers, one barrier per step).  Every warp computes the NC/2 rotations of the step
            // (lane w -> pair w; identical on every warp) and hands them to the lanes owning
            // entries (x, y) by shuffles.
            int gi = 0;
            // skip the steps when none of the pairs this round visits (cross pairs; intra-slot pairs in
            // round 0) exceeds the rotation threshold on the fresh Gram: no step would rotate then
            // (late sweeps; the CTA still does the C·V = C copy of the systolic shift)
            bool work;
            {
                bool need = false;
                for (int e = tid; e < NC * NC; e += Cfg::NT) {
                    const int x = e / NC, y = e - x * NC;
                    if (x < y && (round == 0 || (x < BW) != (y < BW))) {
                        const double g = Gs[x * LDG + y], a = Gs[x * LDG + x], b = Gs[y * LDG + y];
                        need = need || (g * g > tol2 * a * b);
                    }
                }
                work = __syncthreads_or(need) != 0;
            }
            if (work) {
                int rot = 0;
                float mrel = 0.f;
                for (int st = (round == 0 ? 0 : BW - 1); st < NC - 1; ++st) {
                    const double *G0 = Gs + gi * NC * LDG;
                    const double *V0 = Vs + gi * NC * LDG;
                    double *G1 = Gs + (gi ^ 1) * NC * LDG;
                    double *V1 = Vs + (gi ^ 1) * NC * LDG;
                    double cw, sw;
                    {
                        const int pq = ptab[st * (NC / 2) + lane % (NC / 2)];
                        const int p = pq & 255, q = pq >> 8;
                        rot |= pair_rotation(G0[p * LDG + p], G0[q * LDG + q], G0[p * LDG + q], tol2, cw, sw, mrel);
                    }
#pragma unroll
                    for (int j = 0; j < NC * NC / Cfg::NT; ++j) {
                        const int e = tid + Cfg::NT * j;
                        const int x = e / NC, y = e - x * NC;
                        const int tx = tab[st * NC + x], ty = tab[st * NC + y];
                        const int xb = tx & 255, yb = ty & 255;
                        const double cxx = __shfl_sync(0xffffffffu, cw, (tx >> 8) & 255);
                        const double sx0 = __shfl_sync(0xffffffffu, sw, (tx >> 8) & 255);
                        const double cyy = __shfl_sync(0xffffffffu, cw, (ty >> 8) & 255);
                        const double sy0 = __shfl_sync(0xffffffffu, sw, (ty >> 8) & 255);
                        // C'_p = c C_p - s C_q,  C'_q = s C_p + c C_q
                        const double sxx = (tx >> 16) ? -sx0 : sx0, syy = (ty >> 16) ? -sy0 : sy0;
                        const double g = cxx * (cyy * G0[x * LDG + y] + syy * G0[x * LDG + yb]) +
                                         sxx * (cyy * G0[xb * LDG + y] + syy * G0[xb * LDG + yb]);
                        G1[x * LDG + y] = g;
                        V1[x * LDG + y] = V0[x * LDG + y] * cyy + V0[x * LDG + yb] * syy;
                    }
                    __syncthreads();
                    gi ^= 1;
                }
                if (rot) rot_sh = 1;   // benign races: every writer stores 1 / a larger value
                if (lane == 0 && mrel > 0.f) atomicMax(&mrel_sh, __float_as_int(mrel));
            }
            // ---- 3. C·V on the tensor cores, stored into the next-round buffers
            {
                const double *V = Vs + gi * NC * LDG;
                double *nxt_local = bufs + (cur ^ 1) * NC * ldc;
                double *dstA, *dstB;
                if (ncta == 1) { dstA = nxt_local; dstB = nxt_local + blk; }
                else if (c == 0) { dstA = cluster.map_shared_rank(nxt_local, 1) + blk; dstB = nxt_local + blk; }
                else {
                    dstA = cluster.map_shared_rank(nxt_local, c - 1);
                    dstB = (c + 1 < ncta) ? cluster.map_shared_rank(nxt_local, c + 1) + blk : nxt_local;
                }
                // a warp takes two 8-row tiles at a time and all NC/8 column tiles: the row fragments
                // are loaded once per k-step and 2·NC/8 independent DMMA chains overlap their latency
                constexpr int NJ = NC / 8;
                const int nit = m8 / 8;
                for (int it0 = warp; it0 < nit; it0 += 16) {
                    const bool two = it0 + 8 < nit;        // warp-uniform
                    double acc[2][NJ][2];
#pragma unroll
                    for (int h = 0; h < 2; ++h)
#pragma unroll
                        for (int jt = 0; jt < NJ; ++jt) acc[h][jt][0] = acc[h][jt][1] = 0.0;
#pragma unroll
                    for (int k0 = 0; k0 < NC; k0 += 4) {
                        const double *cr = C + ldc * (k0 + (lane & 3)) + (lane >> 2);
                        const double a0 = cr[8 * it0];
                        const double a1 = two ? cr[8 * (it0 + 8)] : 0.0;
#pragma unroll
                        for (int jt = 0; jt < NJ; ++jt) {
                            const double b = V[(k0 + (lane & 3)) * LDG + 8 * jt + (lane >> 2)];
                            dmma884(acc[0][jt][0], acc[0][jt][1], a0, b);
                            if (two) dmma884(acc[1][jt][0], acc[1][jt][1], a1, b);
                        }
                    }
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        if (h == 1 && !two) break;
                        const int row = 8 * (it0 + 8 * h) + (lane >> 2);
#pragma unroll
                        for (int jt = 0; jt < NJ; ++jt) {
                            const int col = 8 * jt + 2 * (lane & 3);   // col, col+1 in the same slot (BW % 8 == 0)
                            double *dst = (col < BW) ? dstA + ldc * col : dstB + ldc * (col - BW);
                            dst[row] = acc[h][jt][0];
                            dst[row + ldc] = acc[h][jt][1];
                        }
                    }
                }
            }
            cluster.sync();
            cur ^= 1;
        }
        // convergence: no rotation anywhere, or the largest relative off-diagonal rotated in this
        // sweep was below `early` (Jacobi converges quadratically: the next sweep would start
        // from ~early², below the rotation threshold)
        if (tid == 0 && rot_sh) atomicOr(cluster.map_shared_rank(&flags[sweep & 1], 0), 1);
        if (tid == 0 && mrel_sh) atomicMax(cluster.map_shared_rank(&mflags[sweep & 1], 0), mrel_sh);
        cluster.sync();
        const int any = *cluster.map_shared_rank(&flags[sweep & 1], 0);
        const float mx = __int_as_float(*cluster.map_shared_rank(&mflags[sweep & 1], 0));
        if (c == 0 && tid == 0) { flags[(sweep + 1) & 1] = 0; mflags[(sweep + 1) & 1] = 0; }
        cluster.sync();
        if (!any || mx < early) break;
    }
    {
        const int tt = t % (nb - 1);
        const int ba = (c == 0) ? tt : (tt + c) % (nb - 1);
        const int bb = (c == 0) ? nb - 1 : (tt - c + (nb - 1)) % (nb - 1);
        const double *C = bufs + cur * NC * ldc;
        for (int h = 0; h < 2; ++h) {
            const int b = h ? bb : ba;
            for (int idx = tid; idx < BW * m; idx += Cfg::NT) {
                const int jl = idx / m, i = idx - jl * m;
                const int col = b * BW + jl;
                if (col < n) A[i + (int64_t)m * col] = C[h * blk + i + ldc * jl];
            }
        }
    }
    if (c == 0 && tid == 0 && sweeps_out) *sweeps_out = sweep + 1;
}

template <int NC>
static bool launch_gram(int m, int n, double *T, int *sweeps, cudaStream_t st, float tol, float early) {
    using Cfg = GramCfg<NC>;
    int nb = (int)cdiv(n, Cfg::BW);
    nb += nb & 1;
    if (nb < 2) nb = 2;
    const int ncta = nb / 2;
    if (ncta > 16) return false;
    const size_t smem = Cfg::smem(m);
    if (smem > 220 * 1024) return false;
    auto kern = jacobi_gram_kernel<NC>;
    set_max_smem(kern);
    if (ncta > 8) SSA_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(ncta);
    cfg.blockDim = dim3(Cfg::NT);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = ncta; attr[0].val.clusterDim.y = 1; attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr; cfg.numAttrs = 1;
    int max_sweeps = 60;
    SSA_CUDA(cudaLaunchKernelEx(&cfg, kern, m, n, nb, T, tol, early, max_sweeps, sweeps));
    after_launch("jacobi_gram");
    return true;
}

template <int MR, int BW>
static bool launch_cluster(int m, int n, double *T, int *sweeps, cudaStream_t st, float tol) {
    int nb = (int)cdiv(n, BW);
    nb += nb & 1;
    if (nb < 2) nb = 2;
    const int ncta = nb / 2;
    if (ncta > 16) return false;
    const size_t smem = sizeof(double) * (size_t)(m | 1) * BW * 4;
    if (smem > 200 * 1024) return false;
    auto kern = jacobi_cluster_kernel<MR, BW>;
    set_max_smem(kern);
    if (ncta > 8) SSA_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(ncta);
    cfg.blockDim = dim3(32 * BW);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = ncta; attr[0].val.clusterDim.y = 1; attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr; cfg.numAttrs = 1;
    int max_sweeps = 60;
    SSA_CUDA(cudaLaunchKernelEx(&cfg, kern, m, n, nb, T, tol, max_sweeps, sweeps));
    after_launch("jacobi_cluster");
    return true;
}

// prefer the cluster kernel; fall back to the cooperative-grid kernel for large n
static bool jacobi_try_cluster(int m, int n, double *T, int *sweeps, cudaStream_t st, float tol, float early) {
    if (launch_gram<16>(m, n, T, sweeps, st, tol, early)) return true;
    if (launch_gram<32>(m, n, T, sweeps, st, tol, early)) return true;
    if (m <= 128) return n <= 256 ? launch_cluster<4, 8>(m, n, T, sweeps, st, tol) : launch_cluster<4, 16>(m, n, T, sweeps, st, tol);
    if (m <= 192) return n <= 256 ? launch_cluster<6, 8>(m, n, T, sweeps, st, tol) : launch_cluster<6, 16>(m, n, T, sweeps, st, tol);
    if (m <= 256) return n <= 256 ? launch_cluster<8, 8>(m, n, T, sweeps, st, tol) : launch_cluster<8, 16>(m, n, T, sweeps, st, tol);
    if (m <= 512) return n <= 256 ? launch_cluster<16, 8>(m, n, T, sweeps, st, tol) : launch_cluster<16, 16>(m, n, T, sweeps, st, tol);
    return false;
}

void jacobi_svd_blocked(int m, int n, double *T, int *counters, int *sweeps, cudaStream_t st, double tol_d,
                        double early) {
    const float tol = (float)tol_d;
    if (jacobi_try_cluster(m, n, T, sweeps, st, tol, (float)early)) return;
    int nb = (int)cdiv(n, kBW);
    nb += nb & 1;
    if (nb < 2) nb = 2;
    const int grid = nb / 2;
    const size_t smem = sizeof(double) * (size_t)(m | 1) * 2 * kBW;
    SSA_REQUIRE(grid <= num_sms() && smem <= 200 * 1024 && m <= 32 * 24, SSA_ERR_ARG,
                "projected matrix too large for the device Jacobi");
    SSA_CUDA(cudaMemsetAsync(counters, 0, sizeof(int) * 64, st));
    int max_sweeps = 60;
    float tol_arg = tol;
    void *args[] = {&m, &n, &nb, &T, &tol_arg, &max_sweeps, &counters, &sweeps};
    void *kern = m <= 32 * 4 ? (void *)jacobi_block_kernel<4>
               : m <= 32 * 8 ? (void *)jacobi_block_kernel<8>
               : m <= 32 * 16 ? (void *)jacobi_block_kernel<16> : (void *)jacobi_block_kernel<24>;
    set_max_smem(kern);
    SSA_CUDA(cudaLaunchCooperativeKernel(kern, dim3(grid), dim3(32 * kBW), args, smem, st));
    after_launch("jacobi_block");
}

// After the Jacobi: nrm[j] = ||A_j|| (the singular values) and W = T0ᵀ·A (n x n), from which
// the caller forms the right vectors z_j = T0ᵀ y_j / θ_j = W[:, j] / θ_j² without a host
// pass over T.  Block j: warp 0 the norm, then the 8 warps over the rows i of W[:, j].
__global__ void __launch_bounds__(256)
ritz_tn_kernel(int m, int n, const double *__restrict__ T0, const double *__restrict__ A, double *__restrict__ W,
               double *__restrict__ nrm) {
    const int j = blockIdx.x, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const double *aj = A + (int64_t)m * j;
    if (warp == 0) {
        double s = 0.0;
        for (int k = lane; k < m; k += 32) s = fma(aj[k], aj[k], s);
        for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (lane == 0) nrm[j] = sqrt(s);
    }
    for (int i = warp; i < n; i += 8) {
        const double *ti = T0 + (int64_t)m * i;
        double s = 0.0;
        for (int k = lane; k < m; k += 32) s = fma(ti[k], aj[k], s);
        for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (lane == 0) W[i + (int64_t)n * j] = s;
    }
}

void ritz_tn(int m, int n, const double *T0, const double *A, double *W, double *nrm, cudaStream_t st) {
    ritz_tn_kernel<<<n, 256, 0, st>>>(m, n, T0, A, W, nrm);
    after_launch("ritz_tn");
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
        jacobi_svd_blocked(m, n, d.as<double>(), dc, ds, nullptr, 1e-12, 1e-6);
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
