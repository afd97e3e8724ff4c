// FFT circular-correlation path for the trajectory-operator products and the
// diagonal averaging (the method of Alg. 1/3/5,
// P:3643-3665, re-derived for the device).
//
// Every product is one 2-D circular correlation of the image with a box array
// evaluated on another box (reading Q1/Q2: the same formula serves X·V and XᵀU,
// only the scatter box and the gather box swap):
//
//     out[p] = Σ_d x[p + d] a[d]  =  IDFT2( X̂ ⊙ conj(DFT2(a)) )[p]      (p in the output box)
//
// on an Mx x My grid (powers of two, Mx >= Nx, My >= Ny, so the gathered cells
// never wrap).  The averaging numerator is a full 2-D convolution summed over a
// group: num_g = IDFT2( Σ_{i∈I_g} σ_i DFT2(Ψ_i) ⊙ DFT2(Φ_i) ) (no conjugate).
//
// Three passes over HBM, each a batch of shared-memory Stockham FFTs
// (radix 8 with one radix-2/4 stage) with zero-padding and output pruning:
//   A  x-direction DFT of the input box columns (real -> half spectrum, Hx = Mx/2+1
//      frequencies), written transposed as A[j][fx][col] so that B reads rows;
//   B  per (j, fx) row: y-direction DFT of the ny_in nonzero entries, multiply by
//      conj(X̂[fx, :]) (products) or accumulate Ψ̂·Φ̂ over a group (averaging),
//      inverse y-DFT, keep the ny_out rows of the output box;
//   C  per output column: Hermitian completion of the half spectrum, inverse
//      x-DFT, keep the output box rows, scale, gather into the compact order
//      (or divide by the hit counts 𝕎 for the averaging).
// X̂ = DFT2(image) is computed once per plan (it "does not depend on L").
#include <cmath>
#include <cstdlib>
#include <vector>

#include "common.h"
#include "fft_reg.h"
#include "kernels.h"
#include "plan.h"

namespace ssa {

template <typename T> struct cplx { T x, y; };
template <typename T> __device__ __forceinline__ cplx<T> cadd(cplx<T> a, cplx<T> b) { return {a.x + b.x, a.y + b.y}; }
template <typename T> __device__ __forceinline__ cplx<T> csub(cplx<T> a, cplx<T> b) { return {a.x - b.x, a.y - b.y}; }
template <typename T> __device__ __forceinline__ cplx<T> cmul(cplx<T> a, cplx<T> b) {
    return {a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x};
}
template <typename T> __device__ __forceinline__ cplx<T> cmulconj(cplx<T> a, cplx<T> b) {   // a * conj(b)
    return {a.x * b.x + a.y * b.y, a.y * b.x - a.x * b.y};
}
// multiply by DIR*i  (DIR = -1 forward, +1 inverse)
template <typename T, int DIR> __device__ __forceinline__ cplx<T> mul_i(cplx<T> a) {
    return DIR > 0 ? cplx<T>{-a.y, a.x} : cplx<T>{a.y, -a.x};
}

__device__ __forceinline__ void sincospi_t(float a, float *s, float *c) { sincospif(a, s, c); }
__device__ __forceinline__ void sincospi_t(double a, double *s, double *c) { sincospi(a, s, c); }

template <typename T, int DIR> __device__ __forceinline__ void dft2(cplx<T> *v) {
    const cplx<T> a = v[0], b = v[1];
    v[0] = cadd(a, b); v[1] = csub(a, b);
}
template <typename T, int DIR> __device__ __forceinline__ void dft4(cplx<T> *v) {
    const cplx<T> t0 = cadd(v[0], v[2]), t1 = csub(v[0], v[2]);
    const cplx<T> t2 = cadd(v[1], v[3]), t3 = mul_i<T, DIR>(csub(v[1], v[3]));
    v[0] = cadd(t0, t2); v[2] = csub(t0, t2);
    v[1] = cadd(t1, t3); v[3] = csub(t1, t3);
}
template <typename T, int DIR> __device__ __forceinline__ void dft8(cplx<T> *v) {
    cplx<T> e[4] = {v[0], v[2], v[4], v[6]}, o[4] = {v[1], v[3], v[5], v[7]};
    dft4<T, DIR>(e); dft4<T, DIR>(o);
    const T h = (T)0.70710678118654752440;
    // o[k] *= exp(DIR*2πi k/8)
    o[1] = cplx<T>{h * (o[1].x - (T)DIR * o[1].y), h * (o[1].y + (T)DIR * o[1].x)};
    o[2] = mul_i<T, DIR>(o[2]);
    o[3] = cplx<T>{h * (-o[3].x - (T)DIR * o[3].y), h * (-o[3].y + (T)DIR * o[3].x)};
#pragma unroll
    for (int k = 0; k < 4; ++k) { v[k] = cadd(e[k], o[k]); v[k + 4] = csub(e[k], o[k]); }
}

// Shared-memory index padding: one spare element per 16 keeps the radix-8 Stockham
// stores (stride R) and the transposed column accesses free of bank conflicts.
__device__ __forceinline__ int sp(int i) { return i + (i >> 4); }
__host__ __device__ constexpr size_t sp_size(size_t n) { return n + (n >> 4) + 1; }

// Twiddles: per transform size 2^LG the plan keeps one table per radix-8 stage with span
// NS = 2^LGS > 1 — w1[k] = exp(−2πi k / (8·NS)), k < NS (fp64-accurate, rounded to T) — concatenated
// (stab_off(LG, LGS) = position of the stage's table; 584 entries for LG = 12).  Each CTA stages
// the table of its transform size in shared memory; a butterfly reads w1 once and forms
// w2 = w1², w3 = w2·w1, w4 = w2², w5..w7 = w4·w1..w3 (the previous two-level table cost three
// lookups with a complex multiply each: ~20% of the stage's instructions, ncu).
__host__ __device__ constexpr int stab_off(int LG, int LGS) {
    int off = 0;
    for (int l = LG % 3; l < LGS; l += 3)
        if (l > 0) off += 1 << l;
    return off;
}
__host__ __device__ constexpr size_t stab_count(int lg) { return (size_t)stab_off(lg, lg); }
template <typename T>
__device__ __forceinline__ void stage_stab(cplx<T> *tws, const cplx<T> *__restrict__ g, int lg) {
    const int n = (int)stab_count(lg);
    for (int i = threadIdx.x; i < n; i += blockDim.x) tws[i] = g[i];
}

// One Stockham radix-R stage for `nbatch` transforms of length N = 2^LGN stored back to back
// (padded indices); NS = 2^LGS is the current span.  Sizes are template constants so the index
// arithmetic folds (the generic version spent half of its instructions on integer address
// math, ncu); loads use one padded base plus constant strides, and the R-1 twiddles of a
// butterfly come from one per-stage table lookup and 6 multiplies.
template <typename T, int DIR, int R, int LGN, int LGS>
__device__ __forceinline__ void stage_t(const cplx<T> *__restrict__ x, cplx<T> *__restrict__ y, int nbatch,
                                        const cplx<T> *__restrict__ tws, int lgtw) {
    constexpr int LR = R == 2 ? 1 : (R == 4 ? 2 : 3);
    constexpr int N = 1 << LGN, NBF = N >> LR, LGB = LGN - LR, NS = 1 << LGS;
    static_assert(NS == 1 || R == 8, "only the first stage may be radix 2/4");
    for (int b = threadIdx.x; b < (nbatch << LGB); b += blockDim.x) {
        const int t = b >> LGB, j = b & (NBF - 1);
        const int a = t * N + j;
        cplx<T> v[R];
        if constexpr (NBF % 16 == 0) {
            const int pa = sp(a);
#pragma unroll
            for (int r = 0; r < R; ++r) v[r] = x[pa + r * (NBF + NBF / 16)];
        } else {
#pragma unroll
            for (int r = 0; r < R; ++r) v[r] = x[sp(a + r * NBF)];
        }
        const int k = j & (NS - 1);
        if constexpr (NS > 1) {
            // radix-8 stages only (the radix-2/4 stage, if any, is the first one: NS = 1)
            cplx<T> w1 = tws[stab_off(LGN, LGS) + k];
            if (DIR > 0) w1.y = -w1.y;
            const cplx<T> w2 = cmul(w1, w1);
            const cplx<T> w3 = cmul(w2, w1);
            v[1] = cmul(v[1], w1); v[2] = cmul(v[2], w2); v[3] = cmul(v[3], w3);
            if constexpr (R == 8) {
                const cplx<T> w4 = cmul(w2, w2);
                v[4] = cmul(v[4], w4);
                v[5] = cmul(v[5], cmul(w4, w1));
                v[6] = cmul(v[6], cmul(w4, w2));
                v[7] = cmul(v[7], cmul(w4, w3));
            }
        }
        if constexpr (R == 2) dft2<T, DIR>(v);
        else if constexpr (R == 4) dft4<T, DIR>(v);
        else dft8<T, DIR>(v);
        const int base = t * N + (j - k) * R + k;
        if constexpr (NS % 16 == 0) {
            const int pb = sp(base);
#pragma unroll
            for (int r = 0; r < R; ++r) y[pb + r * (NS + NS / 16)] = v[r];
        } else {
#pragma unroll
            for (int r = 0; r < R; ++r) y[sp(base + r * NS)] = v[r];
        }
    }
}

template <typename T, int DIR, int LG, int LGS>
__device__ __forceinline__ cplx<T> *stages_from(cplx<T> *x, cplx<T> *y, int nbatch, const cplx<T> *__restrict__ tws,
                                                int lgtw) {
    if constexpr (LGS >= LG) {
        return x;
    } else {
        stage_t<T, DIR, 8, LG, LGS>(x, y, nbatch, tws, lgtw);
        __syncthreads();
        return stages_from<T, DIR, LG, LGS + 3>(y, x, nbatch, tws, lgtw);
    }
}

// Batched ping-pong FFT of nbatch transforms of length 2^LG in shared memory (padded
// indices); returns the buffer that holds the result.  All threads of the CTA take part;
// the caller has synchronised before the call.
template <typename T, int DIR, int LG>
__device__ __forceinline__ cplx<T> *fft_batch_t(cplx<T> *x, cplx<T> *y, int nbatch, const cplx<T> *__restrict__ tws,
                                                int lgtw) {
    constexpr int REM = LG % 3;
    if constexpr (REM == 1) {
        stage_t<T, DIR, 2, LG, 0>(x, y, nbatch, tws, lgtw);
        __syncthreads();
        return stages_from<T, DIR, LG, 1>(y, x, nbatch, tws, lgtw);
    } else if constexpr (REM == 2) {
        stage_t<T, DIR, 4, LG, 0>(x, y, nbatch, tws, lgtw);
        __syncthreads();
        return stages_from<T, DIR, LG, 2>(y, x, nbatch, tws, lgtw);
    } else {
        return stages_from<T, DIR, LG, 0>(x, y, nbatch, tws, lgtw);
    }
}

template <typename T, int DIR>
__device__ cplx<T> *fft_batch(cplx<T> *x, cplx<T> *y, int lg, int nbatch, const cplx<T> *__restrict__ tws, int lgtw) {
    switch (lg) {
    case 0: return x;   // length-1 transforms are the identity
    case 1: return fft_batch_t<T, DIR, 1>(x, y, nbatch, tws, lgtw);
    case 2: return fft_batch_t<T, DIR, 2>(x, y, nbatch, tws, lgtw);
    case 3: return fft_batch_t<T, DIR, 3>(x, y, nbatch, tws, lgtw);
    case 4: return fft_batch_t<T, DIR, 4>(x, y, nbatch, tws, lgtw);
    case 5: return fft_batch_t<T, DIR, 5>(x, y, nbatch, tws, lgtw);
    case 6: return fft_batch_t<T, DIR, 6>(x, y, nbatch, tws, lgtw);
    case 7: return fft_batch_t<T, DIR, 7>(x, y, nbatch, tws, lgtw);
    case 8: return fft_batch_t<T, DIR, 8>(x, y, nbatch, tws, lgtw);
    case 9: return fft_batch_t<T, DIR, 9>(x, y, nbatch, tws, lgtw);
    case 10: return fft_batch_t<T, DIR, 10>(x, y, nbatch, tws, lgtw);
    case 11: return fft_batch_t<T, DIR, 11>(x, y, nbatch, tws, lgtw);
    case 12: return fft_batch_t<T, DIR, 12>(x, y, nbatch, tws, lgtw);
    default: return fft_batch_t<T, DIR, 13>(x, y, nbatch, tws, lgtw);
    }
}

// ---------------------------------------------------------------------------
// Pass A: x-direction DFT of box columns.
//   input : in[map(ix, col) + ld * j] (compact, map = box -> compact or -1), box bx x by,
//           optional per-vector scale (σ_i for the averaging); the image when ld = 0 and map = null
//   output: A[(j * Hx + fx) * by + col], fx < Hx
// grid: (ceil(by / CB), k), CB columns per CTA.
// ---------------------------------------------------------------------------
template <typename T, int MAXT>
__global__ void __launch_bounds__(MAXT, sizeof(T) == 4 ? (MAXT <= 256 ? 6 : 3) : (MAXT <= 256 ? 4 : 2))
fft_pass_a(const T *__restrict__ in, int64_t ld, const int *__restrict__ map, int bx, int by, int jsel_n,
           const int *__restrict__ jsel, const double *__restrict__ scale, int lgx, int CB, cplx<T> *__restrict__ A,
           int lda, const cplx<T> *__restrict__ tw, int lgtw) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int Mx = 1 << lgx, Hx = Mx / 2 + 1;
    cplx<T> *b0 = reinterpret_cast<cplx<T> *>(smem_raw);
    cplx<T> *b1 = b0 + sp_size((size_t)(CB >> 1) * Mx);   // CB/2 complex transforms
    cplx<T> *tws = b1 + sp_size((size_t)(CB >> 1) * Mx);
    stage_stab(tws, tw, lgtw);
    // two real columns per complex transform (NT = CB/2 transforms): z = x_a + i·x_b,
    // X_a[f] = (Z[f] + conj Z[-f]) / 2,  X_b[f] = (Z[f] - conj Z[-f]) / (2i)
    const int NT = CB >> 1;
    const int col0 = blockIdx.x * CB;
    const int jo = blockIdx.y;                       // output vector slot
    const int j = jsel ? jsel[jo] : jo;             // input vector index
    const T sc = scale ? (T)scale[j] : T(1);
    const int ncol = min(CB, by - col0);
    #pragma unroll 8
    for (int idx = threadIdx.x; idx < NT * Mx; idx += blockDim.x) {
        const int t = idx >> lgx, ix = idx & (Mx - 1);
        T v[2] = {T(0), T(0)};
        if (ix < bx) {
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int c = 2 * t + h;
                if (c < ncol) {
                    const int64_t box = ix + (int64_t)bx * (col0 + c);
                    const int64_t ci = map ? (int64_t)map[box] : box;
                    if (ci >= 0) v[h] = sc * in[ci + ld * j];
                }
            }
        }
        b0[sp(idx)] = cplx<T>{v[0], v[1]};
    }
    __syncthreads();
    cplx<T> *res = fft_batch<T, -1>(b0, b1, lgx, NT, tws, lgtw);
    const int lcb = __ffs(CB) - 1;
    // transposed write: consecutive threads -> consecutive columns
    #pragma unroll 8
    for (int idx = threadIdx.x; idx < Hx * CB; idx += blockDim.x) {
        const int fx = idx >> lcb, c = idx & (CB - 1);   // CB is a power of two
        if (c >= ncol) continue;
        const int t = c >> 1;
        const cplx<T> z = res[sp(t * Mx + fx)], zm = res[sp(t * Mx + ((Mx - fx) & (Mx - 1)))];
        const cplx<T> out = (c & 1) ? cplx<T>{(z.y + zm.y) * T(0.5), (zm.x - z.x) * T(0.5)}
                                    : cplx<T>{(z.x + zm.x) * T(0.5), (z.y - zm.y) * T(0.5)};
        A[((int64_t)jo * Hx + fx) * lda + col0 + c] = out;
    }
}

// ---------------------------------------------------------------------------
// Pass B (products): per (j, fx): y-DFT of A row (ny_in entries), multiply by
// conj, inverse y-DFT, keep ny_out entries.  mode 0: Y = X̂ ⊙ conj(Â) (correlation);
// mode 1: forward only, write all My entries (plan-time X̂).
// grid: (ceil(Hx / RB), k)
// ---------------------------------------------------------------------------
template <typename T, int MAXT>
__global__ void __launch_bounds__(MAXT, sizeof(T) == 4 ? (MAXT <= 256 ? 6 : 3) : (MAXT <= 256 ? 4 : 2))
fft_pass_b(const cplx<T> *__restrict__ A, int ny_in, int lda, int Hx, int lgy, int RB, const cplx<T> *__restrict__ Xh,
           int mode, cplx<T> *__restrict__ B, int ny_out, int ldb, const cplx<T> *__restrict__ tw, int lgtw) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int My = 1 << lgy;
    cplx<T> *b0 = reinterpret_cast<cplx<T> *>(smem_raw);
    cplx<T> *b1 = b0 + sp_size((size_t)RB * My);
    cplx<T> *tws = b1 + sp_size((size_t)RB * My);
    stage_stab(tws, tw, lgtw);
    // grid (k, Hx/RB): the k CTAs that multiply by the same X̂ rows run back to back, so
    // X̂ stays in L2 while the (much larger) A stream passes (c5: 4.3 GB of X̂ re-reads from
    // DRAM with the transposed grid order, ncu)
    const int fx0 = blockIdx.y * RB;
    const int j = blockIdx.x;
    const int nrow = min(RB, Hx - fx0);
    // X̂ rows of this CTA: fetched asynchronously into shared memory at the start so their L2
    // latency overlaps the forward transforms (ncu: the multiply waited on these loads)
    cplx<T> *xs = reinterpret_cast<cplx<T> *>((reinterpret_cast<uintptr_t>(tws + stab_count(lgtw)) + 15) & ~uintptr_t(15));
    if (mode == 0) {
        constexpr int PER = 16 / sizeof(cplx<T>);            // complex values per 16-B copy
        const uint32_t xs_u = (uint32_t)__cvta_generic_to_shared(xs);
        for (int q = threadIdx.x; q < (RB * My) / PER; q += blockDim.x) {
            const int idx = q * PER, rr = idx >> lgy;
            const int bytes = rr < nrow ? 16 : 0;
            const cplx<T> *src = Xh + (int64_t)(fx0 + (rr < nrow ? rr : 0)) * My + (idx & (My - 1));
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(xs_u + (uint32_t)(16 * q)), "l"(src),
                         "r"(bytes));
        }
        asm volatile("cp.async.commit_group;");
    }
    #pragma unroll 8
    for (int idx = threadIdx.x; idx < RB * My; idx += blockDim.x) {
        const int rr = idx >> lgy, y = idx & (My - 1);
        cplx<T> v{T(0), T(0)};
        if (rr < nrow && y < ny_in) v = A[((int64_t)j * Hx + fx0 + rr) * lda + y];
        b0[sp(idx)] = v;
    }
    __syncthreads();
    cplx<T> *res = fft_batch<T, -1>(b0, b1, lgy, RB, tws, lgtw);
    cplx<T> *oth = (res == b0) ? b1 : b0;
    if (mode == 1) {
        #pragma unroll 8
        for (int idx = threadIdx.x; idx < RB * My; idx += blockDim.x) {
            const int rr = idx >> lgy, y = idx & (My - 1);
            if (rr < nrow) B[((int64_t)j * Hx + fx0 + rr) * My + y] = res[sp(idx)];
        }
        return;
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    __syncthreads();
    #pragma unroll 8
    for (int idx = threadIdx.x; idx < RB * My; idx += blockDim.x) res[sp(idx)] = cmulconj(xs[idx], res[sp(idx)]);
    __syncthreads();
    cplx<T> *out = fft_batch<T, +1>(res, oth, lgy, RB, tws, lgtw);
    #pragma unroll 8
    for (int idx = threadIdx.x; idx < RB * ny_out; idx += blockDim.x) {
        const int rr = idx / ny_out, y = idx - rr * ny_out;
        if (rr < nrow) B[((int64_t)j * Hx + fx0 + rr) * ldb + y] = out[sp(rr * My + y)];
    }
}

// Pass B (averaging): per (g, fx): Σ_{i∈I_g} DFT_y(AU_i row) ⊙ DFT_y(AV_i row), inverse, keep ny rows.
template <typename T, int MAXT>
__global__ void __launch_bounds__(MAXT, sizeof(T) == 4 ? (MAXT <= 256 ? 6 : 3) : (MAXT <= 256 ? 4 : 2))
fft_pass_b_conv(const cplx<T> *__restrict__ AU, int ly, int ldu, const cplx<T> *__restrict__ AV, int ky, int ldv,
                const int *grp_off, const int *grp_idx, const int *slot, int Hx, int lgy, int RB,
                cplx<T> *__restrict__ B, int ny_out, int ldb, const cplx<T> *__restrict__ tw, int lgtw) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int My = 1 << lgy;
    const size_t bs = sp_size((size_t)RB * My);
    cplx<T> *acc = reinterpret_cast<cplx<T> *>(smem_raw);
    cplx<T> *u0 = acc + bs;
    cplx<T> *u1 = u0 + bs;
    cplx<T> *v0 = u1 + bs;
    cplx<T> *v1 = v0 + bs;
    cplx<T> *tws = v1 + bs;
    stage_stab(tws, tw, lgtw);
    const int fx0 = blockIdx.x * RB;
    const int g = blockIdx.y;
    const int nrow = min(RB, Hx - fx0);
    for (int idx = threadIdx.x; idx < RB * My; idx += blockDim.x) acc[sp(idx)] = cplx<T>{T(0), T(0)};
    for (int t = grp_off[g]; t < grp_off[g + 1]; ++t) {
        const int s = slot[grp_idx[t]];
        __syncthreads();
        #pragma unroll 8
        for (int idx = threadIdx.x; idx < RB * My; idx += blockDim.x) {
            const int rr = idx >> lgy, y = idx & (My - 1);
            cplx<T> a{T(0), T(0)}, b{T(0), T(0)};
            if (rr < nrow) {
                if (y < ly) a = AU[((int64_t)s * Hx + fx0 + rr) * ldu + y];
                if (y < ky) b = AV[((int64_t)s * Hx + fx0 + rr) * ldv + y];
            }
            u0[sp(idx)] = a; v0[sp(idx)] = b;
        }
        __syncthreads();
        cplx<T> *ru = fft_batch<T, -1>(u0, u1, lgy, RB, tws, lgtw);
        cplx<T> *rv = fft_batch<T, -1>(v0, v1, lgy, RB, tws, lgtw);
        for (int idx = threadIdx.x; idx < RB * My; idx += blockDim.x)
            acc[sp(idx)] = cadd(acc[sp(idx)], cmul(ru[sp(idx)], rv[sp(idx)]));
    }
    __syncthreads();
    cplx<T> *out = fft_batch<T, +1>(acc, u0, lgy, RB, tws, lgtw);
    #pragma unroll 8
    for (int idx = threadIdx.x; idx < RB * ny_out; idx += blockDim.x) {
        const int rr = idx / ny_out, y = idx - rr * ny_out;
        if (rr < nrow) B[((int64_t)g * Hx + fx0 + rr) * ldb + y] = out[sp(rr * My + y)];
    }
}

// ---------------------------------------------------------------------------
// Pass C: per output column y: Hermitian completion, inverse x-DFT, keep ox rows.
//   products : out[omap(x, y) + ldo * j] = Re(...) * inv   (omap: box -> compact or -1)
//   averaging: out[x + ldo*y + stride*j] = Re(...) * inv / w  on w > 0, NaN elsewhere
// grid: (ceil(oy / CB), k)
// ---------------------------------------------------------------------------
template <typename T, int MAXT>
__global__ void __launch_bounds__(MAXT, sizeof(T) == 4 ? (MAXT <= 256 ? 6 : 3) : (MAXT <= 256 ? 4 : 2))
fft_pass_c(const cplx<T> *__restrict__ B, int oy, int ldb, int Hx, int lgx, int CB, int ox, T inv, T *__restrict__ out,
           int64_t ldo, const int *__restrict__ omap, const int *__restrict__ w, int64_t stride,
           const cplx<T> *__restrict__ tw, int lgtw, const cplx<T> *__restrict__ Afu, int ny_in, int lda,
           const cplx<T> *__restrict__ gk, int lgy) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int Mx = 1 << lgx;
    cplx<T> *b0 = reinterpret_cast<cplx<T> *>(smem_raw);
    cplx<T> *b1 = b0 + sp_size((size_t)(CB >> 1) * Mx);   // CB/2 complex transforms
    cplx<T> *tws = b1 + sp_size((size_t)(CB >> 1) * Mx);
    stage_stab(tws, tw, lgtw);
    // two output columns per complex inverse transform (NT = CB/2): Z = Y_a + i·Y_b over the
    // full spectrum (Hermitian completion of each half spectrum), Re z = y_a, Im z = y_b
    const int NT = CB >> 1, lnt = __ffs(NT) - 1;
    const int y0 = blockIdx.x * CB;
    const int j = blockIdx.y;
    const int ncol = min(CB, oy - y0);
    #pragma unroll 8
    for (int idx = threadIdx.x; idx < Hx * NT; idx += blockDim.x) {
        const int fx = idx >> lnt, t = idx & (NT - 1);   // NT is a power of two
        cplx<T> ya{T(0), T(0)}, yb{T(0), T(0)};
        if (Afu) {
            // pass B folded in (few rows on both sides, MSSA): the y-correlation with the image as
            // B[fx, y] = Σ_{y'} conj(A[fx, y']) · g[fx, (y + y') mod My], g = unnormalised inverse
            // y-DFT of the X̂ row (plan time)
            const int My = 1 << lgy;
            const cplx<T> *ar = Afu + ((int64_t)j * Hx + fx) * lda;
            const cplx<T> *gr = gk + (int64_t)fx * My;
            const int ya_i = y0 + 2 * t;
            for (int yp = 0; yp < ny_in; ++yp) {
                const cplx<T> a = ar[yp];
                if (2 * t < ncol) ya = cadd(ya, cmulconj(gr[(ya_i + yp) & (My - 1)], a));
                if (2 * t + 1 < ncol) yb = cadd(yb, cmulconj(gr[(ya_i + 1 + yp) & (My - 1)], a));
            }
        } else {
            const int64_t base = ((int64_t)j * Hx + fx) * ldb + y0 + 2 * t;
            if (2 * t < ncol) ya = B[base];
            if (2 * t + 1 < ncol) yb = B[base + 1];
        }
        if (fx == 0 || fx == Mx / 2) { ya.y = T(0); yb.y = T(0); }   // real signals: these bins are real
        b0[sp(t * Mx + fx)] = cplx<T>{ya.x - yb.y, ya.y + yb.x};
        if (fx > 0 && fx < Mx / 2) b0[sp(t * Mx + Mx - fx)] = cplx<T>{ya.x + yb.y, yb.x - ya.y};
    }
    __syncthreads();
    cplx<T> *res = fft_batch<T, +1>(b0, b1, lgx, NT, tws, lgtw);
    #pragma unroll 8
    for (int idx = threadIdx.x; idx < CB * ox; idx += blockDim.x) {
        const int c = idx / ox, x = idx - c * ox;
        if (c >= ncol) continue;
        const int y = y0 + c;
        const cplx<T> z = res[sp((c >> 1) * Mx + x)];
        const T v = ((c & 1) ? z.y : z.x) * inv;
        if (w) {
            const int wn = w[x + (int64_t)ox * y];
            out[(int64_t)j * stride + x + ldo * y] = wn > 0 ? v / (T)wn : (T)NAN;
        } else {
            const int64_t box = x + (int64_t)ox * y;
            const int64_t oi = omap ? (int64_t)omap[box] : box;
            if (oi >= 0) out[oi + ldo * j] = v;
        }
    }
}

// ---------------------------------------------------------------------------
struct FftOperator {
    int lgx = 0, lgy = 0, Mx = 0, My = 0, Hx = 0;
    int lgtw = 0;
    DevBuf stab_x, stab_y;   // per-stage twiddle tables for 2^lgx / 2^lgy point transforms
    DevBuf Xh;        // cplx[Hx][My]: DFT2 of the image
    DevBuf gk;        // cplx[Hx][My]: unnormalised inverse y-DFT of each X̂ row (small My: folded pass B)
    DevBuf rtw_x, rtw_y;     // twiddle tables of the register-resident radix-16 passes (fp32, fft_reg.cu)
    DevBuf lowcells;         // cells with 0 < w_n < w_max / 64 (averaging re-done by direct summation)
    int n_lowcells = -1;
    DevBuf bufA, bufB;
    size_t capA = 0, capB = 0;
};

static int ilog2_ceil(int64_t n) {
    int l = 0;
    while ((int64_t(1) << l) < n) ++l;
    return l;
}

bool fft_supported(const PlanImpl &p) {
    // shared-memory Stockham sizes: up to 8192 points (fp32) / 2048 along y and 4096 along x (fp64).
    // Bands (multi-GPU) are fine: the band's 𝔎 enters through the compaction map like any shape.
    const int lx = ilog2_ceil(p.nx), ly = ilog2_ceil(p.ny);
    return p.dt == SSA_F64 ? (lx <= 12 && ly <= 11) : (lx <= 13 && ly <= 13);
}

// transforms per CTA so that a CTA holds ~target complex points (2 buffers)
// threads per CTA: one radix-8 butterfly per thread per stage, 128..512 (long transforms get
// more threads: the stages are latency chains, so parallel butterflies shorten each one)
// (measured: 512 threads help short grids such as the c2 4096-point columns, 256 are better for
// grids of many waves such as c5 pass B, where occupancy hides the latency instead)
static int threads_for(int lg, int nb, int64_t nctas) {
    const int64_t cap = nctas >= 4 * (int64_t)num_sms() ? 256 : 512;
    return (int)std::min<int64_t>(cap, std::max<int64_t>(128, ((int64_t)nb << lg) / 8));
}

static int batch_for(int lg, int target) {
    return std::max(1, target >> lg);
}

template <typename T>
static size_t smem_ab(int lg, int nb, int /*unused*/) {
    return sizeof(cplx<T>) * (2 * sp_size((size_t)nb << lg) + stab_count(lg));
}

// Row stride of the intermediates A (by columns) and B (oy columns): rounded up to 4 complex
// values, so that rows start 32-B aligned and the transposed column accesses of passes A and C move
// 16-B / 32-B vectors (the padding columns are written by no pass and masked on every read)
static int row_ld(int n) { return (int)rup(n, 4); }

template <typename T>
static void pass_a(FftOperator &f, const T *in, int64_t ld, const int *map, int bx, int by, int k, const int *jsel,
                   const double *scale, cplx<T> *A, cudaStream_t st) {
    const int lda = row_ld(by);
    if constexpr (sizeof(T) == 4) {
        if (f.rtw_x.p) {
            rfft::pass_a(f.lgx, in, ld, map, bx, by, k, jsel, scale, reinterpret_cast<float2 *>(A), lda,
                         f.rtw_x.as<float2>(), st);
            return;
        }
    }
    const int CB = 2 * batch_for(f.lgx, 2048);   // real columns (two per complex transform)
    const size_t smem = smem_ab<T>(f.lgx, CB / 2, 0);
    const int nth = threads_for(f.lgx, CB / 2, cdiv(by, CB) * k);
    auto kern = nth <= 256 ? fft_pass_a<T, 256> : fft_pass_a<T, 512>;
    set_max_smem(kern);
    kern<<<dim3((unsigned)cdiv(by, CB), k), nth, smem, st>>>(in, ld, map, bx, by, k, jsel, scale, f.lgx, CB, A, lda,
                                                                        f.stab_x.as<cplx<T>>(), f.lgx);
    after_launch("fft_pass_a");
}

// B between pass B and pass C is blocked by pass C's column blocks when both run the register
// passes (fft_reg.cu boff); the Stockham passes use the row layout
static int b_blocking(const FftOperator &f) { return (f.rtw_x.p && f.rtw_y.p) ? rfft::cb_of(f.lgx) : 0; }
static size_t b_cols(const FftOperator &f, int oy) { return (size_t)rup(oy, std::max(4, b_blocking(f))); }

template <typename T>
static void pass_b(FftOperator &f, const cplx<T> *A, int ny_in, int k, int mode, cplx<T> *B, int ny_out, cudaStream_t st) {
    const int lda = row_ld(ny_in), ldb = mode == 1 ? f.My : row_ld(ny_out);
    if constexpr (sizeof(T) == 4) {
        if (f.rtw_y.p && mode == 0) {
            rfft::pass_b(f.lgy, reinterpret_cast<const float2 *>(A), ny_in, lda, f.Hx, k,
                         reinterpret_cast<const float2 *>(f.Xh.p), reinterpret_cast<float2 *>(B), ny_out, ldb,
                         b_blocking(f), f.rtw_y.as<float2>(), st);
            return;
        }
    }
    const int RB = batch_for(f.lgy, 2048);
    // + the CTA's X̂ rows (prefetched, mode 0)
    const size_t smem = smem_ab<T>(f.lgy, RB, 0) + sizeof(cplx<T>) * ((size_t)RB << f.lgy) + 16;
    const int nth = threads_for(f.lgy, RB, cdiv(f.Hx, RB) * k);
    auto kern = nth <= 256 ? fft_pass_b<T, 256> : fft_pass_b<T, 512>;
    set_max_smem(kern);
    kern<<<dim3(k, (unsigned)cdiv(f.Hx, RB)), nth, smem, st>>>(A, ny_in, lda, f.Hx, f.lgy, RB,
                                                                         f.Xh.as<cplx<T>>(), mode, B, ny_out, ldb,
                                                                         f.stab_y.as<cplx<T>>(), f.lgy);
    after_launch("fft_pass_b");
}

template <typename T>
// cs (products only): per-column factors; applied here by the register pass, else by scale_columns
static void pass_c(FftOperator &f, const cplx<T> *B, int oy, int k, int ox, T *out, int64_t ldo, const int *omap,
                   const int *w, int64_t stride, cudaStream_t st, const cplx<T> *Afu = nullptr, int ny_in = 0,
                   const double *cs = nullptr) {
    const int ldb = row_ld(oy), lda = row_ld(ny_in);
    if constexpr (sizeof(T) == 4) {
        if (f.rtw_x.p && !Afu) {
            rfft::pass_c(f.lgx, reinterpret_cast<const float2 *>(B), oy, ldb, b_blocking(f), f.Hx, k, ox,
                         (float)(1.0 / ((double)f.Mx * (double)f.My)), out, ldo, omap, w, stride, f.rtw_x.as<float2>(),
                         st, cs);
            return;
        }
    }
    const int CB = 2 * batch_for(f.lgx, 2048);   // output columns (two per complex transform)
    const size_t smem = smem_ab<T>(f.lgx, CB / 2, 0);
    const int nth = threads_for(f.lgx, CB / 2, cdiv(oy, CB) * k);
    auto kern = nth <= 256 ? fft_pass_c<T, 256> : fft_pass_c<T, 512>;
    set_max_smem(kern);
    const T inv = (T)(1.0 / ((double)f.Mx * (double)f.My));
    kern<<<dim3((unsigned)cdiv(oy, CB), k), nth, smem, st>>>(B, oy, ldb, f.Hx, f.lgx, CB, ox, inv, out, ldo, omap,
                                                                       w, stride, f.stab_x.as<cplx<T>>(), f.lgx, Afu,
                                                                       ny_in, lda, Afu ? f.gk.as<cplx<T>>() : nullptr,
                                                                       f.lgy);
    after_launch("fft_pass_c");
}

template <typename T>
static void ensure(FftOperator &f, DevBuf &b, size_t &cap, size_t need, cudaStream_t st) {
    if (need > cap) { b.alloc(need, st); cap = need; }
}

// g[fx, d] = Σ_fy X̂[fx, fy]·exp(+2πi fy d / My), accumulated in fp64 (plan time, small My only)
template <typename T>
__global__ void gk_kernel(const cplx<T> *__restrict__ Xh, int Hx, int lgy, cplx<T> *__restrict__ g) {
    const int My = 1 << lgy;
    const int64_t n = (int64_t)Hx * My;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
        const int fx = (int)(t >> lgy), d = (int)(t & (My - 1));
        double sr = 0.0, si = 0.0;
        for (int fy = 0; fy < My; ++fy) {
            double sn, cs;
            sincospi(2.0 * (double)((fy * d) & (My - 1)) / (double)My, &sn, &cs);
            const cplx<T> x = Xh[(int64_t)fx * My + fy];
            sr += (double)x.x * cs - (double)x.y * sn;
            si += (double)x.x * sn + (double)x.y * cs;
        }
        g[t] = cplx<T>{(T)sr, (T)si};
    }
}

template <typename T>
static void build_impl(PlanImpl &p) {
    FftOperator &f = *p.fft;
    f.lgx = ilog2_ceil(p.nx); f.lgy = ilog2_ceil(p.ny);
    f.Mx = 1 << f.lgx; f.My = 1 << f.lgy; f.Hx = f.Mx / 2 + 1;
    f.lgtw = std::max(f.lgx, f.lgy);
    // per-stage twiddle tables (see stab_off): stage l (radix 8, span 2^l > 1), w1[k] = exp(−2πi k / 2^(l+3))
    auto build_stab = [&](int lg, DevBuf &buf) {
        std::vector<cplx<T>> h(std::max<size_t>(stab_count(lg), 1));
        size_t o = 0;
        for (int l = lg % 3; l < lg; l += 3) {
            if (l == 0) continue;
            const int ns = 1 << l;
            for (int k = 0; k < ns; ++k) {
                const double a = -2.0 * M_PI * (double)k / (double)(8 * ns);
                h[o++] = cplx<T>{(T)std::cos(a), (T)std::sin(a)};
            }
        }
        buf.alloc(sizeof(cplx<T>) * h.size(), p.st);
        SSA_CUDA(cudaMemcpyAsync(buf.p, h.data(), sizeof(cplx<T>) * h.size(), cudaMemcpyHostToDevice, p.st));
        SSA_CUDA(cudaStreamSynchronize(p.st));
    };
    build_stab(f.lgx, f.stab_x);
    build_stab(f.lgy, f.stab_y);
    if constexpr (sizeof(T) == 4) {
        // register-resident radix-16 passes for 2^8..2^12-point axes (fft_reg.cu); the X̂ build
        // below and the other sizes use the shared-memory Stockham passes
        static const bool off = std::getenv("SSA_FFT_STOCKHAM") != nullptr;   // A/B comparison switch
        auto build_rtw = [&](int lg, DevBuf &buf) {
            if (off || !rfft::supported(lg)) return;
            std::vector<float2> h;
            rfft::build_table(lg, h);
            buf.alloc(sizeof(float2) * h.size(), p.st);
            SSA_CUDA(cudaMemcpyAsync(buf.p, h.data(), sizeof(float2) * h.size(), cudaMemcpyHostToDevice, p.st));
            SSA_CUDA(cudaStreamSynchronize(p.st));
        };
        build_rtw(f.lgx, f.rtw_x);
        build_rtw(f.lgy, f.rtw_y);
    }
    f.Xh.alloc(sizeof(cplx<T>) * (size_t)f.Hx * f.My, p.st);
    DevBuf tmp;
    tmp.alloc(sizeof(cplx<T>) * (size_t)f.Hx * row_ld(p.ny), p.st);
    // X̂: x-DFT of the image columns, then the full-length y-DFT (mode 1)
    pass_a<T>(f, p.img.as<T>(), 0, nullptr, p.nx, p.ny, 1, nullptr, nullptr, tmp.as<cplx<T>>(), p.st);
    pass_b<T>(f, tmp.as<cplx<T>>(), p.ny, 1, 1, f.Xh.as<cplx<T>>(), f.My, p.st);
    if (f.My <= 64) {
        f.gk.alloc(sizeof(cplx<T>) * (size_t)f.Hx * f.My, p.st);
        gk_kernel<T><<<(unsigned)cdiv((int64_t)f.Hx * f.My, 256), 256, 0, p.st>>>(f.Xh.as<cplx<T>>(), f.Hx, f.lgy,
                                                                                   f.gk.as<cplx<T>>());
        after_launch("fft_gk");
    }
    SSA_CUDA(cudaStreamSynchronize(p.st));
}

void fft_build(PlanImpl &p) {
    if (!p.fft) p.fft = new FftOperator();
    if (p.dt == SSA_F64) build_impl<double>(p);
    else build_impl<float>(p);
}

// out box (ox x oy) <- correlation of the image with the input box (bx x by)
template <typename T>
static void correlate(PlanImpl &p, const T *in, int64_t ldin, const int *imap, int bx, int by, T *out, int64_t ldo,
                      const int *omap, int ox, int oy, int k, int64_t nout = 0, const double *cs = nullptr) {
    FftOperator &f = *p.fft;
    for (int j0 = 0; j0 < k; j0 += 64) {
        const int kc = std::min(64, k - j0);
        ensure<T>(f, f.bufA, f.capA, sizeof(cplx<T>) * (size_t)kc * f.Hx * row_ld(by), p.st);
        ensure<T>(f, f.bufB, f.capB, sizeof(cplx<T>) * (size_t)kc * f.Hx * b_cols(f, oy), p.st);
        pass_a<T>(f, in + ldin * j0, ldin, imap, bx, by, kc, nullptr, nullptr, f.bufA.as<cplx<T>>(), p.st);
        if (f.gk.p && by <= 2 && (int64_t)by * oy <= 64) {
            // MSSA-like shapes (few rows in and out): pass B folded into pass C
            pass_c<T>(f, nullptr, oy, kc, ox, out + ldo * j0, ldo, omap, nullptr, 0, p.st, f.bufA.as<cplx<T>>(), by);
        } else {
            pass_b<T>(f, f.bufA.as<cplx<T>>(), by, kc, 0, f.bufB.as<cplx<T>>(), oy, p.st);
            const bool reg = sizeof(T) == 4 && f.rtw_x.p;
            pass_c<T>(f, f.bufB.as<cplx<T>>(), oy, kc, ox, out + ldo * j0, ldo, omap, nullptr, 0, p.st, nullptr, 0,
                      (cs && reg) ? cs + j0 : nullptr);
            if (cs && !reg) scale_columns<T>(nout, out + ldo * j0, ldo, kc, cs + j0, p.st);
            continue;
        }
        if (cs) scale_columns<T>(nout, out + ldo * j0, ldo, kc, cs + j0, p.st);
    }
}

template <typename T>
void fft_xv(PlanImpl &p, const T *V, int64_t ldv, T *U, int64_t ldu, int k) {
    correlate<T>(p, V, ldv, p.full_k ? nullptr : p.kmap.as<int>(), p.kx, p.ky, U, ldu,
                 p.full_window ? nullptr : p.lmap.as<int>(), p.lx, p.ly, k);
}

template <typename T>
void fft_xtu(PlanImpl &p, const T *U, int64_t ldu, T *V, int64_t ldv, int k, const double *cs) {
    correlate<T>(p, U, ldu, p.full_window ? nullptr : p.lmap.as<int>(), p.lx, p.ly, V, ldv,
                 p.full_k ? nullptr : p.kmap.as<int>(), p.kx, p.ky, k, p.K, cs);
}

// Grouped averaging via FFT: out_g = IDFT2(Σ_{i∈I_g} σ_i Ψ̂_i Φ̂_i) / 𝕎 (NaN off 𝔑′).
// ---------------------------------------------------------------------------
// Low-weight cells of the FFT averaging.  The FFT forms the numerator Σ_{ℓ+κ=n} σ U[ℓ] V[κ] with an
// absolute rounding error that is uniform over the grid (~ε·RMS of the numerator), and Alg. 4 then
// divides by w_n: at the borders (w_n down to 1 at the corners, against w_max = |𝔏| in the bulk) the
// relative error grows by w_max / w_n (c5 corners: ~1.5e-3 of the reconstruction's RMS in fp32,
// measured).  Cells with w_n < w_max / 1024 are therefore re-done by direct summation over their
// w_n (ℓ, κ) pairs (fp64 accumulation): the error left elsewhere is ≲ 1.5e-3·RMS/64 ≈ 2.3e-5·RMS,
// and the direct work stays small (c5: ~2k cells; at w_max / 64 it was ~50k cells and 4.4 ms).
__global__ void low_weight_cells_kernel(const int *__restrict__ w, int64_t n, int thr, int *list, int *count) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
        const int wn = w[t];
        if (wn > 0 && wn < thr) list[atomicAdd(count, 1)] = (int)t;
    }
}

// one warp per (cell, group): out[g*stride + n] = Σ_{i∈I_g} σ_i Σ_{ℓ∈𝔏, κ=n−ℓ∈𝔎} U_i[ℓ] V_i[κ] / wdiv[n]
template <typename T>
__global__ void diagsums_cells_kernel(const int *__restrict__ cells, int ncells, int nx, int lx, int ly,
                                      const int *__restrict__ lmap, int kx, int ky, const int *__restrict__ kmap,
                                      const T *__restrict__ U, int64_t ldu, const T *__restrict__ V, int64_t ldv,
                                      const double *__restrict__ sig, const int *__restrict__ grp_off,
                                      const int *__restrict__ grp_idx, const int *__restrict__ wdiv, T *out,
                                      int64_t stride) {
    const int lane = threadIdx.x & 31;
    const int c = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int g = blockIdx.y;
    if (c >= ncells) return;
    const int n = cells[c];
    const int i = n % nx, j = n / nx;
    const int a0 = max(0, i - kx + 1), a1 = min(lx - 1, i), b0 = max(0, j - ky + 1), b1 = min(ly - 1, j);
    const int na = a1 - a0 + 1, nb = b1 - b0 + 1;
    double acc = 0.0;
    for (int m = grp_off[g]; m < grp_off[g + 1]; ++m) {
        const int t = grp_idx[m];
        const T *u = U + ldu * t;
        const T *v = V + ldv * t;
        double s = 0.0;
        for (int q = lane; q < na * nb; q += 32) {
            const int la = a0 + q % na, lb = b0 + q / na;          // ℓ = (la, lb), κ = (i − la, j − lb)
            const int lbox = la + lx * lb, kbox = (i - la) + kx * (j - lb);
            const int li = lmap ? lmap[lbox] : lbox;
            const int ki = kmap ? kmap[kbox] : kbox;
            if (li >= 0 && ki >= 0) s += (double)u[li] * (double)v[ki];
        }
        acc += sig[t] * s;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) out[(int64_t)g * stride + n] = (T)(acc / (double)wdiv[n]);
}

template <typename T>
void fft_diagsums(PlanImpl &p, const T *U, const T *V, const double *sig_dev, const int *grp_off_dev,
                  const int *grp_idx_dev, int ng, const std::vector<int> &used, const int *slot_dev, T *out,
                  const int *wdiv) {
    FftOperator &f = *p.fft;
    const int nu = (int)used.size();
    DevBuf jsel, AU, AV, B;
    jsel.alloc(sizeof(int) * std::max(nu, 1), p.st);
    SSA_CUDA(cudaMemcpyAsync(jsel.p, used.data(), sizeof(int) * nu, cudaMemcpyHostToDevice, p.st));
    AU.alloc(sizeof(cplx<T>) * (size_t)nu * f.Hx * row_ld(p.ly), p.st);
    AV.alloc(sizeof(cplx<T>) * (size_t)nu * f.Hx * row_ld(p.ky), p.st);
    B.alloc(sizeof(cplx<T>) * (size_t)ng * f.Hx * b_cols(f, p.ny), p.st);
    pass_a<T>(f, U, p.L, p.full_window ? nullptr : p.lmap.as<int>(), p.lx, p.ly, nu, jsel.as<int>(), sig_dev,
              AU.as<cplx<T>>(), p.st);
    pass_a<T>(f, V, p.K, p.full_k ? nullptr : p.kmap.as<int>(), p.kx, p.ky, nu, jsel.as<int>(), nullptr,
              AV.as<cplx<T>>(), p.st);
    bool done = false;
    if constexpr (sizeof(T) == 4) {
        if (f.rtw_y.p) {
            rfft::pass_bconv(f.lgy, AU.as<float2>(), p.ly, row_ld(p.ly), AV.as<float2>(), p.ky, row_ld(p.ky), grp_off_dev,
                             grp_idx_dev, slot_dev, f.Hx, ng, B.as<float2>(), p.ny, row_ld(p.ny), b_blocking(f),
                             f.rtw_y.as<float2>(), p.st);
            done = true;
        }
    }
    if (!done) {
        const int RB = batch_for(f.lgy, 2048);
        const size_t smem = sizeof(cplx<T>) * (5 * sp_size((size_t)RB << f.lgy) + stab_count(f.lgy));
        const int nth = threads_for(f.lgy, RB, cdiv(f.Hx, RB) * ng);
        auto kern = nth <= 256 ? fft_pass_b_conv<T, 256> : fft_pass_b_conv<T, 512>;
        set_max_smem(kern);
        kern<<<dim3((unsigned)cdiv(f.Hx, RB), ng), nth, smem, p.st>>>(
            AU.as<cplx<T>>(), p.ly, row_ld(p.ly), AV.as<cplx<T>>(), p.ky, row_ld(p.ky), grp_off_dev, grp_idx_dev,
            slot_dev, f.Hx, f.lgy, RB, B.as<cplx<T>>(), p.ny, row_ld(p.ny), f.stab_y.as<cplx<T>>(), f.lgy);
        after_launch("fft_pass_b_conv");
    }
    pass_c<T>(f, B.as<cplx<T>>(), p.ny, ng, p.nx, out, p.nx, nullptr, wdiv, (int64_t)p.nx * p.ny, p.st);
    // low-weight cells by direct summation (see diagsums_cells_kernel)
    const int64_t nxy = (int64_t)p.nx * p.ny;
    if (f.n_lowcells < 0) {
        const int wmax = (int)std::min<int64_t>(p.L, p.K);
        const int thr = wmax / 1024;
        f.n_lowcells = 0;
        if (thr > 1) {
            DevBuf cnt;
            cnt.alloc(sizeof(int), p.st);
            SSA_CUDA(cudaMemsetAsync(cnt.p, 0, sizeof(int), p.st));
            // upper bound on the list: cells with w < thr lie within ~thr/... of the border; size it by nxy
            f.lowcells.alloc(sizeof(int) * nxy, p.st);
            low_weight_cells_kernel<<<(unsigned)std::min<int64_t>(cdiv(nxy, 256), 16 * num_sms()), 256, 0, p.st>>>(
                p.weights.as<int>(), nxy, thr, f.lowcells.as<int>(), cnt.as<int>());
            after_launch("low_weight_cells");
            SSA_CUDA(cudaMemcpyAsync(&f.n_lowcells, cnt.p, sizeof(int), cudaMemcpyDeviceToHost, p.st));
            SSA_CUDA(cudaStreamSynchronize(p.st));
        }
    }
    if (f.n_lowcells > 0 && ng > 0) {
        diagsums_cells_kernel<T><<<dim3((unsigned)cdiv(f.n_lowcells, 8), ng), 256, 0, p.st>>>(
            f.lowcells.as<int>(), f.n_lowcells, p.nx, p.lx, p.ly, p.full_window ? nullptr : p.lmap.as<int>(), p.kx,
            p.ky, p.full_k ? nullptr : p.kmap.as<int>(), U, p.L, V, p.K, sig_dev, grp_off_dev, grp_idx_dev, wdiv, out,
            nxy);
        after_launch("diagsums_cells");
    }
    SSA_CUDA(cudaStreamSynchronize(p.st));
}

template void fft_xv<float>(PlanImpl &, const float *, int64_t, float *, int64_t, int);
template void fft_xv<double>(PlanImpl &, const double *, int64_t, double *, int64_t, int);
template void fft_xtu<float>(PlanImpl &, const float *, int64_t, float *, int64_t, int, const double *);
template void fft_xtu<double>(PlanImpl &, const double *, int64_t, double *, int64_t, int, const double *);
template void fft_diagsums<float>(PlanImpl &, const float *, const float *, const double *, const int *, const int *,
                                  int, const std::vector<int> &, const int *, float *, const int *);
template void fft_diagsums<double>(PlanImpl &, const double *, const double *, const double *, const int *, const int *,
                                   int, const std::vector<int> &, const int *, double *, const int *);

void fft_destroy(FftOperator *f) { delete f; }

}  // namespace ssa
