// Direct (implicit-GEMM) kernels for the trajectory-operator products and the
// diagonal averaging of arXiv 1309.5050, on CUDA cores (sm_100a).
//
// Both products are the same operation: a correlation of the image with k
// filters evaluated on a box of positions,
//
//     out[p, j] = Σ_{d ∈ D-box} x[p + d] · W[d, j]
//
//   Xᵀ·U (K-side):  p ∈ 𝔎-box (kx x ky), d ∈ 𝔏-box, W = U   (v_κ = Σ_ℓ x[ℓ+κ] u_ℓ)
//   X·V  (L-side):  p ∈ 𝔏-box (lx x ly), d ∈ 𝔎-box, W = V   (u_ℓ = Σ_κ x[ℓ+κ] v_κ)
//
// (rows / columns of the quasi-Hankel matrix, eq. P:3020-3028; 0-based, so the
// shifted sum ℓ +‐ κ is plain addition).  Shapes enter only through index maps:
// a filter cell outside its shape has weight 0 (map -1), an output cell outside
// its shape is not written.  The Hankel structure is exploited in registers:
// a thread owns TM consecutive outputs along x, so stepping the reduction
// offset d.x by one shifts its image window by one — one new shared-memory
// load per TM*TN FMAs.  A CTA stages an image tile (+halo) and a filter chunk
// in shared memory per reduction chunk; large reductions (X·V over |𝔎|) are
// split over CTAs along d.y and reduced deterministically by a second kernel.
#include "common.h"
#include "kernels.h"

namespace ssa {

template <typename T> struct DirectCfg;
template <> struct DirectCfg<float> { static constexpr int TM = 8, TN = 8; };
template <> struct DirectCfg<double> { static constexpr int TM = 4, TN = 4; };

constexpr int kThreads = 256;
constexpr int kJG = 4;                   // filter groups per CTA
constexpr int kPT = kThreads / kJG;      // position-threads per CTA (64)

template <typename T, int CDX, int CDY>
__global__ void __launch_bounds__(kThreads, 2)
corr_direct_kernel(CorrParams<T> P) {
    constexpr int TM = DirectCfg<T>::TM, TN = DirectCfg<T>::TN;
    constexpr int KV = kJG * TN;         // filters per CTA
    extern __shared__ __align__(16) unsigned char smem_raw[];
    T *WS = reinterpret_cast<T *>(smem_raw);                 // [CDX*CDY][KV]
    T *XS = WS + CDX * CDY * KV;                              // [YT][XPP]

    const int PX = P.px, PY = kPT / PX;
    const int TX = TM * PX, TY = PY;
    const int XW = TX + CDX - 1;                              // tile rows needed
    const int XPP = P.xpitch;                                 // smem pitch (>= XW)
    const int YT = TY + CDY - 1;

    const int ntx = (P.ox + TX - 1) / TX;
    const int ox0 = (blockIdx.x % ntx) * TX;
    const int oy0 = (blockIdx.x / ntx) * TY;
    const int j0 = blockIdx.y * KV;
    const int split = blockIdx.z;
    const int zx = split % P.nsx, zy = split / P.nsx;   // split-K over both reduction axes
    const int dy_lo = zy * P.dy_split;
    const int dy_hi = min(P.dy, dy_lo + P.dy_split);
    const int dx_lo = zx * P.dx_split;
    const int dx_hi = min(P.dx, dx_lo + P.dx_split);

    const int tid = threadIdx.x;
    const int jg = tid % kJG;
    const int pt = tid / kJG;
    const int pxi = pt % PX, pyi = pt / PX;
    const int xb = pxi * TM;

    T acc[TM][TN];
#pragma unroll
    for (int t = 0; t < TM; ++t)
#pragma unroll
        for (int j = 0; j < TN; ++j) acc[t][j] = T(0);

    for (int dy0 = dy_lo; dy0 < dy_hi; dy0 += CDY) {
        for (int dx0 = dx_lo; dx0 < dx_hi; dx0 += CDX) {
            __syncthreads();
            // ---- stage the image tile: rows ox0+dx0 .. +XW, cols oy0+dy0 .. +YT
            for (int idx = tid; idx < XW * YT; idx += kThreads) {
                const int xl = idx % XW, yl = idx / XW;
                const int gx = ox0 + dx0 + xl, gy = oy0 + dy0 + yl;
                T v = T(0);
                if (gx < P.nx && gy < P.ny) v = P.x[gx + P.ldx * (int64_t)gy];
                XS[xl + XPP * yl] = v;
            }
            // ---- stage the filter chunk, transposed to [d][j] (lane = j)
            for (int idx = tid; idx < CDX * CDY * KV; idx += kThreads) {
                const int jl = idx % KV, dl = idx / KV;
                const int dxl = dl % CDX, dyl = dl / CDX;
                const int gdx = dx0 + dxl, gdy = dy0 + dyl;
                const int jj = j0 + jl;
                T v = T(0);
                if (gdx < dx_hi && gdy < dy_hi && jj < P.k) {
                    const int64_t box = gdx + (int64_t)P.dx * gdy;
                    const int64_t wi = P.wmap ? (int64_t)P.wmap[box] : box;
                    if (wi >= 0) v = P.W[wi + P.ldw * (int64_t)jj];
                }
                WS[dl * KV + jl] = v;
            }
            __syncthreads();
            // ---- compute: sliding window along d.x
#pragma unroll 1
            for (int dyl = 0; dyl < CDY; ++dyl) {
                const T *xrow = XS + (pyi + dyl) * XPP + xb;
                const T *wrow = WS + (CDX * dyl) * KV + jg * TN;
#pragma unroll 2
                for (int dxl = 0; dxl < CDX; dxl += TM) {
                    T win[2 * TM - 1];
#pragma unroll
                    for (int s = 0; s < 2 * TM - 1; ++s) win[s] = xrow[dxl + s];
#pragma unroll
                    for (int dd = 0; dd < TM; ++dd) {
                        T wv[TN];
                        const T *wp = wrow + (dxl + dd) * KV;
#pragma unroll
                        for (int j = 0; j < TN; ++j) wv[j] = wp[j];
#pragma unroll
                        for (int t = 0; t < TM; ++t)
#pragma unroll
                            for (int j = 0; j < TN; ++j) acc[t][j] = fma(win[t + dd], wv[j], acc[t][j]);
                    }
                }
            }
        }
    }
    // ---- epilogue
    const int py = oy0 + pyi;
    if (py >= P.oy) return;
    const int64_t nbox = (int64_t)P.ox * P.oy;
#pragma unroll
    for (int t = 0; t < TM; ++t) {
        const int px = ox0 + xb + t;
        if (px >= P.ox) continue;
        const int64_t pidx = px + (int64_t)P.ox * py;
        if (P.nsplit == 1) {
            const int64_t oi = P.omap ? (int64_t)P.omap[pidx] : pidx;
            if (oi < 0) continue;
#pragma unroll
            for (int j = 0; j < TN; ++j) {
                const int jj = j0 + jg * TN + j;
                if (jj < P.k) P.out[oi + P.ldo * (int64_t)jj] = acc[t][j];
            }
        } else {
#pragma unroll
            for (int j = 0; j < TN; ++j) {
                const int jj = j0 + jg * TN + j;
                if (jj < P.k) P.ws[((int64_t)split * P.k + jj) * nbox + pidx] = acc[t][j];
            }
        }
    }
}

// Deterministic reduction of split-K partials: out[omap(p), j] = Σ_s ws[s][j][p].
template <typename T>
__global__ void reduce_splits_kernel(const T *__restrict__ ws, int nsplit, int64_t nbox, int k,
                                     const int *__restrict__ omap, T *__restrict__ out, int64_t ldo) {
    const int64_t n = nbox * k;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t p = t % nbox, j = t / nbox;
        const int64_t oi = omap ? (int64_t)omap[p] : p;
        if (oi < 0) continue;
        T s = T(0);
        for (int q = 0; q < nsplit; ++q) s += ws[((int64_t)q * k + j) * nbox + p];
        out[oi + ldo * j] = s;
    }
}

template <typename T, int CDX, int CDY>
static void launch_corr(CorrParams<T> P, cudaStream_t st) {
    constexpr int TM = DirectCfg<T>::TM, TN = DirectCfg<T>::TN;
    constexpr int KV = kJG * TN;
    const int PX = P.px, PY = kPT / PX;
    const int TX = TM * PX, TY = PY;
    const int XW = TX + CDX - 1;
    P.xpitch = XW + ((4 - (XW % 32) + 32) % 32);   // pitch ≡ 4 (mod 32): distinct banks per y-row
    const int YT = TY + CDY - 1;
    const size_t smem = sizeof(T) * ((size_t)CDX * CDY * KV + (size_t)P.xpitch * YT);
    auto kern = corr_direct_kernel<T, CDX, CDY>;
    set_max_smem(kern);
    const int ntx = (int)cdiv(P.ox, TX), nty = (int)cdiv(P.oy, TY);
    dim3 grid(ntx * nty, (unsigned)cdiv(P.k, KV), P.nsplit);
    kern<<<grid, kThreads, smem, st>>>(P);
    after_launch("corr_direct");
}

static int choose_px(int ox, int oy, int TM) {
    // pick PX (PY = 64/PX) minimising padded work; ties -> larger PX (longer x runs)
    int best = 1; double bestw = 1e300;
    for (int px = 1; px <= kPT; px *= 2) {
        const int py = kPT / px;
        const double w = (double)cdiv(ox, TM * px) * TM * px * (double)cdiv(oy, py) * py;
        if (w <= bestw) { bestw = w; best = px; }
    }
    return best;
}

template <typename T>
void corr_direct(CorrParams<T> P, T *ws_buf, size_t ws_bytes, cudaStream_t st) {
    constexpr int TM = DirectCfg<T>::TM, TN = DirectCfg<T>::TN;
    constexpr int KV = kJG * TN;
    if (P.k <= 0 || P.ox <= 0 || P.oy <= 0) return;
    P.px = choose_px(P.ox, P.oy, TM);
    const bool flat = (P.dy == 1);            // 1-row reduction box (MSSA X^T U): CDY = 1
    const int cdy = flat ? 1 : 4, cdx = flat ? 128 : 32;
    const int PY = kPT / P.px;
    const int64_t tiles = cdiv(P.ox, TM * P.px) * cdiv(P.oy, PY) * cdiv(P.k, KV);
    // split the reduction (first along d.y, then along d.x) until the grid fills
    // ~3 waves of 2 CTAs/SM, bounded by the partial-sum workspace
    const int64_t want = 3 * 2 * (int64_t)num_sms();
    const int64_t nbox = (int64_t)P.ox * P.oy;
    const int64_t max_ws_splits = std::max<int64_t>(1, (int64_t)(ws_bytes / ((size_t)P.k * nbox * sizeof(T))));
    int64_t need = tiles < want ? cdiv(want, tiles) : 1;
    need = std::min(need, max_ws_splits);
    int64_t nsy = std::min<int64_t>(need, cdiv(P.dy, cdy));
    int64_t nsx = std::min<int64_t>(cdiv(need, nsy), cdiv(P.dx, cdx));
    if (nsx < 1) nsx = 1;
    P.dy_split = (int)rup(cdiv(P.dy, nsy), cdy);
    nsy = cdiv(P.dy, P.dy_split);
    P.dx_split = (int)rup(cdiv(P.dx, nsx), cdx);
    nsx = cdiv(P.dx, P.dx_split);
    while (nsx * nsy > max_ws_splits && nsx > 1) {   // workspace bound after rounding
        --nsx;
        P.dx_split = (int)rup(cdiv(P.dx, nsx), cdx);
        nsx = cdiv(P.dx, P.dx_split);
    }
    const int64_t nsplit = nsx * nsy;
    P.nsx = (int)nsx;
    P.nsplit = (int)nsplit;
    P.ws = ws_buf;
    if (flat) launch_corr<T, 128, 1>(P, st);
    else launch_corr<T, 32, 4>(P, st);
    if (nsplit > 1) {
        const int64_t n = nbox * P.k;
        const int blocks = (int)std::min<int64_t>(cdiv(n, 256), 8 * num_sms());
        reduce_splits_kernel<T><<<blocks, 256, 0, st>>>(ws_buf, P.nsplit, nbox, P.k, P.omap, P.out, P.ldo);
        after_launch("reduce_splits");
    }
}

size_t corr_direct_ws_bytes(int64_t nbox, int64_t k, int elem) {
    // enough for up to 64 splits of the largest output box
    return (size_t)std::min<int64_t>(64, 1 + (int64_t)(2e9 / std::max<int64_t>(1, nbox * k * elem))) *
           (size_t)nbox * k * elem;
}

template void corr_direct<float>(CorrParams<float>, float *, size_t, cudaStream_t);
template void corr_direct<double>(CorrParams<double>, double *, size_t, cudaStream_t);

// ============================================================================
// Diagonal averaging numerator (diagsums of grouped rank-one sums, Alg. 5
// definition P:3894-3914 with the ÷𝕎 epilogue of Alg. 4):
//
//   num_g[n] = Σ_{i ∈ I_g} coef_i Σ_{ℓ ∈ 𝔏-box} U_i[ℓ] · V_i[n − ℓ]      (V_i = 0 off 𝔎)
//   out_g[n] = num_g[n] / w_n on 𝔑′ (w_n > 0), NaN elsewhere
//
// a full 2-D convolution of each eigenarray with its factor array, summed over
// the group.  Thread = TMA consecutive n.x; stepping ℓ.x slides its window of
// the factor-array tile by one.  When `w` is NULL the raw numerator is written
// (used for the plan's weights 𝕎 = diagsums(1_𝔏, 1_𝔎), exact in fp32 below 2^24).
// ============================================================================
template <typename T> struct AvgCfg { static constexpr int TMA = 8; };

template <typename T, int CLX, int CLY>
__global__ void __launch_bounds__(256)
diagsums_kernel(AvgParams<T> P) {
    constexpr int TMA = AvgCfg<T>::TMA;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    T *AS = reinterpret_cast<T *>(smem_raw);           // [CLY][CLX] coef_i * U_i chunk
    T *BS = AS + CLX * CLY;                            // [BYT][BPP] V_i tile (+halo)

    const int PX = P.px, PY = 256 / PX;
    const int TX = TMA * PX, TY = PY;
    const int ntx = (P.nx + TX - 1) / TX;
    const int nx0 = (blockIdx.x % ntx) * TX;
    const int ny0 = (blockIdx.x / ntx) * TY;
    const int g = blockIdx.y;
    const int i_lo = P.grp_off[g], i_hi = P.grp_off[g + 1];

    const int BW = TX + CLX - 1;     // tile rows:  n.x - ℓ.x for n.x in tile, ℓ.x in chunk
    const int BPP = P.bpitch;
    const int BYT = TY + CLY - 1;

    const int tid = threadIdx.x;
    const int pxi = tid % PX, pyi = tid / PX;
    const int xb = pxi * TMA;

    T acc[TMA];
#pragma unroll
    for (int t = 0; t < TMA; ++t) acc[t] = T(0);

    for (int ii = i_lo; ii < i_hi; ++ii) {
        const int i = P.grp_idx[ii];
        const T ci = P.coef ? (T)P.coef[i] : T(1);
        for (int ly0 = 0; ly0 < P.ly; ly0 += CLY) {
            for (int lx0 = 0; lx0 < P.lx; lx0 += CLX) {
                __syncthreads();
                // A chunk: ℓ = (lx0 + a, ly0 + b)
                for (int idx = tid; idx < CLX * CLY; idx += 256) {
                    const int a = idx % CLX, b = idx / CLX;
                    const int gx = lx0 + a, gy = ly0 + b;
                    T v = T(0);
                    if (gx < P.lx && gy < P.ly) {
                        const int64_t box = gx + (int64_t)P.lx * gy;
                        const int64_t li = P.lmap ? (int64_t)P.lmap[box] : box;
                        if (li >= 0) v = P.U ? ci * P.U[li + P.ldu * (int64_t)i] : ci;
                    }
                    AS[idx] = v;
                }
                // B tile: κ = n − ℓ; local row r ↔ κx = nx0 − lx0 − (CLX−1) + r
                const int kx0 = nx0 - lx0 - (CLX - 1), ky0 = ny0 - ly0 - (CLY - 1);
                for (int idx = tid; idx < BW * BYT; idx += 256) {
                    const int rl = idx % BW, cl = idx / BW;
                    const int kx = kx0 + rl, ky = ky0 + cl;
                    T v = T(0);
                    if (kx >= 0 && ky >= 0 && kx < P.kx && ky < P.ky) {
                        const int64_t box = kx + (int64_t)P.kx * ky;
                        const int64_t ki = P.kmap ? (int64_t)P.kmap[box] : box;
                        if (ki >= 0) v = P.V ? P.V[ki + P.ldv * (int64_t)i] : T(1);
                    }
                    BS[rl + BPP * cl] = v;
                }
                __syncthreads();
                // out[n] += Σ_{a,b} AS[a,b] · BS[xl − a + CLX−1, yl − b + CLY−1]
#pragma unroll 1
                for (int b = 0; b < CLY; ++b) {
                    const T *brow = BS + (pyi - b + CLY - 1) * BPP + xb + (CLX - 1);
                    const T *arow = AS + CLX * b;
#pragma unroll 2
                    for (int a0 = 0; a0 < CLX; a0 += TMA) {
                        // window: brow[t − a] for t ∈ [0,TMA), a ∈ [a0, a0+TMA)
                        T win[2 * TMA - 1];
#pragma unroll
                        for (int s = 0; s < 2 * TMA - 1; ++s) win[s] = brow[s - a0 - (TMA - 1)];
#pragma unroll
                        for (int da = 0; da < TMA; ++da) {
                            const T av = arow[a0 + da];
#pragma unroll
                            for (int t = 0; t < TMA; ++t)
                                acc[t] = fma(av, win[t - da + (TMA - 1)], acc[t]);
                        }
                    }
                }
            }
        }
    }
    const int ny = ny0 + pyi;
    if (ny >= P.ny) return;
    T *outg = P.out + (int64_t)g * P.out_stride;
#pragma unroll
    for (int t = 0; t < TMA; ++t) {
        const int nxx = nx0 + xb + t;
        if (nxx >= P.nx) continue;
        const int64_t n = nxx + (int64_t)P.ldout * ny;
        if (P.w) {
            const int wn = P.w[nxx + (int64_t)P.nx * ny];
            outg[n] = wn > 0 ? acc[t] / (T)wn : (T)NAN;
        } else {
            outg[n] = acc[t];
        }
    }
}

template <typename T>
void diagsums_direct(AvgParams<T> P, cudaStream_t st) {
    constexpr int TMA = AvgCfg<T>::TMA;
    constexpr int CLX = 32, CLY = 4;
    if (P.ngroups <= 0) return;
    // PX: positions along x (PY = 256/PX)
    int best = 1; double bestw = 1e300;
    for (int px = 1; px <= 256; px *= 2) {
        const int py = 256 / px;
        if (py > 64) continue;
        const double w = (double)cdiv(P.nx, TMA * px) * TMA * px * (double)cdiv(P.ny, py) * py;
        if (w <= bestw) { bestw = w; best = px; }
    }
    P.px = best;
    const int TX = TMA * P.px, TY = 256 / P.px;
    const int BW = TX + CLX - 1;
    P.bpitch = BW + ((4 - (BW % 32) + 32) % 32);
    const int BYT = TY + CLY - 1;
    const size_t smem = sizeof(T) * ((size_t)CLX * CLY + (size_t)P.bpitch * BYT);
    auto kern = diagsums_kernel<T, CLX, CLY>;
    set_max_smem(kern);
    dim3 grid((unsigned)(cdiv(P.nx, TX) * cdiv(P.ny, TY)), P.ngroups);
    kern<<<grid, 256, smem, st>>>(P);
    after_launch("diagsums_direct");
}

template void diagsums_direct<float>(AvgParams<float>, cudaStream_t);
template void diagsums_direct<double>(AvgParams<double>, cudaStream_t);

}  // namespace ssa
