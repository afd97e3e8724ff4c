// Kernel parameter blocks and launch wrappers of libssa_b200 (device side).
#pragma once
#include "common.h"

namespace ssa {

// out[p, j] = Σ_d x[p + d] W[d, j] over an output box (ox x oy) and a reduction
// box (dx x dy); see direct.cu.
template <typename T>
struct CorrParams {
    const T *x; int64_t ldx; int nx, ny;     // image, zero outside 𝔑
    int ox, oy;                              // output box
    int dx, dy;                              // reduction box
    const T *W; int64_t ldw; const int *wmap;   // filters, compact; wmap: box -> compact or -1 (null = identity)
    T *out; int64_t ldo; const int *omap;       // output, compact; omap: box -> compact or -1 (null = identity)
    int k;                                   // number of filters
    // filled by the launcher
    T *ws; int nsplit; int nsx; int dy_split; int dx_split; int px; int xpitch;
};

template <typename T>
void corr_direct(CorrParams<T> P, T *ws_buf, size_t ws_bytes, cudaStream_t st);
size_t corr_direct_ws_bytes(int64_t nbox, int64_t k, int elem);

// Grouped diagsums with the ÷𝕎 epilogue (direct.cu).
template <typename T>
struct AvgParams {
    int nx, ny;                              // output grid
    int lx, ly; const int *lmap;             // 𝔏 box and map (null = full)
    int kx, ky; const int *kmap;             // 𝔎 box and map (null = full)
    const T *U; int64_t ldu;                 // L x r (null = ones)
    const T *V; int64_t ldv;                 // K x r (null = ones)
    const double *coef;                      // per-triple scale σ_i (null = 1)
    const int *grp_off; const int *grp_idx; int ngroups;
    const int *w;                            // weights (null = raw numerator)
    T *out; int64_t ldout; int64_t out_stride;
    // filled by the launcher
    int px; int bpitch;
};

template <typename T>
void diagsums_direct(AvgParams<T> P, cudaStream_t st);

// ---- tensor-core (tcgen05 3xTF32) implicit GEMM, fp32 only (hankel_tc.cu) -------
// Same operation as CorrParams: out[p, j] = Σ_{d ∈ in-box} x[p + d] in[d, j].
struct TcCorrParams {
    const float *x_hi, *x_lo; int nx, ny;    // tf32 hi / lo planes of the image (tc_build_planes), ld tc_plane_ld(nx)
    int ox, oy;                              // output box
    int bx, by;                              // reduction (input) box
    const float *in; int64_t ldi; const int *imap;   // filters, compact; imap: box -> compact or -1
    float *out; int64_t ldo; const int *omap;        // output, compact; omap: box -> compact or -1
    int k;
    float *ws; size_t ws_bytes;              // split-K partials
    float *bpk; size_t bpk_bytes;            // packed hi/lo filters
};
bool tc_corr_supported(int ox, int oy, int bx, int by, int k);
int tc_plane_ld(int nx);
void tc_build_planes(const float *x, int64_t ldx, int nx, int ny, float *hi, float *lo, cudaStream_t st);
size_t tc_pack_bytes(int bx, int by, int k);
void tc_corr(const TcCorrParams &P, cudaStream_t st);

// ---- FFT path (fft.cu) -----------------------------------------------------
struct FftPlan;   // opaque, defined in fft.cu

// ---- small dense / tall-skinny helpers (blas.cu) -------------------------
// G (n1 x n2, column-major, double, device) = Aᵀ B with A: M x n1 (n1 <= 512), B: M x n2 (n2 <= 64).
template <typename T>
void gram_tn(int64_t M, const T *A, int64_t lda, int n1, const T *B, int64_t ldb, int n2,
             double *G, double *partials, size_t partial_bytes, cudaStream_t st);
size_t gram_partial_bytes(int64_t M, int n1, int n2);
void gram_reduce(const double *partials, int nparts, int n1, int n2, double *G, cudaStream_t st, int ldg = 0);
// TMA streaming probe (measurement only): M x n block in boxes of brow rows, `boxes` per stage
void tma_stream_probe(int64_t M, const float *A, int64_t lda, int n, int brow, int boxes, bool swz, int pd, cudaStream_t st);
// tcgen05 3xTF32 Gram (tall_tc.cu); false when the layout is unsupported
bool gram_tc(int64_t M, const float *A, int64_t lda, int n1, const float *B, int64_t ldb, int n2, double *G,
             double *partials, size_t partial_bytes, cudaStream_t st);
void box_kmask(const uint8_t *nmask, int nx, int ny, int lx, int ly, uint8_t *kmask, int32_t *tmp, cudaStream_t st);
void box_weights(const uint8_t *kmask, int nx, int ny, int lx, int ly, int32_t *w, int32_t *tmp, cudaStream_t st);
// tcgen05 3xTF32 update Out = beta·Out + alpha·A·C (tall_tc.cu); false when unsupported
bool update_tc(int64_t M, const float *A, int64_t lda, int m, const double *C, int ldc, int n, double alpha,
               double beta, float *Out, int64_t ldo, cudaStream_t st);

// Out (M x n) = beta*Out + alpha * A (M x m) * C (m x n, device double, column-major).
// In-place (Out == A, with m == n) is allowed.
template <typename T>
void gemm_small(int64_t M, const T *A, int64_t lda, int m, const double *C, int ldc, int n,
                double alpha, double beta, T *Out, int64_t ldo, cudaStream_t st);

// Out (M x n) = beta*Out + alpha * A (M x m) * C (m x n); m <= 512, n <= 64, Out != A (one launch).
template <typename T>
void gemm_acc(int64_t M, const T *A, int64_t lda, int m, const double *C, int ldc, int n, double alpha,
              double beta, T *Out, int64_t ldo, cudaStream_t st);

// A[:, cols] = N(0,1) from a counter-based generator keyed by (seed, stream_id).
template <typename T>
void fill_normal(int64_t M, T *A, int64_t lda, int ncols, uint64_t seed, uint64_t stream_id,
                 cudaStream_t st);

// ---- plan-time kernels (plan.cu) ------------------------------------------
template <typename T>
void prep_image(const T *src, int64_t ld_src, int nx, int ny, const uint8_t *mask,
                T *dst, uint8_t *nmask, cudaStream_t st);
// counts (kx x ky, as T, exact integers) == L  -> kmask
template <typename T>
void threshold_eq(const T *counts, int64_t n, double value, uint8_t *out, cudaStream_t st);
template <typename T>
void box_ones_to_int(const T *src, int64_t n, int32_t *dst, cudaStream_t st);
// per-column counts of a (bx x by) u8 mask, then compact index map
void column_counts(const uint8_t *m, int bx, int by, int32_t *counts, cudaStream_t st);
void compact_map(const uint8_t *m, int bx, int by, const int32_t *col_start, int32_t *map,
                 int32_t *pos_list, int64_t ld_img, cudaStream_t st);
void weights_rect(int nx, int ny, int lx, int ly, int32_t *w, cudaStream_t st);

template <typename T>
void rest_group(const T *x, const int32_t *w, const T *groups, int ngroups, int64_t stride,
                int64_t n, T *rest, cudaStream_t st);
template <typename T>
void cast_copy(const void *src, int src_is_double, T *dst, int64_t n, cudaStream_t st);
template <typename T>
void scale_columns(int64_t M, T *A, int64_t lda, int n, const double *s, cudaStream_t st);
template <typename T>
void absmax_sign(int64_t M, const T *A, int64_t lda, int n, double *sgn, cudaStream_t st);

}  // namespace ssa
