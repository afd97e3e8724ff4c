// Register-resident radix-16 FFT passes (fp32, transform sizes 2^8 .. 2^12) of the FFT
// correlation products and of the grouped averaging; see fft_reg.cu.  Same operations and
// intermediate layouts as the shared-memory Stockham passes in fft.cu, which remain for the
// other sizes and for fp64 plans.
#pragma once
#include <vector>

#include "common.h"

namespace ssa {
namespace rfft {

constexpr int LG_MIN = 8, LG_MAX = 12;
inline bool supported(int lg) { return lg >= LG_MIN && lg <= LG_MAX; }

// per-stage twiddle table of a 2^lg-point transform (forward sign, fp64-accurate values
// rounded to fp32): stage with span Ns holds e^{-2πi r k / (16 Ns)}, k < Ns, r = 1..15
int tw_count(int lg);
void build_table(int lg, std::vector<float2> &h);

// A[(j*H + fx)*lda + col] = x-DFT (fx < H = 2^lg/2 + 1) of the input box columns; the input is
// in[map(ix, col) + ld*j] (map = box -> compact or -1, null = identity), scaled by scale[j] (null = 1),
// j = jsel[jo] (null = jo).  Two real columns per complex transform.
void pass_a(int lg, const float *in, int64_t ld, const int *map, int bx, int by, int k, const int *jsel,
            const double *scale, float2 *A, int lda, const float2 *tw, cudaStream_t st);
// per (j, fx): B row = IDFT_y( X̂[fx, :] ⊙ conj(DFT_y(A row)) ), first ny_out entries (2^lg = My)
// cbc: layout of B (0 = rows of stride ldb; else blocked by pass C's column blocks of cbc = cb_of(lgx))
void pass_b(int lg, const float2 *A, int ny_in, int lda, int H, int k, const float2 *Xh, float2 *B, int ny_out,
            int ldb, int cbc, const float2 *tw, cudaStream_t st);
int cb_of(int lg);   // block width of the blocked B layout for a 2^lg-point pass C
// per (g, fx): B row = IDFT_y( Σ_{i∈I_g} DFT_y(AU_i row) ⊙ DFT_y(AV_i row) ), first ny_out entries
void pass_bconv(int lg, const float2 *AU, int ly, int ldu, const float2 *AV, int ky, int ldv, const int *grp_off,
                const int *grp_idx, const int *slot, int H, int ng, float2 *B, int ny_out, int ldb, int cbc,
                const float2 *tw, cudaStream_t st);
// per output column y < oy: Hermitian completion, inverse x-DFT (2^lg), rows x < ox, times inv;
// products: out[omap(x, y) + ldo*j]; averaging (w != null): out[j*stride + x + ldo*y] = v / w (NaN if w = 0)
// cs (products only, may be null): output column j is also multiplied by cs[j] (V = XᵀU/σ in one pass)
void pass_c(int lg, const float2 *B, int oy, int ldb, int cblk, int H, int k, int ox, float inv, float *out,
            int64_t ldo, const int *omap, const int *w, int64_t stride, const float2 *tw, cudaStream_t st,
            const double *cs = nullptr);
// Intermediate rows (A: by columns, B: oy columns) have strides lda / ldb = multiples of 4 complex
// values (32-B aligned rows); the transposed accesses of passes A and C move 16-B column pairs.

}  // namespace rfft
}  // namespace ssa
