// FFT circular-correlation path (Alg. 1/3/5) — placeholder until the smem radix
// FFT kernels land; fft_supported() reports false so AUTO picks the direct path.
#include "common.h"
#include "plan.h"

namespace ssa {
struct FftOperator {};
bool fft_supported(const PlanImpl &) { return false; }
void fft_build(PlanImpl &) { throw Error(SSA_ERR_ARG, "FFT path not built"); }
template <typename T>
void fft_xv(PlanImpl &, const T *, int64_t, T *, int64_t, int) { throw Error(SSA_ERR_ARG, "FFT path not built"); }
template <typename T>
void fft_xtu(PlanImpl &, const T *, int64_t, T *, int64_t, int) { throw Error(SSA_ERR_ARG, "FFT path not built"); }
template void fft_xv<float>(PlanImpl &, const float *, int64_t, float *, int64_t, int);
template void fft_xv<double>(PlanImpl &, const double *, int64_t, double *, int64_t, int);
template void fft_xtu<float>(PlanImpl &, const float *, int64_t, float *, int64_t, int);
template void fft_xtu<double>(PlanImpl &, const double *, int64_t, double *, int64_t, int);
void fft_destroy(FftOperator *f) { delete f; }
}  // namespace ssa
