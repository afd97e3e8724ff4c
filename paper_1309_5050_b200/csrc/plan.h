// Plan object behind the opaque ssa_plan handle.
#pragma once
#include <memory>
#include <string>
#include <vector>

#include "common.h"

namespace ssa {

struct FftOperator;   // fft.cu

struct PlanImpl {
    // ---- geometry (0-based; x fastest) -------------------------------------
    int nx = 0, ny = 0, lx = 0, ly = 0, kx = 0, ky = 0;
    int64_t L = 0, K = 0, n_valid = 0, n_excluded = 0;
    bool full_window = true, full_k = true;
    ssa_dtype dt = SSA_F32;
    int path = SSA_PATH_DIRECT;   // requested path (AUTO resolved per product below)
    int path_xv = SSA_PATH_DIRECT, path_xtu = SSA_PATH_DIRECT;   // chosen per product
    int block_k = 32;
    int svd_method = 0;           // SSA_SVD_LANCZOS / SSA_SVD_EIGEN
    double tol = 0;
    int max_products = 0;
    uint64_t seed = 0;
    cudaStream_t st = nullptr;
    ssa_comm comm{};
    bool has_comm = false;
    int64_t band_y0 = 0, band_y1 = 0;   // band plans: this rank's global origin columns
    int64_t ny_global = 0;              // band plans: columns of the global image
    bool broken = false;          // sticky CUDA / comm failure

    // ---- device data ---------------------------------------------------------
    DevBuf img;       // T[nx*ny], 0 outside 𝔑
    DevBuf nmask;     // u8[nx*ny]
    DevBuf lmap;      // int32[lx*ly] box -> 𝔏 index or -1 (only if !full_window)
    DevBuf kmask;     // u8[kx*ky]
    DevBuf kmap;      // int32[kx*ky] box -> 𝔎 index or -1 (only if !full_k)
    DevBuf weights;   // int32[nx*ny]
    DevBuf ws_corr;   // split-K partials of the direct products
    size_t ws_corr_bytes = 0;
    DevBuf ws_gram;   // gram partials
    DevBuf tc_bpk;    // packed tf32 hi/lo filters of the tensor-core path
    DevBuf tc_xhi, tc_xlo;   // tf32 hi / lo planes of the image (built on first use)
    size_t tc_bpk_bytes = 0;
    DevBuf dsmall;    // device scratch for small double matrices
    std::vector<int32_t> lmap_host;   // 𝔏 positions (box indices) in lex order
    FftOperator *fft = nullptr;       // FFT correlation path (null if not built)

    // ---- decomposition ------------------------------------------------------
    int r = 0;
    std::vector<double> sigma;
    std::vector<double> residuals;   // per-triple residual bounds ||Xᵀu_i − σ_i v_i|| of the last decomposition
    DevBuf U;          // T[L*r]
    DevBuf V;          // T[K*r] (valid if v_valid)
    bool v_valid = false;
    std::vector<char> v_have;   // per-column validity of V when !v_valid (reconstruction computes only used columns)
    ssa_decomp_info last_info{};

    size_t elem() const { return dt == SSA_F64 ? 8 : 4; }
    ~PlanImpl();
};

// the implementation behind an ABI handle (api.cu); throws SSA_ERR_CUDA for a broken plan
PlanImpl &ssa_plan_impl(ssa_plan p);

// product dispatch (api.cu)
template <typename T>
void op_xv(PlanImpl &p, const T *V, int64_t ldv, T *U, int64_t ldu, int k);    // U = X V
template <typename T>
void op_xtu(PlanImpl &p, const T *U, int64_t ldu, T *V, int64_t ldv, int k,
            const double *cs = nullptr);   // V = Xᵀ U (column j times cs[j] if cs: device array of k)
double *small_dev(PlanImpl &p, size_t n_doubles);

// solver.cu
double sigma_floor(const PlanImpl &p);   // reading Q10: measured σ floor τ of the plan's product paths
// eigen.cu: svd.method = "eigen": S = XXᵀ by the fast products, full eigendecomposition
template <typename T>
void decompose_eigen(PlanImpl &p, int r, ssa_decomp_info *info);
template <typename T>
void decompose(PlanImpl &p, int r, ssa_decomp_info *info);
void release_workspace();   // the calling thread's grow-only K-side solver buffers (solver.cu)

// fft.cu
bool fft_supported(const PlanImpl &p);
void fft_build(PlanImpl &p);
template <typename T>
void fft_xv(PlanImpl &p, const T *V, int64_t ldv, T *U, int64_t ldu, int k);
template <typename T>
void fft_xtu(PlanImpl &p, const T *U, int64_t ldu, T *V, int64_t ldv, int k, const double *cs = nullptr);
template <typename T>
void fft_diagsums(PlanImpl &p, const T *U, const T *V, const double *sig_dev, const int *grp_off_dev,
                  const int *grp_idx_dev, int ng, const std::vector<int> &used, const int *slot_dev, T *out,
                  const int *wdiv);   // wdiv: hit counts of the ÷𝕎 epilogue
void fft_destroy(FftOperator *f);

}  // namespace ssa
