/*
 * ssa_b200.h — C ABI of the B200-native hot path of multidimensional singular
 * spectrum analysis (2D-SSA, MSSA, Shaped 2D-SSA) of arXiv 1309.5050
 * (Golyandina, Korobeynikov, Shlemov, Usevich, "Multivariate and 2D extensions
 * of singular spectrum analysis with the Rssa package").
 *
 * The four steps of the method (Fig. 1 / §2.1) map onto the calls:
 *   1. Embedding        ssa_plan_create      (𝒯 of eq. P:3004-3028: shapes 𝔑, 𝔏, 𝔎)
 *   2. SVD              ssa_decompose        (top-r eigentriples)
 *   3. Grouping         ssa_reconstruct args (index sets I_g)
 *   4. Reconstruction   ssa_reconstruct      (diagonal averaging, Alg. 4)
 * plus the trajectory-operator products themselves (ssa_matmul: X·V and Xᵀ·U,
 * Alg. 1/3 P:3643-3662) that drive step 2.
 *
 * CONVENTIONS (all entry points)
 *  - Arrays are column-major with x fastest: element (i, j) of an Nx x Ny array
 *    is at i + ld*j.  This is the paper's vec(); x is the paper's
 *    first (downward) axis, y the second.  Indices are 0-based.
 *  - MSSA is the 2D packing of P:3340-3354: pass an N_max x s array
 *    whose columns are the series (NaN-padded to equal length) and the window
 *    (L, 1).  No separate entry point.
 *  - Shapes: 𝔑 = {finite cells} ∩ mask; 𝔏 = wmask;
 *    𝔎 = {κ : 𝔏 +‐ {κ} ⊆ 𝔑} (eq. P:3004-3005).  Window cells and origins are
 *    ordered lexicographically (x fastest); L = |𝔏|, K = |𝔎|.
 *  - L-side vectors (eigenvectors U, "eigenarrays" P:2443-2456) have L entries in
 *    𝔏-lex order; K-side vectors (factor vectors V) have K entries in 𝔎-lex
 *    order.  Blocks of k vectors are column-major with leading dimension L or K.
 *  - Element type: the plan's dtype (SSA_F32 or SSA_F64) for every array
 *    argument unless stated otherwise; singular values are always double.
 *  - on_device: 1 = the pointer is CUDA device memory of the plan's device,
 *    0 = host memory (copied through pageable/pinned staging inside the call).
 *  - Every call is stream-ordered on opts.stream and returns after the stream
 *    has completed the work (synchronous), except ssa_matmul with
 *    on_device = 1, which only enqueues (the caller synchronises).
 *  - Ownership: the plan deep-copies its inputs; the caller may free them after
 *    ssa_plan_create.  The plan owns every device buffer it allocates.  Outputs
 *    go to caller buffers.  A plan is not thread-safe; distinct plans are
 *    independent.
 *  - Errors: every entry point returns an ssa_status; ssa_last_error() gives a
 *    thread-local message for the last failure.  No exception crosses the ABI.
 *    SSA_ERR_CUDA and SSA_ERR_COMM are sticky: the plan must be destroyed.
 *    There is NO CPU fallback: without a usable CUDA device every compute entry
 *    point fails with SSA_ERR_CUDA.
 */
#ifndef SSA_B200_H
#define SSA_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    SSA_OK = 0,
    SSA_ERR_ARG = 1,            /* bad pointer / size / dtype / group index */
    SSA_ERR_WINDOW = 2,         /* not 1<=Lx<=Nx, 1<=Ly<=Ny, 1<Lx*Ly<Nx*Ny */
    SSA_ERR_EMPTY_KSHAPE = 3,   /* 𝔎 = ∅: no window position fits inside 𝔑 */
    SSA_ERR_RANK = 4,           /* r < 1 or r > min(L, K), or a group index >= r */
    SSA_ERR_NOT_CONVERGED = 5,  /* decomposition hit max_iter; info->n_converged says how many */
    SSA_ERR_OOM = 6,            /* device allocation failed */
    SSA_ERR_CUDA = 7,           /* CUDA runtime / launch error, or no device (sticky) */
    SSA_ERR_COMM = 8,           /* collective callback failed (sticky) */
    SSA_ERR_STATE = 9           /* call out of order (e.g. reconstruct before decompose) */
} ssa_status;

typedef enum { SSA_F32 = 0, SSA_F64 = 1 } ssa_dtype;

/* Product path.  AUTO picks per shape. */
typedef enum {
    SSA_PATH_AUTO = 0,
    SSA_PATH_DIRECT = 1,   /* smem-tiled implicit GEMM on CUDA cores (Hankel sliding window) */
    SSA_PATH_FFT = 2,      /* shared-memory radix FFT circular correlation (Alg. 1/3) */
    SSA_PATH_TC = 3        /* tcgen05 tensor-core implicit GEMM, 3xTF32 split (fp32 plans; products
                              whose output box has < 256 rows fall back to FFT / direct) */
} ssa_path;

/* Decomposition method (the user's choice is always honoured). */
typedef enum {
    SSA_SVD_LANCZOS = 0,   /* block Golub-Kahan-Lanczos truncated SVD (default) */
    SSA_SVD_EIGEN = 1      /* "eigen": S = XXᵀ by the fast products, full
                              eigendecomposition of S (L <= 768); squares the condition number */
} ssa_svd_method;

typedef struct {
    int64_t nx, ny;        /* array size Nx x Ny (Ny = number of series for MSSA) */
    int64_t ld;            /* leading dimension >= nx; 0 means nx */
    ssa_dtype dtype;       /* element type of data; also the plan's arithmetic type */
    const void *data;      /* column-major; NaN = missing cell */
    int on_device;
} ssa_array;

typedef struct {
    int32_t lx, ly;        /* window bounding box */
    const uint8_t *wmask;  /* host lx*ly column-major 0/1 mask of 𝔏; NULL = full rectangle */
} ssa_window;

/* Collective hook for the window-position (𝔎) band partition.
 * allreduce_sum must sum `count` elements of type `dtype` in place across all
 * ranks (device buffer, stream-ordered on `stream`) and return 0 on success. */
typedef struct {
    int rank, world;
    void *user;
    int (*allreduce_sum)(void *user, void *dev_buf, int64_t count, int dtype, void *stream);
} ssa_comm;

typedef struct {
    void *stream;          /* cudaStream_t; NULL = the legacy default stream */
    int path;              /* ssa_path (0 = auto) */
    int block_k;           /* Lanczos block width (0 = auto: 16 for f64, 32 for f32) */
    double tol;            /* residual tolerance ||Xᵀu - σv|| <= tol*σ_1 (0 = auto) */
    int max_products;      /* cap on block products in ssa_decompose (0 = auto) */
    uint64_t seed;         /* seed of the Lanczos start block (counter-based RNG) */
    const ssa_comm *comm;  /* NULL = single GPU */
    int64_t band_y0, band_y1; /* band plans (comm != NULL, world > 1): this rank's global origin columns
                                 [y0, y1); x is then the sub-image of global columns [y0, y1 + Ly − 1)
                                 (band + (Ly−1)-column halo) */
    int precision;         /* arithmetic type of the plan: 0 = the input's dtype, 1 = fp32, 2 = fp64
                              (the input is cast once at plan creation); SSA_ERR_ARG otherwise */
    int64_t ny_global;     /* band plans: number of columns of the global image */
    int svd_method;        /* ssa_svd_method (0 = Lanczos) */
} ssa_opts;

typedef struct {
    int64_t nx, ny, lx, ly, kx, ky;   /* array, window box, origin box (kx = nx-lx+1) */
    int64_t L, K;                     /* |𝔏|, |𝔎| */
    int64_t n_valid;                  /* |𝔑| */
    int64_t n_excluded;               /* |𝔑 \ 𝔑′| (cells that enter no window) */
    int path;                         /* path chosen for X·V (kept for compatibility) */
    int dtype;
    int full_window, full_kshape;     /* 1 if 𝔏 / 𝔎 are full rectangles (trivial-mask fast path) */
    int path_xv, path_xtu;            /* ssa_path chosen for X·V and for Xᵀ·U (AUTO: measured per shape) */
} ssa_plan_info_t;

typedef struct {
    int32_t r_requested, n_converged;
    int32_t block_k, n_restarts;
    int64_t n_block_products;         /* Xᵀ·U plus X·V block calls */
    int64_t n_vector_products;        /* vectors pushed through the operator */
    double max_rel_residual;          /* max_i ||Xᵀu_i - σ_i v_i|| / σ_1 over i < r */
    double ms_products, ms_total;     /* device time in products; wall time of the call */
    double ms_ritz;                   /* host time in the projected (Ritz) SVDs */
    double ms_products_xv, ms_products_xtu;   /* device time of the X·V / Xᵀ·U block products */
    int64_t n_products_xv, n_products_xtu;    /* block products of each kind */
    int64_t n_vectors_xv, n_vectors_xtu;      /* vectors pushed through each product */
    /* reading Q10: the σ floor τ of the product path (σ_i < τ·σ_1 cannot be resolved
     * in the path's arithmetic; τ measured on the noiseless twins) and how many returned triples lie
     * below it */
    double sigma_floor_rel;
    int32_t n_below_floor;
    int32_t warm_start_cols;          /* start-block columns taken from the previous decomposition */
    double drop_norm_rel;             /* norm of block columns discarded as numerically zero, / ||X|| */
} ssa_decomp_info;

typedef struct ssa_plan_s *ssa_plan;

/* Step 1 (embedding, P:334-376 / eq. P:3004-3028).  Validates sizes
 * (SSA_ERR_WINDOW), builds 𝔑 = finite ∩ mask (mask: host nx*ny 0/1 or NULL),
 * 𝔏 = wmask, 𝔎 by Alg. 6, the hit-count weights 𝕎 =
 * diagsums(1_𝔏, 1_𝔎) (Alg. 4 step 1) and the per-path operator data.
 * Returns SSA_ERR_EMPTY_KSHAPE if 𝔎 = ∅. */
ssa_status ssa_plan_create(const ssa_array *x, const ssa_window *w, const uint8_t *mask,
                           const ssa_opts *opts, ssa_plan *out);
void ssa_plan_destroy(ssa_plan p);
ssa_status ssa_plan_info(ssa_plan p, ssa_plan_info_t *info);

/* Plan-time shapes: weights w_n = |𝒜_n| (int32 nx*ny, column-major; Rssa
 * "$weights"; 0 outside 𝔑′) and the 𝔎 indicator over the kx*ky origin box. */
ssa_status ssa_get_weights(ssa_plan p, int32_t *w, int on_device);
ssa_status ssa_get_kmask(ssa_plan p, uint8_t *kmask, int on_device);

/* The trajectory-operator products on a block of k vectors (never forming X):
 *   transpose = 0 :  out (L x k) = X · in (K x k)    u_ℓ = Σ_{κ∈𝔎} x[ℓ +‐ κ] v_κ
 *   transpose = 1 :  out (K x k) = Xᵀ · in (L x k)   v_κ = Σ_{ℓ∈𝔏} x[ℓ +‐ κ] u_ℓ
 * (rows/columns of eq. P:3020-3028; Alg. 1 P:3647-3658 and its transpose P:3659-3662;
 * Alg. 3 P:3838-3847 under reading Q1).  ldin/ldout 0 = packed.  With on_device = 1
 * the call only enqueues on opts.stream. */
ssa_status ssa_matmul(ssa_plan p, int transpose, const void *in, int64_t ldin,
                      void *out, int64_t ldout, int64_t k, int on_device);

/* Step 2: top-r eigentriples (σ_i, U_i, V_i) of X by block Golub-Kahan-Lanczos
 * bidiagonalisation with thick restarts, σ descending.  Converged means
 * ||Xᵀu_i − σ_i v_i|| <= tol·σ_1 for all i < r (residual bounds: ssa_get_residuals).  Called again
 * on a plan that holds a decomposition (e.g. with a larger r), the Lanczos start block is warm-started
 * from the stored eigenvectors U_1..U_min(r_prev, k) ("automatically continued").
 * SSA_ERR_NOT_CONVERGED when max_products is reached first (the r triples are still returned,
 * with their residual bounds).  info may be NULL. */
ssa_status ssa_decompose(ssa_plan p, int32_t r, ssa_decomp_info *info);

/* Getters (valid after ssa_decompose or ssa_set_triples).  sigma: r doubles.
 * U: L x r.  V: K x r, V_i = Xᵀ U_i / σ_i recomputed on request (P:383,
 * P:1720-1723).  Signs: the largest-|.| entry of each U_i is positive. */
ssa_status ssa_get_rank(ssa_plan p, int32_t *r);
ssa_status ssa_get_sigma(ssa_plan p, double *sigma);
/* Per-triple residual bounds ||Xᵀu_i − σ_i v_i|| (r doubles, absolute) of the last decomposition.
 * When the final convergence check was taken with the K-side orthonormalisation of the last block
 * deferred, the bounds use A_last ≈ R₁ (the pass-1 Cholesky factor) and convergence was
 * only accepted with every bound below tol·σ_1 / 2. */
ssa_status ssa_get_residuals(ssa_plan p, double *res);
ssa_status ssa_get_u(ssa_plan p, void *U, int on_device);
ssa_status ssa_get_v(ssa_plan p, void *V, int on_device);

/* Install externally computed triples (e.g. to reconstruct from a stored
 * decomposition).  U: L x r; V may be NULL (then V = XᵀU/σ). */
ssa_status ssa_set_triples(ssa_plan p, int32_t r, const double *sigma, const void *U,
                           const void *V, int on_device);

/* Steps 3-4.  Groups in CSR form: group g = grp_idx[grp_off[g] .. grp_off[g+1]),
 * 0-based eigentriple indices < r.  out: (n_groups + add_rest) arrays of nx*ny
 * (column-major, ld = nx), each  X̃_g = diagsums(Σ_{i∈I_g} σ_i U_i V_iᵀ) / 𝕎  on 𝔑′
 * and NaN elsewhere (Alg. 4; values exist only inside 𝔑′,
 * P:3214-3217).  add_rest appends 𝕏 − Σ_g X̃_g on 𝔑′ (eq. P:440-443).
 * A group index >= the computed rank continues the decomposition first (decompose(max index + 1),
 * P:869-873); SSA_ERR_RANK if an index is >= min(L, K). */
ssa_status ssa_reconstruct(ssa_plan p, const int32_t *grp_off, const int32_t *grp_idx,
                           int32_t n_groups, int add_rest, void *out, int on_device);

/* w-correlation matrix of the groups' reconstructions:
 * rho (n_groups x n_groups, column-major double) = (X̃_a, X̃_b)_w / (‖X̃_a‖_w ‖X̃_b‖_w), with the
 * weighted inner product (Y, Z)_w = Σ_n w_n y_n z_n; and, when contrib is non-NULL,
 * the contributions ‖X̃_g‖²_w / ‖𝕏‖²_w (n_groups doubles).  1 <= n_groups <= 63. */
ssa_status ssa_wcor(ssa_plan p, const int32_t *grp_off, const int32_t *grp_idx,
                    int32_t n_groups, double *rho, double *contrib);

/* Parameter estimation: LS-ESPRIT / 2D-ESPRIT on the
 * eigenvectors U_i, i ∈ idx[0..n) (n <= 64, indices < the computed rank): shift matrices Φ_x, Φ_y
 * (least squares between the eigenarrays restricted to 𝔏 and to 𝔏 shifted by one cell along x / y)
 * and their joint diagonalisation.  lambda, mu: n complex values each (re, im interleaved: 2n
 * doubles), the pairs (λ_k, μ_k) of x_{m,n} = Σ_k c_k λ_k^m μ_k^n; mu may be NULL; for a window of one
 * column mu = 1.  The order of the pairs is unspecified. */
ssa_status ssa_esprit(ssa_plan p, const int32_t *idx, int32_t n, double *lambda, double *mu);

/* Vector forecast (Alg. 7 fast column vector forecast, of the vector
 * MSSA forecast P:1416-1460): 1-D SSA / MSSA plans (window (L, 1), series = columns, NaN-padded at
 * the end).  For every series p the reconstruction of the group idx (eigenvectors P = U_idx, lagged
 * vectors W_k = (σ_i V_i[κ_k])) is continued by W_k = D W_{k−1}, D = the LS-ESPRIT shift matrix,
 * and hankelized: out (ld_out >= nx + M, one column per series, plan dtype) receives z_1 .. z_{N_p+M}
 * (the reconstruction updated near the end, then M forecast values) and NaN below.  SSA_ERR_ARG for
 * other plans, band plans, or series whose window positions are not a contiguous prefix. */
ssa_status ssa_forecast(ssa_plan p, const int32_t *idx, int32_t n, int32_t M, void *out, int64_t ld_out,
                        int on_device);

/* The solver's projected-matrix SVD as a utility: one-sided
 * block Jacobi in fp64 on the device (one thread-block cluster for n <= 256, a
 * cooperative grid above), for m >= n, m <= 768.  A (host, m x n column-major)
 * is overwritten with A·J whose columns are σ_j·y_j (unsorted); sweeps and
 * device milliseconds are returned when the pointers are non-NULL.
 * SSA_ERR_ARG if the matrix does not fit. */
ssa_status ssa_small_svd(int32_t m, int32_t n, double *A, int32_t *sweeps, double *ms);

/* Micro-benchmark of the solver's tall-skinny fp32 kernels on seeded device data
 * (test / tuning hook, no host data): which = 0 times the Gram G = AᵀB (A: M x n1,
 * B: M x n2, n1 <= 512, n2 <= 64), which = 1 the update W -= A·C (A: M x n1,
 * W: M x n2).  Leading dimension M rounded up to 32 (the solver's layout).
 * *ms = average device milliseconds over `reps` launches after one warm-up;
 * *check = max relative error against an fp64 host evaluation (update: on ~1000 sampled
 * rows; Gram: all entries when M·n1·n2 <= 5e8, else the checksum Σ|G|).  which = 3 times
 * the self Gram AᵀA[:, :n2]; which = 4 times a TMA streaming probe of n1 <= 128 columns in
 * boxes of |n2| rows (n2 = 32: 128-B swizzled, else unswizzled; 128 rows per stage or one box);
 * which = 5 times the projection Gram AᵀB with B = the last n2 columns of A (n2 <= n1).
 * SSA_ERR_ARG on bad sizes. */
ssa_status ssa_bench_tall(int32_t which, int64_t M, int32_t n1, int32_t n2, int32_t reps, double *ms,
                          double *check);

/* Measured tensor-core peak (roofline denominator of the tcgen05 kernels): `ctas` CTAs (0 = one per
 * SM) each issue `iters` back-to-back tcgen05.mma kind::tf32 M=128 N=256 K=8 from shared memory.
 * *ms = device time, *tflops = dense tf32 TFLOP/s (2·128·256·8 per MMA). */
ssa_status ssa_bench_mma(int32_t iters, int32_t ctas, double *ms, double *tflops);

/* Release the calling thread's solver workspace.  The K-side Lanczos basis and its restart copy
 * (ssa_decompose; c5: 15 + 9 GB) are kept per host thread across decompositions and plans, grow-only,
 * so that repeated plan / decompose / destroy cycles reuse them instead of fragmenting the
 * stream-ordered memory pool; this call frees them (they are also freed at thread exit).  It also
 * empties the thread's cache of large freed device blocks: every internal buffer of 8 MB or more is
 * kept, when freed, for the next allocation of exactly that size on this thread (at most 64 GB in all,
 * oldest returned to the pool first), so that steady-state plans of one shape never go back to the
 * pool allocator.  Safe to call at any time outside a running ssa_decompose on the same thread; SSA_OK. */
ssa_status ssa_release_workspace(void);

const char *ssa_last_error(void);
const char *ssa_version(void);
/* Number of kernels this library launched on the calling thread since the last
 * reset (evidence counter for bench.py's gpu_launches). */
int64_t ssa_launch_count(int reset);

#ifdef __cplusplus
}
#endif
#endif /* SSA_B200_H */
