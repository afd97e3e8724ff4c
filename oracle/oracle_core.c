/*
 * ORACLE — TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, obviously-correct fp64 CPU loops for the multidimensional-SSA hot
 * path of arXiv 1309.5050 (Golyandina, Korobeynikov, Shlemov, Usevich), written
 * from PAPER.md.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  It shares no code
 * with the CUDA path (paper_1309_5050_b200/) and must never be linked into it.
 *
 * No FFT, no blocking, no reordering: every function is the definition written
 * out as a loop nest (OpenMP only splits the outermost loop over outputs).
 *
 * Conventions:
 *  - Arrays are column-major with x fastest: element (i, j) of an nx x ny array is
 *    at i + nx*j.  This is the paper's vec().  Indices are 0-based,
 *    so the paper's shifted sum  l +- k = (lx+kx-1, ly+ky-1)
 *    becomes plain addition  (lx+kx, ly+ky).
 *  - Shapes are uint8 masks.  The window shape L (wmask, lx x ly box) and the
 *    origin shape K (kmask, kx x ky box, kx = nx-lx+1, ky = ny-ly+1) are ordered
 *    lexicographically = column-major order of their boxes.
 *  - Vectors on the L side have |L| entries in L-lex order; vectors on the K
 *    side have |K| entries in K-lex order; blocks of k vectors are |L| x k or
 *    |K| x k column-major.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* Enumerate the set cells of a bx x by mask in lexicographic (column-major)
 * order.  Returns the count; px/py receive coordinates (caller frees). */
static int64_t enum_shape(int64_t bx, int64_t by, const uint8_t *m,
                          int64_t **px, int64_t **py) {
    int64_t n = 0;
    for (int64_t t = 0; t < bx * by; ++t) n += (m == NULL) ? 1 : (m[t] != 0);
    *px = (int64_t *)malloc(sizeof(int64_t) * (n ? n : 1));
    *py = (int64_t *)malloc(sizeof(int64_t) * (n ? n : 1));
    int64_t c = 0;
    for (int64_t j = 0; j < by; ++j)
        for (int64_t i = 0; i < bx; ++i)
            if (m == NULL || m[i + bx * j]) { (*px)[c] = i; (*py)[c] = j; ++c; }
    return n;
}

/* 𝔎 = { κ : 𝔏 +‐ {κ} ⊆ 𝔑 }   (eq. P:3004-3005), by brute force over the
 * (nx-lx+1) x (ny-ly+1) box of origins.  nmask: nx*ny, wmask: lx*ly (NULL = full
 * rectangle), kmask_out: kx*ky.  Returns |𝔎|. */
int64_t orc_kshape(int64_t nx, int64_t ny, const uint8_t *nmask,
                   int64_t lx, int64_t ly, const uint8_t *wmask, uint8_t *kmask_out) {
    int64_t kx = nx - lx + 1, ky = ny - ly + 1;
    int64_t *lpx, *lpy;
    int64_t L = enum_shape(lx, ly, wmask, &lpx, &lpy);
    int64_t count = 0;
    #pragma omp parallel for reduction(+:count) schedule(static)
    for (int64_t b = 0; b < ky; ++b) {
        for (int64_t a = 0; a < kx; ++a) {
            int ok = 1;
            for (int64_t q = 0; q < L; ++q) {
                int64_t i = lpx[q] + a, j = lpy[q] + b;
                if (!nmask[i + nx * j]) { ok = 0; break; }
            }
            kmask_out[a + kx * b] = (uint8_t)ok;
            count += ok;
        }
    }
    free(lpx); free(lpy);
    return count;
}

/* Weights w_n = |𝒜_n| = ||𝒯(E_n)||_F^2 = #{(ℓ, κ) ∈ 𝔏 x 𝔎 : ℓ +‐ κ = n}
 * (Alg. 4 step 1 P:3886).  w_out: nx*ny int32. */
void orc_weights(int64_t nx, int64_t ny, int64_t lx, int64_t ly, const uint8_t *wmask,
                 const uint8_t *kmask, int32_t *w_out) {
    int64_t kx = nx - lx + 1, ky = ny - ly + 1;
    int64_t *lpx, *lpy, *kpx, *kpy;
    int64_t L = enum_shape(lx, ly, wmask, &lpx, &lpy);
    int64_t K = enum_shape(kx, ky, kmask, &kpx, &kpy);
    memset(w_out, 0, sizeof(int32_t) * nx * ny);
    for (int64_t c = 0; c < K; ++c)
        for (int64_t q = 0; q < L; ++q)
            w_out[(lpx[q] + kpx[c]) + nx * (lpy[q] + kpy[c])] += 1;
    free(lpx); free(lpy); free(kpx); free(kpy);
}

/* Materialise the trajectory (quasi-Hankel) matrix, columns kstart..kstart+kcount-1
 * of 𝒯(𝕏):  X[q, c] = x[ℓ_q +‐ κ_c]   (eq. P:3020-3028; for full shapes this is the
 * HbH matrix of eq. P:2411-2419).  out: L x kcount column-major. */
void orc_trajcols(const double *x, int64_t nx, int64_t ny, int64_t lx, int64_t ly,
                  const uint8_t *wmask, const uint8_t *kmask,
                  int64_t kstart, int64_t kcount, double *out) {
    int64_t kx = nx - lx + 1, ky = ny - ly + 1;
    int64_t *lpx, *lpy, *kpx, *kpy;
    int64_t L = enum_shape(lx, ly, wmask, &lpx, &lpy);
    (void)enum_shape(kx, ky, kmask, &kpx, &kpy);
    #pragma omp parallel for schedule(static)
    for (int64_t c = 0; c < kcount; ++c) {
        int64_t a = kpx[kstart + c], b = kpy[kstart + c];
        for (int64_t q = 0; q < L; ++q)
            out[q + L * c] = x[(lpx[q] + a) + nx * (lpy[q] + b)];
    }
    free(lpx); free(lpy); free(kpx); free(kpy);
}

/* L-side product  U = X V :  u_ℓ = Σ_{κ∈𝔎} x[ℓ +‐ κ] v_κ  for each of k vectors
 * (rows of eq. P:3020-3028; the operation of Alg. 1/3, P:3647-3658, P:3838-3847,
 * written as its plain definition).  V: |𝔎| x k, U: |𝔏| x k (column-major). */
void orc_xv(const double *x, int64_t nx, int64_t ny, int64_t lx, int64_t ly,
            const uint8_t *wmask, const uint8_t *kmask,
            const double *V, int64_t k, double *U) {
    int64_t kx = nx - lx + 1, ky = ny - ly + 1;
    int64_t *lpx, *lpy, *kpx, *kpy;
    int64_t L = enum_shape(lx, ly, wmask, &lpx, &lpy);
    int64_t K = enum_shape(kx, ky, kmask, &kpx, &kpy);
    #pragma omp parallel for schedule(static)
    for (int64_t q = 0; q < L; ++q) {
        for (int64_t v = 0; v < k; ++v) {
            double s = 0.0;
            for (int64_t c = 0; c < K; ++c)
                s += x[(lpx[q] + kpx[c]) + nx * (lpy[q] + kpy[c])] * V[c + K * v];
            U[q + L * v] = s;
        }
    }
    free(lpx); free(lpy); free(kpx); free(kpy);
}

/* K-side product  V = Xᵀ U :  v_κ = Σ_{ℓ∈𝔏} x[ℓ +‐ κ] u_ℓ   ("the same algorithm
 * suits for multiplication by the transpose").  Only the K-side
 * rows listed in [kstart, kstart+kcount) are produced (kcount = |𝔎| for all);
 * this lets the tests sample rows at sizes where the full product is too slow.
 * U: |𝔏| x k, Vout: kcount x k. */
void orc_xtu_rows(const double *x, int64_t nx, int64_t ny, int64_t lx, int64_t ly,
                  const uint8_t *wmask, const uint8_t *kmask,
                  const double *U, int64_t k, int64_t kstart, int64_t kcount, double *Vout) {
    int64_t kx = nx - lx + 1, ky = ny - ly + 1;
    int64_t *lpx, *lpy, *kpx, *kpy;
    int64_t L = enum_shape(lx, ly, wmask, &lpx, &lpy);
    (void)enum_shape(kx, ky, kmask, &kpx, &kpy);
    #pragma omp parallel for schedule(static)
    for (int64_t c = 0; c < kcount; ++c) {
        int64_t a = kpx[kstart + c], b = kpy[kstart + c];
        for (int64_t v = 0; v < k; ++v) {
            double s = 0.0;
            for (int64_t q = 0; q < L; ++q)
                s += x[(lpx[q] + a) + nx * (lpy[q] + b)] * U[q + L * v];
            Vout[c + kcount * v] = s;
        }
    }
    free(lpx); free(lpy); free(kpx); free(kpy);
}

/* L-side product restricted to listed rows: like orc_xv but only for the window
 * cells with L-lex positions in rows[0..nrows) (sampled-row checks at sizes
 * where the full product is too slow).  Uout: nrows x k. */
void orc_xv_rows(const double *x, int64_t nx, int64_t ny, int64_t lx, int64_t ly,
                 const uint8_t *wmask, const uint8_t *kmask,
                 const double *V, int64_t k, const int64_t *rows, int64_t nrows, double *Uout) {
    int64_t kx = nx - lx + 1, ky = ny - ly + 1;
    int64_t *lpx, *lpy, *kpx, *kpy;
    (void)enum_shape(lx, ly, wmask, &lpx, &lpy);
    int64_t K = enum_shape(kx, ky, kmask, &kpx, &kpy);
    #pragma omp parallel for schedule(static)
    for (int64_t t = 0; t < nrows * k; ++t) {
        int64_t rr = t % nrows, v = t / nrows;
        int64_t q = rows[rr];
        double s = 0.0;
        for (int64_t c = 0; c < K; ++c)
            s += x[(lpx[q] + kpx[c]) + nx * (lpy[q] + kpy[c])] * V[c + K * v];
        Uout[rr + nrows * v] = s;
    }
    free(lpx); free(lpy); free(kpx); free(kpy);
}

/* diagsums of a sum of rank-one terms (Alg. 5 definition, with the
 * numerator of P:3862-3872):
 *    out_n = Σ_{i<r} coef_i Σ_{(ℓ,κ) ∈ 𝔏x𝔎, ℓ +‐ κ = n} U_i[ℓ] V_i[κ]
 * i.e. <Σ_i coef_i U_i V_iᵀ, 𝒯(E_n)>_F.  U: |𝔏| x r, V: |𝔎| x r, out: nx*ny.
 * Brute force: every (ℓ, κ) pair of the trajectory matrix is visited once and
 * added to its cell (the sets 𝒜_n of P:355-360). */
void orc_diagsums(int64_t nx, int64_t ny, int64_t lx, int64_t ly,
                  const uint8_t *wmask, const uint8_t *kmask,
                  const double *U, const double *V, const double *coef, int64_t r,
                  double *out) {
    int64_t kx = nx - lx + 1, ky = ny - ly + 1;
    int64_t *lpx, *lpy, *kpx, *kpy;
    int64_t L = enum_shape(lx, ly, wmask, &lpx, &lpy);
    int64_t K = enum_shape(kx, ky, kmask, &kpx, &kpy);
    memset(out, 0, sizeof(double) * nx * ny);
    /* 𝔎 is in lex order, so the origins with κy = b form the contiguous run
     * [kcol[b], kcol[b+1]).  Split by output column j: each thread owns whole
     * columns of `out` and visits exactly the pairs (ℓ, κ) with ℓy + κy = j, so
     * every pair of 𝔏 x 𝔎 is visited once overall. */
    int64_t *kcol = (int64_t *)calloc(ky + 1, sizeof(int64_t));
    for (int64_t c = 0; c < K; ++c) kcol[kpy[c] + 1] += 1;
    for (int64_t b = 0; b < ky; ++b) kcol[b + 1] += kcol[b];
    #pragma omp parallel for schedule(dynamic, 1)
    for (int64_t j = 0; j < ny; ++j) {
        for (int64_t q = 0; q < L; ++q) {
            int64_t b = j - lpy[q];
            if (b < 0 || b >= ky) continue;
            for (int64_t c = kcol[b]; c < kcol[b + 1]; ++c) {
                double s = 0.0;
                for (int64_t i = 0; i < r; ++i) s += coef[i] * U[q + L * i] * V[c + K * i];
                out[(lpx[q] + kpx[c]) + nx * j] += s;
            }
        }
    }
    free(kcol);
    free(lpx); free(lpy); free(kpx); free(kpy);
}

/* diagsums at listed cells only (sampled checks at full sizes):
 *   out[t] = Σ_i coef_i Σ_{ℓ∈𝔏, κ = n_t − ℓ ∈ 𝔎} U_i[ℓ] V_i[κ]
 * where V_i[κ] must be supplied for every κ ∈ 𝔎 (|𝔎| x r).  cells: flat indices
 * i + nx*j. */
void orc_diagsums_cells(int64_t nx, int64_t ny, int64_t lx, int64_t ly,
                        const uint8_t *wmask, const uint8_t *kmask,
                        const double *U, const double *V, const double *coef, int64_t r,
                        const int64_t *cells, int64_t ncells, double *out) {
    int64_t kx = nx - lx + 1, ky = ny - ly + 1;
    int64_t *lpx, *lpy, *kpx, *kpy;
    int64_t L = enum_shape(lx, ly, wmask, &lpx, &lpy);
    int64_t K = enum_shape(kx, ky, kmask, &kpx, &kpy);
    /* position of each box cell in 𝔎-lex order (-1 if not in 𝔎) */
    int64_t *kpos = (int64_t *)malloc(sizeof(int64_t) * kx * ky);
    for (int64_t t = 0; t < kx * ky; ++t) kpos[t] = -1;
    for (int64_t c = 0; c < K; ++c) kpos[kpx[c] + kx * kpy[c]] = c;
    #pragma omp parallel for schedule(static)
    for (int64_t t = 0; t < ncells; ++t) {
        int64_t n = cells[t], ni = n % nx, nj = n / nx;
        double acc = 0.0;
        for (int64_t q = 0; q < L; ++q) {
            int64_t a = ni - lpx[q], b = nj - lpy[q];
            if (a < 0 || b < 0 || a >= kx || b >= ky) continue;
            int64_t c = kpos[a + kx * b];
            if (c < 0) continue;
            for (int64_t i = 0; i < r; ++i) acc += coef[i] * U[q + L * i] * V[c + K * i];
        }
        out[t] = acc;
    }
    free(kpos); free(lpx); free(lpy); free(kpx); free(kpy);
}
