// Host-side dense kernels of the CholeskyQR projection (see hostla.h): register-blocked dot
// products over contiguous columns (CᵀC), axpys over contiguous columns (the projection
// coefficients), right-looking Cholesky and column-oriented triangular inverse — all
// vectorisable; built twice (baseline x86-64 and AVX2/FMA, chosen at run time).
#include "hostla.h"

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <vector>

namespace ssa {
namespace hostla {
namespace {

#define SSA_HOSTLA_BODY                                                                              \
    /* dots over contiguous t, 4 lanes, register-blocked 4 (a) x 2 (b) */                          \
    static void gram_minus_ctc_impl(int kc, int na, int nn, int off, const double *G, double *Gp) { \
        typedef double v4 __attribute__((vector_size(32)));                                          \
        for (int b0 = 0; b0 < kc; b0 += 2)                                                           \
            for (int a0 = 0; a0 <= b0 + 1 && a0 < kc; a0 += 4) {                                     \
                const double *ca[4], *cb[2];                                                         \
                for (int q = 0; q < 4; ++q) ca[q] = G + (long)nn * std::min(a0 + q, kc - 1);         \
                for (int q = 0; q < 2; ++q) cb[q] = G + (long)nn * std::min(b0 + q, kc - 1);         \
                v4 acc[4][2];                                                                        \
                for (int x = 0; x < 4; ++x)                                                          \
                    for (int y = 0; y < 2; ++y) acc[x][y] = (v4){0.0, 0.0, 0.0, 0.0};                \
                int t = 0;                                                                           \
                for (; t + 4 <= na; t += 4) {                                                        \
                    v4 xa[4], xb[2];                                                                 \
                    for (int q = 0; q < 4; ++q) std::memcpy(&xa[q], ca[q] + t, sizeof(v4));          \
                    for (int q = 0; q < 2; ++q) std::memcpy(&xb[q], cb[q] + t, sizeof(v4));          \
                    for (int x = 0; x < 4; ++x)                                                      \
                        for (int y = 0; y < 2; ++y) acc[x][y] += xa[x] * xb[y];                      \
                }                                                                                    \
                for (int x = 0; x < 4; ++x)                                                          \
                    for (int y = 0; y < 2; ++y) {                                                    \
                        const int aa = a0 + x, bb = b0 + y;                                          \
                        if (aa >= kc || bb >= kc || aa > bb) continue;                               \
                        double sum = (acc[x][y][0] + acc[x][y][1]) + (acc[x][y][2] + acc[x][y][3]);  \
                        for (int u = t; u < na; ++u) sum += ca[x][u] * cb[y][u];                     \
                        const double v = G[off + aa + (long)nn * bb] - sum;                          \
                        Gp[aa + (long)kc * bb] = v;                                                  \
                        Gp[bb + (long)kc * aa] = v;                                                  \
                    }                                                                                \
            }                                                                                        \
    }                                                                                                \
    static void proj_coef_impl(int kc, int na, int n1, const double *G, const double *S, double *Mc) { \
        for (int b = 0; b < kc; ++b) {                                                               \
            double *mc = Mc + (long)n1 * b;                                                          \
            for (int t = 0; t < na; ++t) mc[t] = 0.0;                                                \
            for (int a = 0; a <= b; ++a) {                                                           \
                const double sv = S[a + (long)kc * b], *ga = G + (long)n1 * a;                       \
                for (int t = 0; t < na; ++t) mc[t] -= ga[t] * sv;                                     \
            }                                                                                        \
            for (int a = 0; a < kc; ++a) mc[na + a] = S[a + (long)kc * b];                           \
        }                                                                                            \
    }                                                                                                \
    /* right-looking: every entry sees its updates in the left-looking (dot-product) order */       \
    static bool cholesky_upper_impl(int n, const double *G, double shift, double thr, double *R) {  \
        double dmax = 0.0;                                                                           \
        for (int j = 0; j < n; ++j) dmax = std::max(dmax, G[j + (long)n * j]);                      \
        if (!(dmax > 0.0)) return false;                                                             \
        for (int l = 0; l < n; ++l)                                                                  \
            for (int i = 0; i < n; ++i)                                                              \
                R[i + (long)n * l] = i < l ? G[i + (long)n * l] : (i == l ? G[i + (long)n * l] + shift : 0.0); \
        std::vector<double> row((size_t)n);                                                          \
        for (int j = 0; j < n; ++j) {                                                                \
            const double s = R[j + (long)n * j];                                                     \
            if (!(s > thr * dmax)) return false;                                                     \
            const double rjj = std::sqrt(s);                                                         \
            R[j + (long)n * j] = rjj;                                                                \
            for (int l = j + 1; l < n; ++l) row[l] = (R[j + (long)n * l] /= rjj);                    \
            for (int l = j + 1; l < n; ++l) {                                                        \
                const double rl = row[l];                                                            \
                double *cl = R + (long)n * l;                                                        \
                for (int i = j + 1; i <= l; ++i) cl[i] -= row[i] * rl;                               \
            }                                                                                        \
        }                                                                                            \
        return true;                                                                                 \
    }                                                                                                \
    static void upper_inverse_impl(int n, const double *R, double *S) {                              \
        for (long e = 0; e < (long)n * n; ++e) S[e] = 0.0;                                           \
        std::vector<double> acc((size_t)n);                                                          \
        for (int j = 0; j < n; ++j) {                                                                \
            double *s = S + (long)n * j;                                                             \
            for (int i = 0; i < j; ++i) acc[i] = 0.0;                                                \
            s[j] = 1.0 / R[j + (long)n * j];                                                         \
            for (int t = j; t > 0; --t) {                                                            \
                const double st = s[t], *rt = R + (long)n * t;                                       \
                for (int i = 0; i < t; ++i) acc[i] += rt[i] * st;                                    \
                s[t - 1] = -acc[t - 1] / R[(t - 1) + (long)n * (t - 1)];                              \
            }                                                                                        \
        }                                                                                            \
    }

namespace generic {
SSA_HOSTLA_BODY
}
#if defined(__x86_64__)
#pragma GCC push_options
#pragma GCC target("avx2,fma")
namespace avx2 {
SSA_HOSTLA_BODY
}
#pragma GCC pop_options
bool use_avx2() {
    static const bool v = __builtin_cpu_supports("avx2") && __builtin_cpu_supports("fma") &&
                          std::getenv("SSA_HOSTLA_GENERIC") == nullptr;   // (tests force the baseline build)
    return v;
}
#else
bool use_avx2() { return false; }
#endif
}  // namespace

void gram_minus_ctc(int kc, int na, int nn, int off, const double *G, double *Gp) {
#if defined(__x86_64__)
    if (use_avx2()) return avx2::gram_minus_ctc_impl(kc, na, nn, off, G, Gp);
#endif
    generic::gram_minus_ctc_impl(kc, na, nn, off, G, Gp);
}
void proj_coef(int kc, int na, int n1, const double *G, const double *S, double *Mc) {
#if defined(__x86_64__)
    if (use_avx2()) return avx2::proj_coef_impl(kc, na, n1, G, S, Mc);
#endif
    generic::proj_coef_impl(kc, na, n1, G, S, Mc);
}

bool cholesky_upper(int n, const double *G, double shift, double thr, double *R) {
#if defined(__x86_64__)
    if (use_avx2()) return avx2::cholesky_upper_impl(n, G, shift, thr, R);
#endif
    return generic::cholesky_upper_impl(n, G, shift, thr, R);
}
void upper_inverse(int n, const double *R, double *S) {
#if defined(__x86_64__)
    if (use_avx2()) return avx2::upper_inverse_impl(n, R, S);
#endif
    generic::upper_inverse_impl(n, R, S);
}

}  // namespace hostla
}  // namespace ssa
