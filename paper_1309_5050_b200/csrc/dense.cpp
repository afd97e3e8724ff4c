// Small dense fp64 linear algebra on the host for the block Lanczos solver
// ("mk x mk SVD (fp64)"): the projected matrix T is at most a
// few hundred columns.  Everything here is textbook:
//   * sym_eig      cyclic two-sided Jacobi for symmetric matrices (k x k Grams)
//   * svd_jacobi   one-sided (Hestenes) Jacobi SVD, parallel round-robin ordering;
//                  high relative accuracy of σ, no squaring of the spread
//                  (σ is never taken from eigenvalues of TᵀT, SURVEY finding 6).
#include "dense.h"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <numeric>
#include <vector>
#ifdef _OPENMP
#include <omp.h>
#endif

namespace ssa {

void sym_eig(int n, const double *A, double *lam, double *E) {
    std::vector<double> a(A, A + (size_t)n * n);
    for (int i = 0; i < n * n; ++i) E[i] = 0.0;
    for (int i = 0; i < n; ++i) E[i + (size_t)n * i] = 1.0;
    auto at = [&](int i, int j) -> double & { return a[i + (size_t)n * j]; };
    for (int sweep = 0; sweep < 60; ++sweep) {
        double off = 0.0, tot = 0.0;
        for (int j = 0; j < n; ++j)
            for (int i = 0; i < n; ++i) {
                tot += at(i, j) * at(i, j);
                if (i != j) off += at(i, j) * at(i, j);
            }
        if (off <= 1e-30 * tot || off == 0.0) break;
        for (int p = 0; p < n - 1; ++p)
            for (int q = p + 1; q < n; ++q) {
                const double apq = at(p, q);
                if (std::fabs(apq) < 1e-300) continue;
                const double app = at(p, p), aqq = at(q, q);
                const double theta = (aqq - app) / (2.0 * apq);
                const double t = (theta >= 0 ? 1.0 : -1.0) / (std::fabs(theta) + std::sqrt(1.0 + theta * theta));
                const double c = 1.0 / std::sqrt(1.0 + t * t), s = t * c;
                for (int k = 0; k < n; ++k) {   // A <- Jᵀ A J
                    const double akp = at(k, p), akq = at(k, q);
                    at(k, p) = c * akp - s * akq;
                    at(k, q) = s * akp + c * akq;
                }
                for (int k = 0; k < n; ++k) {
                    const double apk = at(p, k), aqk = at(q, k);
                    at(p, k) = c * apk - s * aqk;
                    at(q, k) = s * apk + c * aqk;
                }
                for (int k = 0; k < n; ++k) {
                    double *e = E;
                    const double ekp = e[k + (size_t)n * p], ekq = e[k + (size_t)n * q];
                    e[k + (size_t)n * p] = c * ekp - s * ekq;
                    e[k + (size_t)n * q] = s * ekp + c * ekq;
                }
            }
    }
    // sort descending
    std::vector<int> idx(n);
    std::iota(idx.begin(), idx.end(), 0);
    std::sort(idx.begin(), idx.end(), [&](int x, int y) { return at(x, x) > at(y, y); });
    std::vector<double> Ec(E, E + (size_t)n * n);
    for (int j = 0; j < n; ++j) {
        lam[j] = at(idx[j], idx[j]);
        std::memcpy(E + (size_t)n * j, Ec.data() + (size_t)n * idx[j], sizeof(double) * n);
    }
}

// One-sided Jacobi: rotate column pairs of A (m x n) until all are orthogonal;
// then σ_j = ||a_j||, Y_j = a_j / σ_j and Z accumulates the rotations.
void svd_jacobi(int m, int n, const double *M, int ldm, double *s, double *Y, double *Z) {
    const int nn = n + (n & 1);                 // round-robin needs an even count
    std::vector<double> A((size_t)m * nn, 0.0), V((size_t)n * nn, 0.0);
    for (int j = 0; j < n; ++j) {
        std::memcpy(&A[(size_t)m * j], M + (size_t)ldm * j, sizeof(double) * m);
        V[j + (size_t)n * j] = 1.0;
    }
    // de Rijk-style start: columns sorted by decreasing norm
    {
        std::vector<double> nrm(n);
        for (int j = 0; j < n; ++j) {
            double t = 0; for (int i = 0; i < m; ++i) t += A[i + (size_t)m * j] * A[i + (size_t)m * j];
            nrm[j] = t;
        }
        std::vector<int> idx(n); std::iota(idx.begin(), idx.end(), 0);
        std::stable_sort(idx.begin(), idx.end(), [&](int x, int y) { return nrm[x] > nrm[y]; });
        std::vector<double> A2(A), V2(V);
        for (int j = 0; j < n; ++j) {
            std::memcpy(&A[(size_t)m * j], &A2[(size_t)m * idx[j]], sizeof(double) * m);
            std::memcpy(&V[(size_t)n * j], &V2[(size_t)n * idx[j]], sizeof(double) * n);
        }
    }
    std::vector<int> perm(nn);
    std::iota(perm.begin(), perm.end(), 0);
    const double tol = 2.220446049250313e-16 * std::sqrt((double)m);
    const bool par = (size_t)m * n * n > 200000;
    for (int sweep = 0; sweep < 80; ++sweep) {
        int rotated = 0;
        for (int round = 0; round < nn - 1; ++round) {
#pragma omp parallel for reduction(+ : rotated) schedule(static) if (par)
            for (int h = 0; h < nn / 2; ++h) {
                int p = perm[h], q = perm[nn - 1 - h];
                if (p >= n || q >= n) continue;
                if (p > q) std::swap(p, q);
                double *ap = &A[(size_t)m * p], *aq = &A[(size_t)m * q];
                double alpha = 0, beta = 0, gamma = 0;
                for (int i = 0; i < m; ++i) { alpha += ap[i] * ap[i]; beta += aq[i] * aq[i]; gamma += ap[i] * aq[i]; }
                if (std::fabs(gamma) <= tol * std::sqrt(alpha * beta) || gamma == 0.0) continue;
                ++rotated;
                const double zeta = (beta - alpha) / (2.0 * gamma);
                const double t = (zeta >= 0 ? 1.0 : -1.0) / (std::fabs(zeta) + std::sqrt(1.0 + zeta * zeta));
                const double c = 1.0 / std::sqrt(1.0 + t * t), sn = c * t;
                for (int i = 0; i < m; ++i) {
                    const double x = ap[i], y = aq[i];
                    ap[i] = c * x - sn * y;
                    aq[i] = sn * x + c * y;
                }
                double *vp = &V[(size_t)n * p], *vq = &V[(size_t)n * q];
                for (int i = 0; i < n; ++i) {
                    const double x = vp[i], y = vq[i];
                    vp[i] = c * x - sn * y;
                    vq[i] = sn * x + c * y;
                }
            }
            // rotate the round-robin table (position 0 fixed)
            const int last = perm[nn - 1];
            for (int i = nn - 1; i > 1; --i) perm[i] = perm[i - 1];
            perm[1] = last;
        }
        if (rotated == 0) break;
    }
    std::vector<double> nrm(n);
    for (int j = 0; j < n; ++j) {
        double t = 0; for (int i = 0; i < m; ++i) t += A[i + (size_t)m * j] * A[i + (size_t)m * j];
        nrm[j] = std::sqrt(t);
    }
    std::vector<int> idx(n); std::iota(idx.begin(), idx.end(), 0);
    std::stable_sort(idx.begin(), idx.end(), [&](int x, int y) { return nrm[x] > nrm[y]; });
    for (int j = 0; j < n; ++j) {
        const int c = idx[j];
        s[j] = nrm[c];
        const double inv = nrm[c] > 0 ? 1.0 / nrm[c] : 0.0;
        for (int i = 0; i < m; ++i) Y[i + (size_t)m * j] = A[i + (size_t)m * c] * inv;
        std::memcpy(Z + (size_t)n * j, &V[(size_t)n * c], sizeof(double) * n);
    }
}

}  // namespace ssa
