// Host fp64 small dense kernels (dense.cpp).
#pragma once

namespace ssa {
// A = E diag(lam) Eᵀ for symmetric n x n A (column-major); lam descending.
void sym_eig(int n, const double *A, double *lam, double *E);
// M (m x n, m >= n, column-major, leading dim ldm) = Y diag(s) Zᵀ, s descending;
// Y is m x n, Z is n x n (both column-major, packed).
void svd_jacobi(int m, int n, const double *M, int ldm, double *s, double *Y, double *Z);
}  // namespace ssa
