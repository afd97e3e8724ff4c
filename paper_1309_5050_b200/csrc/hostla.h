// Small dense kernels of the solver's host side (orthonormalisation coefficients), vectorised
// for the host CPU: an AVX2/FMA build is selected at run time when the CPU has it.
#pragma once

namespace ssa {
namespace hostla {
// Gp (kc x kc, symmetric) = G[off:off+kc, 0:kc] − C^T C,  C = G[0:na, 0:kc]  (G column-major, ld nn)
void gram_minus_ctc(int kc, int na, int nn, int off, const double *G, double *Gp);
// Mc (n1 x kc, ld n1) = [−C·S; S],  C = G[0:na, 0:kc] (ld n1), S upper triangular (kc x kc)
void proj_coef(int kc, int na, int n1, const double *G, const double *S, double *Mc);
// (G + shift·I) = RᵀR, R upper (column-major, zero below); false when a pivot is not > thr·max diag
bool cholesky_upper(int n, const double *G, double shift, double thr, double *R);
// S = R⁻¹ for R upper triangular (column-major); S upper, zero below
void upper_inverse(int n, const double *R, double *S);
}  // namespace hostla
}  // namespace ssa
