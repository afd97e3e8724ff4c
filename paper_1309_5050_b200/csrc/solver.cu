// Step 2 of the method (SVD) for the implicit trajectory operator:
// block Golub-Kahan-Lanczos bidiagonalisation with full reorthogonalisation and
// thick restarts.  The paper only names
// Lanczos back-ends (nu-TRLan, PROPACK: P:806-823);
// the recurrences below are standard linear algebra:
//
//   X·Q_j   = Pb·C_j + P_{j+1} B_{j+1}      (L side; C_j = full projection onto Pb)
//   Xᵀ·P_j  = (…)    + Q_{j+1} A_{j+1}      (K side, CGS2 against the K basis)
//   X·Qb'   = Pb·T   with T the projected matrix (block bidiagonal, plus an
//                    arrow part after a restart)
//
// Ritz triples come from the fp64 SVD T = Y Θ Zᵀ (one-sided Jacobi on the
// host, never from eigenvalues of TᵀT), U = Pb·Y, σ = Θ, and the residual of
// triple i is ||Xᵀu_i − θ_i v_i|| = ||A_last · y_i(last block)||.  A restart
// keeps the top p Ritz pairs: Pb ← Pb·Y_p, Qb ← [Qb'·Z_p, Q_last], T ← diag(Θ_p)
// (X·(Qb'Z_p) = Pb·Y_p·Θ_p holds exactly).  Bases are orthonormalised with
// SVQB (eigen-decomposition of the column-scaled Gram, Stathopoulos & Wu) run
// twice; numerically dependent directions are replaced by seeded random ones
// (or zeroed once the space is exhausted).  V is recomputed as XᵀU/σ.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "common.h"
#include "dense.h"
#include "hostla.h"
#include "kernels.h"
#include "plan.h"

namespace ssa {

// Host wait for everything queued on `st`: an event polled in a tight loop (the solver waits
// ~60 times per decomposition for small Gram results; a blocking stream synchronisation adds
// the OS wake-up latency to every one of these round trips).
static void stream_wait(cudaStream_t st) {
    static thread_local cudaEvent_t ev = nullptr;
    if (!ev) SSA_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    SSA_CUDA(cudaEventRecord(ev, st));
    cudaError_t e;
    while ((e = cudaEventQuery(ev)) == cudaErrorNotReady) {
    }
    SSA_CUDA(e);
}

// Pinned host staging + matching device ring for the small matrices exchanged
// with the host (Gram results, projection coefficients).  Regions are never
// reused before a stream synchronisation, so uploads need no sync of their own.
struct Staging {
    double *h = nullptr;
    DevBuf d;
    size_t cap = 0, off = 0;
    cudaStream_t st = nullptr;
    void init(size_t n_doubles, cudaStream_t s) {
        // one pinned block per thread, allocated once and kept for the process
        // lifetime (pinned allocation is slow; plans are cheap to create)
        static thread_local double *pinned = nullptr;
        static thread_local size_t pinned_cap = 0;
        if (pinned_cap < n_doubles) {
            if (pinned) cudaFreeHost(pinned);
            SSA_CUDA(cudaMallocHost(&pinned, sizeof(double) * n_doubles));
            pinned_cap = n_doubles;
        }
        st = s;
        cap = n_doubles;
        h = pinned;
        d.alloc(sizeof(double) * cap, st);
    }
    // reserve n doubles; returns the index (host h[idx], device d[idx])
    size_t take(size_t n) {
        n = (n + 31) & ~size_t(31);
        if (off + n > cap) {
            stream_wait(st);
            off = 0;
        }
        SSA_REQUIRE(n <= cap, SSA_ERR_ARG, "staging buffer too small");
        const size_t i = off;
        off += n;
        return i;
    }
    double *dev(size_t i) { return d.as<double>() + i; }
    void sync() {
        stream_wait(st);
        off = 0;
    }
};

void jacobi_svd_blocked(int m, int n, double *T, int *counters, int *sweeps, cudaStream_t st, double tol, double early);
bool jacobi_blocked_fits(int m, int n);
void ritz_tn(int m, int n, const double *T0, const double *A, double *W, double *nrm, cudaStream_t st);

// per-thread grow-only K-side workspace (see Gkl::Qb; freed by ssa_release_workspace or at thread exit)
struct KCache { DevBuf Qb, Qtmp; };
static KCache &kside_cache() { static thread_local KCache c; return c; }
void release_workspace() {
    KCache &c = kside_cache();
    c.Qb.release();
    c.Qtmp.release();
    big_release_all();
}

template <typename T>
struct Gkl {
    PlanImpl &p;
    cudaStream_t st;
    int64_t L, K;
    int k, r, pk, nQmax;
    DevBuf Pb, Ptmp, Jd;
    // The K-side basis and its restart copy (c5: 15 + 9 GB) are grow-only buffers kept per host thread
    // across decompositions: allocated and freed per decomposition, they fragmented the stream-ordered
    // pool with the plans' FFT intermediates, so later decompositions had to map new memory (host
    // stalls of 25-600 ms in the first steps of a process, +10-30 ms on the first timed bench step).
    DevBuf &Qb = kside_cache().Qb, &Qtmp = kside_cache().Qtmp;
    Staging sg;
    int nP = 0, nQ = 0;
    std::vector<double> Tm;   // nQmax x nQmax host, column-major
    int ldT;
    std::vector<double> Alast;
    double anorm = 0.0;
    double ms_ritz = 0.0;
    int last_sweeps = 0;
    float last_kernel_ms = 0.f;
    int64_t nblock = 0, nvec = 0, n_cgs = 0;
    uint64_t sid = 1;
    double thr_abs, thr_rel, thr_chol;
    bool gpu_ritz = true;
    bool debug = std::getenv("SSA_DEBUG") != nullptr;
    double tw_prod = 0, tw_orthA = 0, tw_orthB = 0, tw_rec = 0, tw_restart = 0;   // host wall ms (SSA_DEBUG)
    double tw_o3_gram[2] = {0, 0}, tw_o3_host[2] = {0, 0}, tw_o3_apply[2] = {0, 0};   // orth3 split [L, K side]
    static double now_ms() {
        return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
    }
    int64_t n_fast = 0, n_fallback = 0;
    int64_t o3_exit[2][6] = {{0}};   // SSA_DEBUG: orth3 exits per side [pass], [5] = reprojections
    std::vector<double> res;      // residual bounds of the current Ritz triples
    bool anorm_from_next_gram = false;
    double drop2 = 0.0;           // Σ squared norms of block columns discarded as numerically zero
    int warm_cols = 0;            // start-block columns taken from a previous decomposition
    DevBuf agree_buf;

    // Average `n` host doubles over the ranks of a band partition (identical result on every rank:
    // the collective returns the same bits everywhere), so per-rank timing decisions agree.
    void agree(double *v, int n) {
        agree_buf.alloc(sizeof(double) * 8, st);
        SSA_CUDA(cudaMemcpyAsync(agree_buf.p, v, sizeof(double) * n, cudaMemcpyHostToDevice, st));
        if (p.comm.allreduce_sum(p.comm.user, agree_buf.p, n, SSA_F64, st) != 0)
            throw Error(SSA_ERR_COMM, "allreduce of the convergence-check timings failed");
        SSA_CUDA(cudaMemcpyAsync(v, agree_buf.p, sizeof(double) * n, cudaMemcpyDeviceToHost, st));
        stream_wait(st);
        for (int i = 0; i < n; ++i) v[i] /= p.comm.world;
    }

    explicit Gkl(PlanImpl &pl) : p(pl), st(pl.st), L(pl.L), K(pl.K) {
        // breakdown threshold (relative to ||X||): well below both the convergence tolerance and the
        // fp32 product rounding (~1e-7), so only numerically zero columns are discarded (and their
        // norms enter the residual bound, drop2); decoupled from tol
        thr_abs = (sizeof(T) == 4) ? 1e-8 : 1e-14;
        thr_rel = (sizeof(T) == 4) ? 1e-10 : 1e-26;
        thr_chol = (sizeof(T) == 4) ? 1e-6 : 1e-13;
        sg.init(1 << 18, st);
    }

    // basis leading dimensions: L and K rounded up to 32 elements (16-byte aligned columns for
    // vector / async copies); the padding rows are zero and never written
    int64_t ldP = 0, ldQ = 0;
    int64_t LD(int64_t M) const { return M == K ? ldQ : ldP; }
    T *P(int col) { return Pb.as<T>() + (int64_t)col * ldP; }
    T *Q(int col) { return Qb.as<T>() + (int64_t)col * ldQ; }

    bool kside_comm() const { return p.has_comm && p.comm.world > 1; }

    // G (n1 x n2, host, column-major ld n1) = Aᵀ B; one launch per 512 x 64 chunk, one sync.  Without a
    // cross-rank reduction the Gram's final reduce kernel writes straight into the pinned staging block
    // (host memory mapped into the device address space): no copy-engine transfer on the round trip.
    void gram(int64_t M, const T *A, int64_t lda, int n1, const T *B, int64_t ldb, int n2, double *G, bool kside) {
        struct Chunk { int a0, na, b0, nb; size_t idx; };
        const bool reduce = kside && kside_comm();
        const bool zc = !reduce;
        std::vector<Chunk> ch;
        for (int a0 = 0; a0 < n1; a0 += 512) {
            const int na = std::min(512, n1 - a0);
            for (int b0 = 0; b0 < n2; b0 += 64) {
                const int nb = std::min(64, n2 - b0);
                const size_t idx = sg.take((size_t)na * nb);
                gram_tn<T>(M, A + lda * a0, lda, na, B + ldb * b0, ldb, nb, zc ? sg.h + idx : sg.dev(idx),
                           p.ws_gram.as<double>(), p.ws_gram.bytes, st);
                if (reduce) {
                    if (p.comm.allreduce_sum(p.comm.user, sg.dev(idx), (int64_t)na * nb, SSA_F64, st) != 0)
                        throw Error(SSA_ERR_COMM, "allreduce of a K-side Gram failed");
                }
                if (!zc)
                    SSA_CUDA(cudaMemcpyAsync(sg.h + idx, sg.dev(idx), sizeof(double) * na * nb, cudaMemcpyDeviceToHost, st));
                ch.push_back({a0, na, b0, nb, idx});
            }
        }
        stream_wait(st);
        for (const Chunk &c : ch)
            for (int b = 0; b < c.nb; ++b)
                for (int a = 0; a < c.na; ++a)
                    G[(c.a0 + a) + (int64_t)n1 * (c.b0 + b)] = sg.h[c.idx + a + (size_t)c.na * b];
        sg.off = 0;   // everything staged so far has been consumed
    }

    // Out[:, 0:n] = beta*Out + alpha * A[:, 0:m] * C (C: m x n host, ld ldc); no sync.
    // Not in place: one gemm_acc launch per 512 x 64 chunk; in place (Out == A, m = n <= 64): gemm_small.
    void gemm(int64_t M, const T *A, int64_t lda, int m, const double *C, int ldc, int n, double alpha, double beta,
              T *Out, int64_t ldo) {
        const bool inplace = (Out == A);
        const int mstep = inplace ? 64 : 512;
        for (int c0 = 0; c0 < n; c0 += 64) {
            const int nc = std::min(64, n - c0);
            for (int m0 = 0; m0 < m; m0 += mstep) {
                const int mc = std::min(mstep, m - m0);
                const size_t idx = sg.take((size_t)mc * nc);
                double *h = sg.h + idx;
                for (int b = 0; b < nc; ++b)
                    for (int a = 0; a < mc; ++a) h[a + (size_t)mc * b] = C[(m0 + a) + (int64_t)ldc * (c0 + b)];
                // (a kernel reading the pinned block through its device mapping was slower: c2 7.6 -> 7.7-8.0 ms)
                SSA_CUDA(cudaMemcpyAsync(sg.dev(idx), h, sizeof(double) * mc * nc, cudaMemcpyHostToDevice, st));
                if (inplace)
                    gemm_small<T>(M, A + lda * m0, lda, mc, sg.dev(idx), mc, nc, alpha, (m0 == 0) ? beta : 1.0,
                                  Out + ldo * c0, ldo, st);
                else
                    gemm_acc<T>(M, A + lda * m0, lda, mc, sg.dev(idx), mc, nc, alpha, (m0 == 0) ? beta : 1.0,
                                Out + ldo * c0, ldo, st);
            }
        }
    }

    // W -= Bm * (Bmᵀ W); accumulates the coefficients into coef (nb x kc) if given
    void cgs(int64_t M, T *W, int kc, const T *Bm, int nb, bool kside, double *coef) {
        if (nb <= 0) return;
        std::vector<double> C((size_t)nb * kc);
        gram(M, Bm, LD(M), nb, W, LD(M), kc, C.data(), kside);
        gemm(M, Bm, LD(M), nb, C.data(), nb, kc, -1.0, 1.0, W, LD(M));
        if (coef)
            for (size_t t = 0; t < C.size(); ++t) coef[t] += C[t];
    }

    // Cholesky (G + shift·I) = RᵀR (R upper, column-major); false if a pivot is not
    // positive or tiny relative to the largest diagonal entry.
    bool cholesky(int n, const double *G, double shift, double thr, std::vector<double> &R) {
        R.assign((size_t)n * n, 0.0);
        return hostla::cholesky_upper(n, G, shift, thr, R.data());
    }

    static void upper_inverse(int n, const std::vector<double> &R, std::vector<double> &S) {
        S.assign((size_t)n * n, 0.0);
        hostla::upper_inverse(n, R.data(), S.data());
    }

    // Orthonormalise W (M x kc) against `against` (na orthonormal columns) and internally,
    // by (shifted) CholeskyQR passes (Fukaya, Kannan, Nakatsukasa, Yamamoto, Yanagisawa:
    // shifted CholeskyQR3): a pass whose Gram is too ill-conditioned for Cholesky uses
    // G + s·I (s relative to the largest diagonal), which shrinks the condition number
    // without losing directions; passes repeat until an unshifted pass succeeds after at
    // least one full pass.  Zero columns (exact breakdown) are replaced by seeded random
    // directions; when the space is exhausted they stay zero.  SVQB is the last resort.
    // Returns B (kc x kc, column-major) with W_in ≈ against·(·) + W_out·B.
    std::vector<double> orth(int64_t M, T *W, int kc, const T *against, int na, bool kside,
                             double *coef = nullptr) {
        std::vector<double> B((size_t)kc * kc, 0.0);
        for (int i = 0; i < kc; ++i) B[i + (size_t)kc * i] = 1.0;
        std::vector<double> G((size_t)kc * kc), Gh((size_t)kc * kc), E((size_t)kc * kc), lam(kc);
        std::vector<double> S((size_t)kc * kc), Bp((size_t)kc * kc), Bn((size_t)kc * kc), R;
        const double shift_rel = (sizeof(T) == 4) ? 1e-6 : 1e-13;
        // ---- projection against the basis: one CGS pass, a second only when DGKS asks
        // (||w_after||² < ½||w_before||², with ||w_before||² = ||c||² + ||w_after||²)
        auto project = [&](bool force_twice) {
            std::vector<double> C((size_t)na * kc);
            gram(M, against, LD(M), na, W, LD(M), kc, C.data(), kside);
            gemm(M, against, LD(M), na, C.data(), na, kc, -1.0, 1.0, W, LD(M));
            if (coef)
                for (size_t t = 0; t < C.size(); ++t) coef[t] += C[t];
            gram(M, W, LD(M), kc, W, LD(M), kc, G.data(), kside);
            bool need = force_twice;
            for (int j = 0; j < kc && !need; ++j) {
                double c2 = 0.0;
                for (int a2 = 0; a2 < na; ++a2) c2 += C[a2 + (size_t)na * j] * C[a2 + (size_t)na * j];
                need = c2 > G[j + (size_t)kc * j];
            }
            if (need) {
                gram(M, against, LD(M), na, W, LD(M), kc, C.data(), kside);
                gemm(M, against, LD(M), na, C.data(), na, kc, -1.0, 1.0, W, LD(M));
                if (coef)
                    for (size_t t = 0; t < C.size(); ++t) coef[t] += C[t];
                gram(M, W, LD(M), kc, W, LD(M), kc, G.data(), kside);
            }
            n_cgs += need ? 2 : 1;
        };
        bool have_gram = false;
        if (na > 0) { project(false); have_gram = true; }
        int refills = 0;
        for (int pass = 0; pass < 6; ++pass) {
            if (!have_gram) gram(M, W, LD(M), kc, W, LD(M), kc, G.data(), kside);
            if (anorm_from_next_gram) {
                anorm_from_next_gram = false;
                for (int j = 0; j < kc; ++j) anorm = std::max(anorm, std::sqrt(std::max(G[j + (size_t)kc * j], 0.0)));
            }
            have_gram = false;
            // exact breakdown: columns with (numerically) zero norm
            std::vector<int> zero;
            double dmax = 0.0;
            for (int j = 0; j < kc; ++j) dmax = std::max(dmax, G[j + (size_t)kc * j]);
            for (int j = 0; j < kc; ++j) {
                // the absolute test (relative to ||X||) only makes sense on the raw input;
                // after a pass the columns are normalised and only the relative test applies
                const double d = std::sqrt(std::max(G[j + (size_t)kc * j], 0.0));
                const bool tiny_abs = (pass == 0 && refills == 0) && !(d > thr_abs * std::max(anorm, 1e-300));
                if (tiny_abs || !(d * d > 1e-24 * dmax) || !(dmax > 0.0)) zero.push_back(j);
            }
            for (int j : zero) drop2 += std::max(G[j + (size_t)kc * j], 0.0);
            if (!zero.empty() && refills < 2) {
                ++refills;
                for (int j : zero)
                    for (int i = 0; i < kc; ++i) B[j + (size_t)kc * i] = 0.0;   // W_in has no component there
                // one launch per run of consecutive zero columns (c5: ~130 refilled columns per decomposition)
                for (size_t a = 0; a < zero.size();) {
                    size_t b = a + 1;
                    while (b < zero.size() && zero[b] == zero[b - 1] + 1) ++b;
                    fill_normal<T>(M, W + LD(M) * zero[a], LD(M), (int)(b - a), p.seed, 0x5eed0000ull + (sid++), st);
                    a = b;
                }
                if (na > 0) {
                    double *keep = coef;
                    coef = nullptr;            // the random directions are not part of W_in
                    project(true);
                    coef = keep;
                    have_gram = true;
                }
                --pass;   // redo the pass with the refreshed columns (bounded by `refills`)
                continue;
            }
            bool shifted = false, ok = cholesky(kc, G.data(), 0.0, thr_chol, R);
            if (!ok) {
                ok = cholesky(kc, G.data(), shift_rel * dmax, 1e-300, R);
                shifted = ok;
            }
            std::vector<int> bad;
            if (ok) {
                upper_inverse(kc, R, S);
                Bp = R;
            } else {   // SVQB: eigen-decomposition of the column-scaled Gram
                std::vector<double> d(kc);
                for (int j = 0; j < kc; ++j) d[j] = std::sqrt(std::max(G[j + (size_t)kc * j], 0.0));
                for (int b2 = 0; b2 < kc; ++b2)
                    for (int a2 = 0; a2 < kc; ++a2)
                        Gh[a2 + (size_t)kc * b2] = (d[a2] > 0 && d[b2] > 0) ? G[a2 + (size_t)kc * b2] / (d[a2] * d[b2]) : 0.0;
                sym_eig(kc, Gh.data(), lam.data(), E.data());
                for (int j = 0; j < kc; ++j) {
                    const bool good = lam[j] > thr_rel;
                    const double isq = good ? 1.0 / std::sqrt(lam[j]) : 0.0;
                    const double sq = good ? std::sqrt(lam[j]) : 0.0;
                    for (int a2 = 0; a2 < kc; ++a2) {
                        S[a2 + (size_t)kc * j] = (d[a2] > 0 ? 1.0 / d[a2] : 0.0) * E[a2 + (size_t)kc * j] * isq;
                        Bp[j + (size_t)kc * a2] = sq * E[a2 + (size_t)kc * j] * d[a2];
                    }
                    if (!good) bad.push_back(j);
                }
            }
            if (debug)
                std::fprintf(stderr, "[ssa] orth M=%lld pass=%d na=%d zero=%zu chol=%d shifted=%d bad=%zu anorm=%.3e\n",
                             (long long)M, pass, na, zero.size(), (int)ok, (int)shifted, bad.size(), anorm);
            gemm(M, W, LD(M), kc, S.data(), kc, kc, 1.0, 0.0, W, LD(M));   // in place (kc <= 64)
            for (int b2 = 0; b2 < kc; ++b2)
                for (int a2 = 0; a2 < kc; ++a2) {
                    double s2 = 0.0;
                    for (int t = 0; t < kc; ++t) s2 += Bp[a2 + (size_t)kc * t] * B[t + (size_t)kc * b2];
                    Bn[a2 + (size_t)kc * b2] = s2;
                }
            B.swap(Bn);
            if (ok && !shifted && pass >= 1 && bad.empty()) break;
        }
        return B;
    }


    // Projection + CholeskyQR2 with two host round trips (the default).  W (M x kc) follows the
    // na orthonormal columns `against` in the same buffer:
    //   1. one Gram [A W]ᵀW gives C = AᵀW and WᵀW; the projected Gram is Gp = WᵀW − CᵀC
    //      (= W'ᵀW' for W' = W − A C); its Cholesky factor R gives the fused update
    //      W ← [A W]·[−C R⁻¹; R⁻¹] (one streaming pass, tile-level in place);
    //   2. CholeskyQR on W alone (Gram WᵀW, W ← W R₂⁻¹), repeated once more only if a pass was
    //      shifted or far from orthonormal.
    // DGKS (P:… standard CGS safeguard): if projection removed more than half of a column's
    // norm (Gp_jj < ½ (WᵀW)_jj), or a column is numerically zero, or Cholesky fails, W is left
    // untouched and the robust `orth` (second projection, shifts, refills, SVQB) takes over.
    // Returns B with W_in = A·coef + W_out·B (coef accumulated, as in `orth`).
    // G1 (optional): the pass-1 Gram [A W]ᵀW, already computed (a deferred orthonormalisation, below)
    std::vector<double> orth3(int64_t M, T *W, int kc, const T *against, int na, bool kside, double *coef,
                              const std::vector<double> *G1 = nullptr) {
        const int64_t ld = LD(M);
        if (kc > 64 || na <= 0 || na + kc > 512 || against + (int64_t)na * ld != W)
            return orth(M, W, kc, against, na, kside, coef);
        T *A = const_cast<T *>(against);
        const int n1 = na + kc;
        std::vector<double> G((size_t)n1 * kc), Gp((size_t)kc * kc), R, Sinv, Mc((size_t)n1 * kc);
        std::vector<double> Ctot((size_t)na * kc, 0.0), Btot, Bn((size_t)kc * kc);
        const double shift_rel = (sizeof(T) == 4) ? 1e-6 : 1e-13;
        bool project = true, reproject = false;
        for (int pass = 1; pass <= 4; ++pass) {
            bool shifted = false;
            double dev = 0.0;
            {
                const int nn = project ? n1 : kc;                       // Gram columns: [A W] or W
                T *Ab = project ? A : W;
                const double tg0 = now_ms();
                if (pass == 1 && G1 && project) G = *G1;
                else gram(M, Ab, ld, nn, W, ld, kc, G.data(), kside);
                const double tg1 = now_ms();
                tw_o3_gram[kside] += tg1 - tg0;
                const int off = project ? na : 0;
                // (the na-long host loops run vectorised in hostla.cpp: as scalar dependent-FMA chains
                // they were a large part of a small-M block step)
                if (project) {
                    hostla::gram_minus_ctc(kc, na, nn, off, G.data(), Gp.data());
                } else {
                    for (int bb = 0; bb < kc; ++bb)
                        for (int aa = 0; aa < kc; ++aa) Gp[aa + (size_t)kc * bb] = G[off + std::min(aa, bb) + (size_t)nn * std::max(aa, bb)];
                }
                double dmax = 0.0;
                dev = 0.0;
                for (int j = 0; j < kc; ++j) dmax = std::max(dmax, Gp[j + (size_t)kc * j]);
                for (int bb = 0; bb < kc; ++bb)
                    for (int aa = 0; aa < kc; ++aa)
                        dev = std::max(dev, std::fabs(Gp[aa + (size_t)kc * bb] - (aa == bb ? 1.0 : 0.0)));
                if (pass == 1) {
                    // breakdown (numerically zero column) -> robust path, W untouched
                    bool zero = !(dmax > 0.0) || !std::isfinite(dmax);
                    for (int j = 0; j < kc && !zero; ++j) {
                        const double d = Gp[j + (size_t)kc * j], h = G[na + j + (size_t)n1 * j];
                        zero = !(std::sqrt(std::max(d, 0.0)) > thr_abs * std::max(anorm, 1e-300)) || !(d > 1e-24 * dmax) ||
                               !(d > (sizeof(T) == 4 ? 1e-12 : 1e-24) * h);
                        reproject = reproject || !(d > 0.5 * h);   // DGKS: "twice is enough"
                    }
                    if (zero) { ++n_fallback; return orth(M, W, kc, against, na, kside, coef); }
                }
                shifted = false;
                bool ok = cholesky(kc, Gp.data(), 0.0, thr_chol, R);
                if (!ok) { ok = cholesky(kc, Gp.data(), shift_rel * dmax, 1e-300, R); shifted = ok; }
                if (!ok) {
                    if (pass == 1) { ++n_fallback; return orth(M, W, kc, against, na, kside, coef); }
                    break;
                }
                upper_inverse(kc, R, Sinv);
                double ta0 = 0.0;
                if (project) {
                    // W ← [A W]·[−C R⁻¹; R⁻¹]; coefficients W_in = A·(Ctot + C·Btot) + W_new·(R·Btot)
                    hostla::proj_coef(kc, na, n1, G.data(), Sinv.data(), Mc.data());
                    ta0 = now_ms();
                    tw_o3_host[kside] += ta0 - tg1;
                    gemm(M, A, ld, n1, Mc.data(), n1, kc, 1.0, 0.0, W, ld);
                    tw_o3_apply[kside] += now_ms() - ta0;
                    std::vector<double> cv((size_t)std::max(na, 1));
                    for (int bb = 0; bb < kc; ++bb) {
                        double *ct = Ctot.data() + (size_t)na * bb;
                        if (Btot.empty()) {
                            const double *gb = G.data() + (size_t)n1 * bb;
                            for (int t = 0; t < na; ++t) ct[t] += gb[t];
                            continue;
                        }
                        for (int t = 0; t < na; ++t) cv[t] = 0.0;
                        for (int aa = 0; aa < kc; ++aa) {
                            const double bv = Btot[aa + (size_t)kc * bb], *ga = G.data() + (size_t)n1 * aa;
    #pragma omp simd
                            for (int t = 0; t < na; ++t) cv[t] += ga[t] * bv;
                        }
                        for (int t = 0; t < na; ++t) ct[t] += cv[t];
                    }
                } else {
                    ta0 = now_ms();
                    tw_o3_host[kside] += ta0 - tg1;
                    gemm(M, W, ld, kc, Sinv.data(), kc, kc, 1.0, 0.0, W, ld);   // in place
                    tw_o3_apply[kside] += now_ms() - ta0;
                }
            }
            if (Btot.empty()) Btot = R;
            else {
                // Bn = R·Btot (R upper): per output the same t order as the dot-product form
                for (int bb = 0; bb < kc; ++bb) {
                    double *bn = Bn.data() + (size_t)kc * bb;
                    for (int aa = 0; aa < kc; ++aa) bn[aa] = 0.0;
                    for (int t = 0; t < kc; ++t) {
                        const double bt = Btot[t + (size_t)kc * bb], *rt = R.data() + (size_t)kc * t;
                        for (int aa = 0; aa <= t; ++aa) bn[aa] += rt[aa] * bt;
                    }
                }
                Btot.swap(Bn);
            }
            const bool was_projection = project;
            project = (pass == 1 && reproject);
            if (project) ++o3_exit[kside][5];
            if (pass >= 2 && !project && !shifted && !was_projection && dev <= 0.1) {
                ++o3_exit[kside][pass];
                if (coef)
                    for (size_t t = 0; t < Ctot.size(); ++t) coef[t] += Ctot[t];
                ++n_fast;
                return Btot;
            }
            if (pass >= 2 && !project && !shifted && was_projection && dev <= 1e-3) {
                // the second projection pass already left W orthonormal
                ++o3_exit[kside][pass];
                if (coef)
                    for (size_t t = 0; t < Ctot.size(); ++t) coef[t] += Ctot[t];
                ++n_fast;
                return Btot;
            }
        }
        // not orthonormal after the passes: the robust path finishes from the current W
        ++n_fallback;
        std::vector<double> C2((size_t)na * kc, 0.0);
        std::vector<double> B2 = orth(M, W, kc, against, na, kside, C2.data());
        if (coef)
            for (int bb = 0; bb < kc; ++bb)
                for (int t = 0; t < na; ++t) {
                    double v = Ctot[t + (size_t)na * bb];
                    for (int aa = 0; aa < kc; ++aa) v += C2[t + (size_t)na * aa] * Btot[aa + (size_t)kc * bb];
                    coef[t + (size_t)na * bb] += v;
                }
        for (int bb = 0; bb < kc; ++bb)
            for (int aa = 0; aa < kc; ++aa) {
                double v = 0.0;
                for (int t = 0; t < kc; ++t) v += B2[aa + (size_t)kc * t] * Btot[t + (size_t)kc * bb];
                Bn[aa + (size_t)kc * bb] = v;
            }
        return Bn;
    }

    // every block product is bracketed by CUDA events on the plan's stream so the
    // device time spent in the trajectory products is reported (ms_products)
    std::vector<cudaEvent_t> ev;
    std::vector<char> ev_xv;   // per event pair: 1 = X·V, 0 = Xᵀ·U
    int64_t n_xv = 0, n_xtu = 0, vec_xv = 0, vec_xtu = 0;
    void mark() {
        cudaEvent_t e;
        SSA_CUDA(cudaEventCreate(&e));
        SSA_CUDA(cudaEventRecord(e, st));
        ev.push_back(e);
    }
    // device milliseconds of the X·V (which = 1) / Xᵀ·U (0) / all (-1) block products
    double product_ms(int which = -1) {
        double ms = 0.0;
        if (!ev.empty()) SSA_CUDA(cudaEventSynchronize(ev.back()));
        for (size_t i = 0; i + 1 < ev.size(); i += 2) {
            if (which >= 0 && ev_xv[i / 2] != which) continue;
            float t = 0.f;
            SSA_CUDA(cudaEventElapsedTime(&t, ev[i], ev[i + 1]));
            ms += t;
        }
        return ms;
    }
    ~Gkl() {
        for (auto e : ev) cudaEventDestroy(e);
    }
    void product_xv(const T *Qin, T *Out, int kc) {
        mark();
        op_xv<T>(p, Qin, ldQ, Out, ldP, kc);
        mark();
        ev_xv.push_back(1);
        ++nblock; nvec += kc; ++n_xv; vec_xv += kc;
    }
    void product_xtu(const T *Pin, T *Out, int kc) {
        mark();
        op_xtu<T>(p, Pin, ldP, Out, ldQ, kc);
        mark();
        ev_xv.push_back(0);
        ++nblock; nvec += kc; ++n_xtu; vec_xtu += kc;
    }

    double &Tat(int i, int j) { return Tm[(size_t)i + (size_t)ldT * j]; }

    void stepA() {
        const int qc = nQ - k;
        T *W = P(nP);
        double t0 = now_ms();
        product_xv(Q(qc), W, k);
        tw_prod += now_ms() - t0;
        t0 = now_ms();
        if (anorm == 0.0) {
            std::vector<double> G((size_t)k * k);
            gram(L, W, ldP, k, W, ldP, k, G.data(), false);
            for (int j = 0; j < k; ++j) anorm = std::max(anorm, std::sqrt(std::max(G[j + (size_t)k * j], 0.0)));
        }
        // full projection onto the L basis; all CGS coefficients go into T so that
        // X·Qb = Pb·T holds exactly
        std::vector<double> C((size_t)nP * k, 0.0);
        std::vector<double> B;
        B = orth3(L, W, k, P(0), nP, false, C.data());
        tw_orthA += now_ms() - t0;
        for (int b = 0; b < k; ++b)
            for (int a = 0; a < nP; ++a) Tat(a, qc + b) = C[a + (size_t)nP * b];
        for (int b = 0; b < k; ++b)
            for (int a = 0; a < k; ++a) Tat(nP + a, qc + b) = B[a + (size_t)k * b];
        nP += k;
    }

    // Lanczos recurrence term of a new K block W = Xᵀ·P(pc): W −= Q_prev·Bᵀ with B = T[P_new, Q_prev]
    // (known exactly), removed before the full projection so that the projection only removes
    // rounding-level components and one CGS pass normally suffices
    void remove_recurrence(T *W, int pc) {
        const int qc = nQ - k;
        std::vector<double> Bt((size_t)k * k);
        for (int a = 0; a < k; ++a)
            for (int b = 0; b < k; ++b) Bt[b + (size_t)k * a] = Tat(pc + a, qc + b);   // (T block)ᵀ
        gemm(K, Q(qc), ldQ, k, Bt.data(), k, k, -1.0, 1.0, W, ldQ);
    }

    void stepB() {
        const int pc = nP - k;
        T *W = Q(nQ);
        double t0 = now_ms();
        product_xtu(P(pc), W, k);
        tw_prod += now_ms() - t0;
        // ||X|| estimate = the largest column norm of the first Xᵀ·U block, taken from the first Gram of
        // its orthonormalisation (na = 0: orth's pass-0 WᵀW) instead of a Gram of its own (a 3.8 GB
        // stream on c5)
        anorm_from_next_gram = anorm == 0.0;
        auto recurrence = [&]() { if (nQ > 0) remove_recurrence(W, pc); };
        t0 = now_ms();
        // full reorthogonalisation of the K side as well (CGS2 against the whole K basis): the
        // one-sided variant needed several times more products with thick restarts.
        // The recurrence term is removed first by its own streaming update: folding it into the
        // projection's Gram (WᵀW − CᵀC with the large recurrence part inside C) cancels catastrophically
        // — squared norms, ε·||b||²/||w'||² — and broke convergence on c1-c3 (measured), whereas the
        // vector subtraction loses only ε·||b||/||w'||
        const T *againstK = Q(0);
        const int naK = nQ;
        recurrence();
        tw_rec += now_ms() - t0;
        t0 = now_ms();
        Alast = orth3(K, W, k, againstK, naK, true, nullptr);

        tw_orthB += now_ms() - t0;
        nQ += k;
    }

    // Deferred K-side orthonormalisation.  When a Ritz check follows a block pair, the
    // new K block only matters through A_last (the residual bound) unless the iteration continues:
    // stepB_check stops after the recurrence and the pass-1 Gram [Q W]ᵀW and takes A_last ≈ R₁,
    // the Cholesky factor of the projected Gram (the second CholeskyQR pass changes it by the
    // pass-1 output's deviation from orthonormality).  A check that converges with margin skips
    // the block's remaining passes (c5: 3 of its 5 K-side streams); otherwise stepB_finish runs
    // orth3 from the stored Gram and the residuals are recomputed with the exact A_last.
    std::vector<double> G1def;
    bool deferred = false;
    void stepB_check() {
        const int pc = nP - k, na = nQ, n1 = nQ + k;
        if (na <= 0 || k > 64 || n1 > 512) { stepB(); return; }
        T *W = Q(nQ);
        double t0 = now_ms();
        product_xtu(P(pc), W, k);
        tw_prod += now_ms() - t0;
        t0 = now_ms();
        remove_recurrence(W, pc);
        G1def.assign((size_t)n1 * k, 0.0);
        gram(K, Q(0), ldQ, n1, W, ldQ, k, G1def.data(), true);
        // orth3's pass-1 tests; any of them (breakdown, DGKS reprojection, failed or shifted
        // Cholesky) -> the full orthonormalisation now, from the same Gram
        std::vector<double> Gp((size_t)k * k), R;
        hostla::gram_minus_ctc(k, na, n1, na, G1def.data(), Gp.data());
        double dmax = 0.0;
        for (int j = 0; j < k; ++j) dmax = std::max(dmax, Gp[j + (size_t)k * j]);
        bool fine = dmax > 0.0 && std::isfinite(dmax);
        for (int j = 0; j < k && fine; ++j) {
            const double d = Gp[j + (size_t)k * j], h = G1def[na + j + (size_t)n1 * j];
            fine = std::sqrt(std::max(d, 0.0)) > thr_abs * std::max(anorm, 1e-300) && d > 1e-24 * dmax &&
                   d > (sizeof(T) == 4 ? 1e-12 : 1e-24) * h && d > 0.5 * h;
        }
        fine = fine && cholesky(k, Gp.data(), 0.0, thr_chol, R);
        if (fine) {
            Alast = R;
            deferred = true;
        } else {
            Alast = orth3(K, W, k, Q(0), na, true, nullptr, &G1def);
        }
        tw_orthB += now_ms() - t0;
        nQ += k;
    }
    void stepB_finish() {
        if (!deferred) return;
        deferred = false;
        const double t0 = now_ms();
        Alast = orth3(K, Q(nQ - k), k, Q(0), nQ - k, true, nullptr, &G1def);
        tw_orthB += now_ms() - t0;
    }

    // SVD of T[0:m, 0:n] (m >= n): th (n), Y (m x n), Z (n x n), descending.
    void ritz_svd(int m, int n, std::vector<double> &th, std::vector<double> &Y, std::vector<double> &Z) {
        const auto t0 = std::chrono::steady_clock::now();
        th.assign(n, 0.0); Y.assign((size_t)m * n, 0.0); Z.assign((size_t)n * n, 0.0);
        bool done = false;
        if (gpu_ritz && jacobi_blocked_fits(m, n)) {
            // device layout: A (m x n, rotated in place) | T0 (copy of T) | W (n x n) | nrm (n) | ints
            const size_t mn = (size_t)m * n;
            Jd.alloc(sizeof(double) * (2 * mn + (size_t)n * n + n + 80), st);
            double *Ad = Jd.as<double>(), *T0d = Ad + mn, *Wd = T0d + mn, *nrmd = Wd + (size_t)n * n;
            int *dints = reinterpret_cast<int *>(nrmd + n + 8);
            // upload and read-back through grow-only pinned blocks kept per thread (the staging ring
            // is too small for the largest projected matrices; pageable buffers cost page faults and
            // bounce copies on every Ritz step)
            static thread_local double *upin = nullptr;
            static thread_local size_t ucap = 0;
            if (ucap < mn) {
                if (upin) { stream_wait(st); SSA_CUDA(cudaFreeHost(upin)); }
                ucap = std::max(mn, 2 * ucap);
                SSA_CUDA(cudaMallocHost(&upin, sizeof(double) * ucap));
            }
            stream_wait(st);   // the previous upload from upin has completed
            for (int j = 0; j < n; ++j)
                std::memcpy(upin + (size_t)m * j, &Tm[(size_t)ldT * j], sizeof(double) * m);
            SSA_CUDA(cudaMemcpyAsync(Ad, upin, sizeof(double) * mn, cudaMemcpyHostToDevice, st));
            SSA_CUDA(cudaMemcpyAsync(T0d, Ad, sizeof(double) * mn, cudaMemcpyDeviceToDevice, st));
            // off-diagonal tolerance: fp32 products resolve ~1e-7 relative, so 1e-9 (fp32) / 1e-12
            // (fp64) leaves the Ritz values exact to rounding and saves the last Jacobi sweep(s)
            const double tolj = sizeof(T) == 4 ? 1e-9 : 1e-12;
            int *dsw = dints + 64;
            cudaEvent_t je0 = nullptr, je1 = nullptr;
            if (debug) {
                SSA_CUDA(cudaEventCreate(&je0)); SSA_CUDA(cudaEventCreate(&je1));
                SSA_CUDA(cudaEventRecord(je0, st));
            }
            // early stop once a sweep's largest rotated relative off-diagonal is below 1e-4 (fp32) /
            // 1e-6 (fp64): the columns then end orthogonal to ~1e-8 / 1e-12 (quadratic convergence)
            const double early = sizeof(T) == 4 ? 1e-4 : 1e-6;
            jacobi_svd_blocked(m, n, Ad, dints, debug ? dsw : nullptr, st, tolj, early);
            if (debug) {
                SSA_CUDA(cudaEventRecord(je1, st));
                SSA_CUDA(cudaMemcpyAsync(&last_sweeps, dsw, sizeof(int), cudaMemcpyDeviceToHost, st));
            }
            ritz_tn(m, n, T0d, Ad, Wd, nrmd, st);
            // A | T0 | W | nrm: fetch A, then W and nrm (contiguous)
            // read-back into a grow-only pinned block kept per thread (pageable / freshly allocated
            // host buffers cost page faults and bounce-buffer copies on every Ritz step)
            static thread_local double *rpin = nullptr;
            static thread_local size_t rcap = 0;
            const size_t need_d = mn + (size_t)n * n + n;
            if (rcap < need_d) {
                if (rpin) SSA_CUDA(cudaFreeHost(rpin));
                rcap = std::max(need_d, 2 * rcap);
                SSA_CUDA(cudaMallocHost(&rpin, sizeof(double) * rcap));
            }
            double *const A = rpin, *const Wn = rpin + mn;
            SSA_CUDA(cudaMemcpyAsync(A, Ad, sizeof(double) * mn, cudaMemcpyDeviceToHost, st));
            SSA_CUDA(cudaMemcpyAsync(Wn, Wd, sizeof(double) * ((size_t)n * n + n), cudaMemcpyDeviceToHost, st));
            sg.sync();
            if (debug) {
                float jms = 0.f;
                SSA_CUDA(cudaEventElapsedTime(&jms, je0, je1));
                last_kernel_ms = jms;
                cudaEventDestroy(je0); cudaEventDestroy(je1);
            }
            const double *nrm = Wn + (size_t)n * n;
            std::vector<int> idx(n);
            for (int j = 0; j < n; ++j) idx[j] = j;
            std::stable_sort(idx.begin(), idx.end(), [&](int a, int b) { return nrm[a] > nrm[b]; });
            for (int j = 0; j < n; ++j) {
                const int c = idx[j];
                th[j] = nrm[c];
                const double inv = nrm[c] > 0 ? 1.0 / nrm[c] : 0.0;
                for (int i = 0; i < m; ++i) Y[i + (size_t)m * j] = A[i + (size_t)m * c] * inv;
            }
            // right vectors of the kept triples: z_j = Tᵀ y_j / θ_j = W[:, c] / θ_j² (needs θ_j well above 0)
            const int need = std::min(n, std::max(pk, r));
            const double floor_rel = (sizeof(T) == 4) ? 1e-9 : 1e-13;
            if (th[need - 1] > floor_rel * th[0]) {
                for (int j = 0; j < need; ++j) {
                    const double inv2 = 1.0 / (th[j] * th[j]);
                    const double *wc = Wn + (size_t)n * idx[j];
                    for (int c = 0; c < n; ++c) Z[c + (size_t)n * j] = wc[c] * inv2;
                }
                done = true;
            }
        }
        if (!done) svd_jacobi(m, n, Tm.data(), ldT, th.data(), Y.data(), Z.data());
        const double dt = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
        ms_ritz += dt;
        if (debug) std::fprintf(stderr, "[ssa] ritz_svd %dx%d %s %.3f ms (kernel %.3f ms, %d sweeps)\n", m, n, done ? "device" : "host", dt,
                                last_kernel_ms, last_sweeps);
    }

    void run(int r_, ssa_decomp_info *info) {
        r = r_;
        const int64_t mn = std::min(L, K);
        k = std::max(1, std::min<int>(p.block_k, 64));
        if (k > mn) k = (int)mn;
        int extra = std::max(k / 2, r);        // keep ~2r Ritz pairs (parameter sweep)
        if (const char *e = std::getenv("SSA_PK_EXTRA")) extra = std::atoi(e);
        pk = (int)std::min<int64_t>(r + extra, mn);
        // blocks per restart cycle (measured sweep over k and the cycle length on c1-c4, DESIGN.md §5:
        // the projected SVD grows as n³, fewer cycles cost more products); the projected SVD runs
        // on the device for n up to ~2000
        // cycle length: the warm-decomposition sweep (scripts/sweep_warm.py) has
        // c2-sized operators (L·K ~ 2.5e7) fastest at 4 blocks per cycle and c3-sized ones
        // (L·K ~ 8e8, products and K-side Grams dominate) at 6
        int mcyc = ((double)L * (double)K >= 1e8) ? 6 : 4;
        if (const char *e = std::getenv("SSA_MCYC")) mcyc = std::max(1, std::atoi(e));
        while (mcyc > 2 && !jacobi_blocked_fits(pk + (mcyc + 1) * k, pk + mcyc * k)) --mcyc;
        nQmax = pk + k * (mcyc + 1);
        ldT = nQmax;
        Tm.assign((size_t)ldT * ldT, 0.0);
        ldP = (L + 31) / 32 * 32;
        ldQ = (K + 31) / 32 * 32;
        Pb.alloc(sizeof(T) * ldP * nQmax, st);
        Qb.alloc(sizeof(T) * ldQ * nQmax, st);
        Ptmp.alloc(sizeof(T) * ldP * pk, st);
        Qtmp.alloc(sizeof(T) * ldQ * pk, st);
        // zero only the padding rows (L..ldP-1, K..ldQ-1) of every column
        auto zero_pad = [&](void *base, int64_t rows, int64_t ld, int64_t cols) {
            if (ld > rows)
                SSA_CUDA(cudaMemset2DAsync(static_cast<T *>(base) + rows, sizeof(T) * ld, 0, sizeof(T) * (ld - rows),
                                           (size_t)cols, st));
        };
        zero_pad(Pb.p, L, ldP, nQmax);
        zero_pad(Qb.p, K, ldQ, nQmax);
        zero_pad(Ptmp.p, L, ldP, pk);
        zero_pad(Qtmp.p, K, ldQ, pk);
        const double tol = p.tol > 0 ? p.tol : (sizeof(T) == 4 ? 1e-6 : 1e-10);
        const int64_t maxprod = p.max_products > 0 ? p.max_products : std::max<int64_t>(400, 40 * (nQmax / k));

        // P_1: a seeded Gaussian block, or — when the plan already holds a decomposition — a warm
        // start from its eigenvectors (the paper's "decomposition will be automatically continued",
        // P:869-873): the stored U_1..U_min(r_prev,k) lead the start block, random columns fill it
        fill_normal<T>(L, P(0), ldP, k, p.seed, 0, st);
        if (p.r > 0 && p.U.p) {
            const int nw = std::min(p.r, k);
            SSA_CUDA(cudaMemcpy2DAsync(P(0), sizeof(T) * ldP, p.U.p, sizeof(T) * L, sizeof(T) * L, nw,
                                       cudaMemcpyDeviceToDevice, st));
            warm_cols = nw;
        }
        orth(L, P(0), k, nullptr, 0, false);
        nP = k;
        stepB();
        std::vector<double> th, Y, Z;
        int nconv = 0, restarts = 0;
        double t_block = 0.0, t_ritz = 0.0;   // host wall ms of the last block pair / Ritz step
        double maxres = 0.0;
        static const bool defer_on = [] { const char *e = std::getenv("SSA_DEFER"); return e ? std::atoi(e) != 0 : true; }();
        for (;;) {
            const double tb0 = now_ms();
            stepA();
            // Will a Ritz check follow this pair?  (decided before stepB, so that its
            // orthonormalisation can be deferred past the check)  The cycle ends when the basis is
            // full or the product budget is spent.  When a block step costs at least as much as a
            // Ritz step (c4, c5: large operators, few blocks to convergence), check after every block
            // once the basis holds r vectors (cost of the previous pair); cheap blocks (c2, c3) wait
            // for the cycle end.  With a band partition every rank must take the same decision (each
            // check is followed by collectives or by none): the timings are averaged over the ranks
            // first.
            const bool cycle_end = !(nQ + 2 * k <= nQmax && nblock + 1 < maxprod);
            double tt[2] = {t_block, t_ritz > 0.0 ? t_ritz : 1.0};
            if (kside_comm()) agree(tt, 2);
            const bool costly_blocks = nQ >= r && tt[0] >= tt[1];
            const bool check = cycle_end || costly_blocks;
            if (check && defer_on) stepB_check();
            else stepB();
            t_block = now_ms() - tb0;
            if (!check) continue;
            // ---- Ritz extraction from T (nP x nc)
            const int nc = nQ - k;
            const double tr = ms_ritz;
            ritz_svd(nP, nc, th, Y, Z);
            t_ritz = ms_ritz - tr;
            anorm = std::max(anorm, th[0]);
            // residual bound of triple i: ||Xᵀu_i − θ_i v_i|| <= ||A_last·y_i(last block)||
            // + sqrt(drop2), drop2 = the squared norms of every block column that orthonormalisation
            // discarded as numerically zero (a refilled column has no A / B entry, so without this
            // term its part of the residual would be invisible)
            auto residuals = [&]() {
                res.assign(nc, 0.0);
                std::vector<double> sv((size_t)k);
                const double dropn = std::sqrt(drop2);
                for (int i = 0; i < nc; ++i) {
                    // s = Alast · y_i(last block): k independent accumulators, each in the original b order
                    for (int a = 0; a < k; ++a) sv[a] = 0.0;
                    for (int b = 0; b < k; ++b) {
                        const double y = Y[(nP - k + b) + (size_t)nP * i], *al = Alast.data() + (size_t)k * b;
                        for (int a = 0; a < k; ++a) sv[a] += al[a] * y;
                    }
                    double s2 = 0.0;
                    for (int a = 0; a < k; ++a) s2 += sv[a] * sv[a];
                    res[i] = std::sqrt(s2) + dropn;
                }
            };
            residuals();
            if (deferred) {
                // the estimated A_last decides only with a factor-2 margin on every wanted triple
                bool sure = nc >= r;
                for (int i = 0; i < std::min(r, nc) && sure; ++i) sure = res[i] <= 0.5 * tol * th[0];
                if (!sure) {
                    stepB_finish();
                    residuals();
                }
            }
            nconv = 0; maxres = 0.0;
            for (int i = 0; i < std::min(r, nc); ++i) {
                maxres = std::max(maxres, res[i] / th[0]);
                if (res[i] <= tol * th[0]) ++nconv;
            }
            if (debug) {
                double an = 0, bn = 0;
                for (double v : Alast) an += v * v;
                for (int b = 0; b < nc; ++b)
                    for (int a = nP - k; a < nP; ++a) bn += Tat(a, b) * Tat(a, b);
                std::fprintf(stderr, "[ssa] ritz nP=%d nc=%d prod=%lld th0=%.6e th[r-1]=%.6e res0=%.3e resr=%.3e |Alast|=%.3e |Tlast|=%.3e drop=%.3e conv=%d\n",
                             nP, nc, (long long)nblock, th[0], th[std::min(r, nc) - 1], res[0] / th[0],
                             res[std::min(r, nc) - 1] / th[0], std::sqrt(an), std::sqrt(bn), std::sqrt(drop2), nconv);
            }
            const bool done = (nconv >= r) || (nblock >= maxprod && nc >= r);
            if (done) {
                // U = Pb · Y[:, 0:r]
                p.U.alloc(sizeof(T) * L * r, st);
                gemm(L, P(0), ldP, nP, Y.data(), nP, r, 1.0, 0.0, p.U.as<T>(), L);
                p.sigma.assign(th.begin(), th.begin() + r);
                p.residuals.assign(res.begin(), res.begin() + r);
                p.r = r;
                break;
            }
            if (!cycle_end) continue;   // early check only: keep growing the Krylov basis
            // ---- thick restart keeping pk Ritz pairs
            ++restarts;
            const double tr0 = now_ms();
            gemm(L, P(0), ldP, nP, Y.data(), nP, pk, 1.0, 0.0, Ptmp.as<T>(), ldP);
            gemm(K, Q(0), ldQ, nc, Z.data(), nc, pk, 1.0, 0.0, Qtmp.as<T>(), ldQ);
            SSA_CUDA(cudaMemcpyAsync(P(0), Ptmp.p, sizeof(T) * ldP * pk, cudaMemcpyDeviceToDevice, st));
            SSA_CUDA(cudaMemcpyAsync(Q(pk), Q(nc), sizeof(T) * ldQ * k, cudaMemcpyDeviceToDevice, st));
            SSA_CUDA(cudaMemcpyAsync(Q(0), Qtmp.p, sizeof(T) * ldQ * pk, cudaMemcpyDeviceToDevice, st));
            std::fill(Tm.begin(), Tm.end(), 0.0);
            for (int i = 0; i < pk; ++i) Tat(i, i) = th[i];
            nP = pk;
            nQ = pk + k;
            tw_restart += now_ms() - tr0;
        }
        if (debug)
            std::fprintf(stderr, "[ssa] host ms: products %.2f orthL %.2f orthK %.2f recurrence %.2f restart %.2f ritz %.2f "
                                 "(fast %lld, fallback %lld)\n",
                         tw_prod, tw_orthA, tw_orthB, tw_rec, tw_restart, ms_ritz, (long long)n_fast,
                         (long long)n_fallback);
        if (debug)
            std::fprintf(stderr, "[ssa] orth3 host ms: L gram(wait) %.2f host %.2f apply(launch) %.2f | K gram %.2f host %.2f apply %.2f\n",
                         tw_o3_gram[0], tw_o3_host[0], tw_o3_apply[0], tw_o3_gram[1], tw_o3_host[1], tw_o3_apply[1]);
        if (debug)
            for (int sd = 0; sd < 2; ++sd)
                std::fprintf(stderr, "[ssa] orth3 %s side: exits at pass 2/3/4 %lld/%lld/%lld, reprojections %lld\n", sd ? "K" : "L",
                             (long long)o3_exit[sd][2], (long long)o3_exit[sd][3], (long long)o3_exit[sd][4], (long long)o3_exit[sd][5]);
        // sign convention: largest-|.| entry of each U_i positive
        for (int c0 = 0; c0 < r; c0 += 1024) {
            const int nc = std::min(1024, r - c0);
            const size_t idx = sg.take(nc);
            absmax_sign<T>(L, p.U.as<T>() + L * c0, L, nc, sg.dev(idx), st);
            scale_columns<T>(L, p.U.as<T>() + L * c0, L, nc, sg.dev(idx), st);
        }
        sg.sync();
        p.v_valid = false;
        p.v_have.clear();
        if (info) {
            info->r_requested = r;
            info->n_converged = nconv;
            info->block_k = k;
            info->n_restarts = restarts;
            info->n_block_products = nblock;
            info->n_vector_products = nvec;
            info->max_rel_residual = maxres;
            info->ms_products = product_ms();
            info->ms_products_xv = product_ms(1);
            info->ms_products_xtu = product_ms(0);
            info->n_products_xv = n_xv;
            info->n_products_xtu = n_xtu;
            info->n_vectors_xv = vec_xv;
            info->n_vectors_xtu = vec_xtu;
            info->ms_ritz = ms_ritz;
            // reading Q10: triples below the product path's measured σ floor τ·σ_1 are not resolvable
            // in this arithmetic (their σ and vectors are rounding-level); report how many there are
            const double tau = sigma_floor(p);
            info->sigma_floor_rel = tau;
            info->n_below_floor = 0;
            for (int i = 0; i < r; ++i) info->n_below_floor += p.sigma[i] < tau * p.sigma[0] ? 1 : 0;
            info->drop_norm_rel = anorm > 0 ? std::sqrt(drop2) / anorm : 0.0;
            info->warm_start_cols = warm_cols;
        }
        if (nconv < r)
            throw Error(SSA_ERR_NOT_CONVERGED, "decomposition stopped at max_products with " + std::to_string(nconv) +
                                                   " of " + std::to_string(r) + " triples converged");
    }
};

// Reading Q10: the σ floor τ = the smallest σ_i/σ_1 down to which the
// decomposition's σ_i meet the σ bar (relative error <= 1e-4), MEASURED on the noiseless c5 twin
// against the closed-form spectrum (scripts/measure_tau.py, profiles/r02/tau.json): 8.7e-5 for the
// fp32 FFT and tensor-core paths at the default tolerance.  fp64 plans resolve to rounding.
double sigma_floor(const PlanImpl &p) { return p.dt == SSA_F64 ? 1e-12 : 8.7e-5; }

template <typename T>
void decompose(PlanImpl &p, int r, ssa_decomp_info *info) {
    Gkl<T> g(p);
    g.run(r, info);
}
template void decompose<float>(PlanImpl &, int, ssa_decomp_info *);
template void decompose<double>(PlanImpl &, int, ssa_decomp_info *);

}  // namespace ssa
