"""The solver's host-side dense kernels (csrc/hostla.cpp: CᵀC-corrected Gram, projection coefficients,
right-looking Cholesky, triangular inverse) against their plain definitions, for both builds (AVX2/FMA when
the CPU has it, and the baseline x86-64 build forced by SSA_HOSTLA_GENERIC).  Host logic only: compiled
here with g++ and run on the CPU."""
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CSRC = os.path.join(ROOT, "paper_1309_5050_b200", "csrc")

DRIVER = r"""
#include "hostla.h"
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <random>
#include <vector>
using namespace ssa::hostla;
int main() {
    std::mt19937_64 g(7);
    std::normal_distribution<double> nd;
    double worst = 0.0;
    int fails = 0;
    for (int kc : {1, 2, 3, 8, 31, 32, 33, 64})
        for (int na : {1, 3, 4, 5, 17, 256, 448}) {
            const int nn = na + kc, off = na;
            std::vector<double> G((size_t)nn * kc), Gp((size_t)kc * kc), S((size_t)kc * kc, 0.0), Mc((size_t)nn * kc);
            for (auto &v : G) v = nd(g);
            gram_minus_ctc(kc, na, nn, off, G.data(), Gp.data());
            double sc = 1.0;
            for (int a = 0; a < kc; ++a)
                for (int b = 0; b < kc; ++b) {
                    const int lo = std::min(a, b), hi = std::max(a, b);
                    double v = G[off + lo + (size_t)nn * hi];
                    for (int t = 0; t < na; ++t) v -= G[t + (size_t)nn * a] * G[t + (size_t)nn * b];
                    worst = std::max(worst, std::fabs(v - Gp[a + (size_t)kc * b]) / (na + 1.0));
                }
            for (int b = 0; b < kc; ++b)
                for (int a = 0; a <= b; ++a) S[a + (size_t)kc * b] = (a == b) ? 1.0 + std::fabs(nd(g)) : 0.1 * nd(g);
            proj_coef(kc, na, nn, G.data(), S.data(), Mc.data());
            for (int b = 0; b < kc; ++b) {
                for (int t = 0; t < na; ++t) {
                    double v = 0.0;
                    for (int a = 0; a <= b; ++a) v -= G[t + (size_t)nn * a] * S[a + (size_t)kc * b];
                    worst = std::max(worst, std::fabs(v - Mc[t + (size_t)nn * b]) / sc);
                }
                for (int a = 0; a < kc; ++a) fails += Mc[na + a + (size_t)nn * b] != S[a + (size_t)kc * b];
            }
        }
    for (int n : {1, 2, 5, 32, 64}) {
        std::vector<double> A((size_t)n * n), G((size_t)n * n), R((size_t)n * n), Sv((size_t)n * n);
        for (auto &v : A) v = nd(g);
        for (int i = 0; i < n; ++i)
            for (int j = 0; j < n; ++j) {
                double s = (i == j) ? n : 0.0;
                for (int t = 0; t < n; ++t) s += A[t + (size_t)n * i] * A[t + (size_t)n * j];
                G[i + (size_t)n * j] = s;
            }
        fails += !cholesky_upper(n, G.data(), 0.0, 1e-14, R.data());
        upper_inverse(n, R.data(), Sv.data());
        for (int i = 0; i < n; ++i)
            for (int j = 0; j < n; ++j) {
                double s = 0.0, p = 0.0;
                for (int t = 0; t < n; ++t) { s += R[t + (size_t)n * i] * R[t + (size_t)n * j]; p += R[i + (size_t)n * t] * Sv[t + (size_t)n * j]; }
                worst = std::max(worst, std::fabs(s - G[i + (size_t)n * j]) / (4.0 * n * n));
                worst = std::max(worst, std::fabs(p - (i == j ? 1.0 : 0.0)));
                if (i > j) fails += (R[i + (size_t)n * j] != 0.0) + (Sv[i + (size_t)n * j] != 0.0);
            }
    }
    std::vector<double> Gi = {1, 2, 2, 1}, Ri(4);
    fails += cholesky_upper(2, Gi.data(), 0.0, 1e-14, Ri.data());           // indefinite: rejected
    fails += !cholesky_upper(2, Gi.data(), 2.0, 1e-14, Ri.data());          // shifted: accepted
    std::vector<double> Z(4, 0.0);
    fails += cholesky_upper(2, Z.data(), 0.0, 1e-14, Ri.data());            // zero Gram: rejected
    std::printf("%d %.3e\n", fails, worst);
    return 0;
}
"""


@pytest.fixture(scope="module")
def driver(tmp_path_factory):
    if shutil.which("g++") is None:
        pytest.skip("g++ not available")
    d = tmp_path_factory.mktemp("hostla")
    src = d / "drv.cpp"
    src.write_text(DRIVER)
    exe = d / "drv"
    subprocess.run(["g++", "-O2", "-std=c++17", "-I", CSRC, str(src), os.path.join(CSRC, "hostla.cpp"), "-o", str(exe)],
                   check=True, capture_output=True)
    return str(exe)


@pytest.mark.parametrize("generic", [False, True])
def test_hostla_matches_definitions(driver, generic):
    env = dict(os.environ)
    if generic:
        env["SSA_HOSTLA_GENERIC"] = "1"
    out = subprocess.run([driver], capture_output=True, text=True, env=env, check=True).stdout.split()
    fails, worst = int(out[0]), float(out[1])
    assert fails == 0
    assert worst < 1e-12
