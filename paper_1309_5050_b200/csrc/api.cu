// C ABI of libssa_b200 (include/ssa_b200.h): plan creation (embedding, step 1),
// product dispatch, decomposition (step 2), reconstruction (steps 3-4).
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstring>
#include <map>
#include <mutex>
#include <tuple>
#include <vector>

#include "common.h"
#include "kernels.h"
#include "plan.h"

namespace ssa {

static thread_local std::string g_err;
static thread_local int64_t g_launches = 0;

void count_launch(int n) { g_launches += n; }
void ssa_set_error(const std::string &msg) { g_err = msg; }
void after_launch(const char *what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) throw Error(SSA_ERR_CUDA, std::string("launch of ") + what + ": " + cudaGetErrorString(e));
    ++g_launches;
}

void pool_init() {
    static thread_local int done_dev = -1;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return;
    if (done_dev == dev) return;
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        uint64_t keep = UINT64_MAX;   // retain freed blocks for reuse by later plans
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
    done_dev = dev;
}

namespace {
struct BigBlock { void *p; size_t bytes; cudaStream_t st; cudaEvent_t ev; int dev; };
// free a cached block: ordered after its last use through its event (the stream it was last used on may
// be gone by now)
void big_free(const BigBlock &b) {
    if (cudaStreamWaitEvent(cudaStreamPerThread, b.ev, 0) == cudaSuccess) cudaFreeAsync(b.p, cudaStreamPerThread);
    else { cudaGetLastError(); cudaFree(b.p); }
    cudaEventDestroy(b.ev);
}
// blocks of host threads that have exited: any thread may take them.  Allocated once and never destroyed:
// no CUDA call and no destructor may run during process exit (the runtime may already be gone).
struct Orphans { std::mutex m; std::vector<BigBlock> blocks; std::atomic<size_t> n{0}; };
Orphans &orphans() { static Orphans *o = new Orphans; return *o; }
thread_local bool tl_big_dead = false;   // trivially destructible: still valid after ~BigCache
struct BigCache {
    std::vector<BigBlock> blocks;   // oldest first
    size_t total = 0;
    void drop(size_t i) {
        const BigBlock b = blocks[i];
        blocks.erase(blocks.begin() + (std::ptrdiff_t)i);
        total -= b.bytes;
        big_free(b);
    }
    void clear() { while (!blocks.empty()) drop(blocks.size() - 1); }
    // thread exit (for the main thread: process exit): no CUDA calls here; the blocks go to the orphan list
    ~BigCache() {
        tl_big_dead = true;
        if (blocks.empty()) return;
        Orphans &o = orphans();
        std::lock_guard<std::mutex> g(o.m);
        o.blocks.insert(o.blocks.end(), blocks.begin(), blocks.end());
        o.n = o.blocks.size();
    }
};
BigCache &big_cache() { static thread_local BigCache c; return c; }
constexpr size_t kBigCacheCap = (size_t)64 << 30;

bool big_match(const BigBlock &b, size_t n, int dev, cudaStream_t st) {
    if (b.bytes != n || b.dev != dev) return false;
    if (b.st != st && cudaStreamWaitEvent(st, b.ev, 0) != cudaSuccess) { cudaGetLastError(); return false; }
    return true;
}
}  // namespace

void *big_take(size_t n, cudaStream_t st) {
    if (tl_big_dead) return nullptr;
    BigCache &c = big_cache();
    Orphans &o = orphans();
    if (c.blocks.empty() && o.n == 0) return nullptr;
    int dev = 0;
    cudaGetDevice(&dev);
    for (size_t i = c.blocks.size(); i-- > 0;) {
        if (!big_match(c.blocks[i], n, dev, st)) continue;
        void *p = c.blocks[i].p;
        cudaEventDestroy(c.blocks[i].ev);
        c.total -= n;
        c.blocks.erase(c.blocks.begin() + (std::ptrdiff_t)i);
        return p;
    }
    if (o.n != 0) {
        std::lock_guard<std::mutex> g(o.m);
        for (size_t i = o.blocks.size(); i-- > 0;) {
            if (!big_match(o.blocks[i], n, dev, st)) continue;
            void *p = o.blocks[i].p;
            cudaEventDestroy(o.blocks[i].ev);
            o.blocks.erase(o.blocks.begin() + (std::ptrdiff_t)i);
            o.n = o.blocks.size();
            return p;
        }
    }
    return nullptr;
}

bool big_give(void *p, size_t n, cudaStream_t st) {
    if (tl_big_dead || n > kBigCacheCap) return false;   // dead: a thread_local holder outlived the cache
    BigCache &c = big_cache();
    BigBlock b{p, n, st, nullptr, 0};
    if (cudaGetDevice(&b.dev) != cudaSuccess || cudaEventCreateWithFlags(&b.ev, cudaEventDisableTiming) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    if (cudaEventRecord(b.ev, st) != cudaSuccess) {
        cudaGetLastError();
        cudaEventDestroy(b.ev);
        return false;
    }
    c.blocks.push_back(b);
    c.total += n;
    while (c.total > kBigCacheCap && c.blocks.size() > 1) c.drop(0);
    return true;
}

void big_release_all() {
    if (!tl_big_dead) big_cache().clear();
    Orphans &o = orphans();
    std::lock_guard<std::mutex> g(o.m);
    for (const BigBlock &b : o.blocks) big_free(b);
    o.blocks.clear();
    o.n = 0;
}

int num_sms() {
    static int n = 0;
    if (n == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        if (n <= 0) n = 148;
    }
    return n;
}

PlanImpl::~PlanImpl() {
    if (fft) fft_destroy(fft);
    fft = nullptr;
}

double *small_dev(PlanImpl &p, size_t n) {
    p.dsmall.alloc(std::max<size_t>(n, 64 * 64) * sizeof(double), p.st);
    return p.dsmall.as<double>();
}

template <typename T>
__global__ void u8_to_T_kernel(const uint8_t *m, int64_t n, T *out) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x)
        out[t] = m[t] ? T(1) : T(0);
}

// band assembly (multi-GPU reconstruction): dst[g][x, y0 + y] = src[g][x, y] for the band's columns,
// zero elsewhere (nb = number of arrays, each nx x ny_src into nx x ny_dst)
template <typename T>
__global__ void place_band_kernel(const T *src, int nx, int ny_src, int64_t ncols, T *dst, int ny_dst, int64_t y0,
                                  int nb) {
    const int64_t per = (int64_t)nx * ny_dst, tot = per * nb;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < tot; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t g = t / per, r = t - g * per;
        const int64_t y = r / nx - y0, x = r % nx;
        dst[t] = (y >= 0 && y < ncols) ? src[g * (int64_t)nx * ny_src + x + (int64_t)nx * y] : T(0);
    }
}
template <typename T>
__global__ void int_to_T_kernel(const int32_t *w, int64_t n, T *out) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x)
        out[t] = (T)w[t];
}
// out[g][n] = num[g][n] / w[n] on w > 0, NaN elsewhere (Alg. 4 step 3 on the assembled bands)
template <typename T>
__global__ void divide_weights_kernel(T *num, const T *w, int64_t n, int ng) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n * ng; t += (int64_t)gridDim.x * blockDim.x) {
        const T wn = w[t % n];
        num[t] = wn > T(0) ? num[t] / wn : (T)NAN;
    }
}

template <typename T>
__global__ void weighted_sqrt_kernel(T *a, const int32_t *w, int64_t n, int ng) {
    const int64_t tot = n * ng;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < tot; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t c = t % n;
        const T v = a[t];
        a[t] = (w[c] > 0 && isfinite((double)v)) ? v * (T)sqrt((double)w[c]) : T(0);
    }
}

// number of nonzero entries of a u8 mask or of an int32 array, on the device
__global__ void count_nonzero_kernel(const uint8_t *m8, const int32_t *m32, int64_t n, unsigned long long *out) {
    unsigned long long c = 0;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x)
        c += m8 ? (m8[t] != 0) : (m32[t] > 0);
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(out, c);
}
static int64_t count_device(PlanImpl &p, const uint8_t *m8, const int32_t *m32, int64_t n) {
    DevBuf d;
    d.alloc(sizeof(unsigned long long), p.st);
    SSA_CUDA(cudaMemsetAsync(d.p, 0, sizeof(unsigned long long), p.st));
    count_nonzero_kernel<<<(unsigned)std::min<int64_t>(cdiv(n, 256), 8 * num_sms()), 256, 0, p.st>>>(
        m8, m32, n, d.as<unsigned long long>());
    after_launch("count_nonzero");
    unsigned long long h = 0;
    SSA_CUDA(cudaMemcpyAsync(&h, d.p, sizeof(h), cudaMemcpyDeviceToHost, p.st));
    SSA_CUDA(cudaStreamSynchronize(p.st));
    return (int64_t)h;
}

// ---------------------------------------------------------------- products
template <typename T>
static CorrParams<T> base_corr(PlanImpl &p) {
    CorrParams<T> c{};
    c.x = p.img.as<T>(); c.ldx = p.nx; c.nx = p.nx; c.ny = p.ny;
    return c;
}

template <typename T>
static void tc_dispatch(PlanImpl &p, bool xv, const T *in, int64_t ldi, T *out, int64_t ldo, int k) {
    if constexpr (sizeof(T) == 4) {
        if (!p.tc_xhi.p) {
            const size_t nb = sizeof(float) * (size_t)tc_plane_ld(p.nx) * p.ny;
            p.tc_xhi.alloc(nb, p.st);
            p.tc_xlo.alloc(nb, p.st);
            tc_build_planes(p.img.as<float>(), p.nx, p.nx, p.ny, p.tc_xhi.as<float>(), p.tc_xlo.as<float>(), p.st);
        }
        TcCorrParams c{};
        c.x_hi = p.tc_xhi.as<float>(); c.x_lo = p.tc_xlo.as<float>(); c.nx = p.nx; c.ny = p.ny;
        if (xv) {
            c.ox = p.lx; c.oy = p.ly; c.bx = p.kx; c.by = p.ky;
            c.imap = p.full_k ? nullptr : p.kmap.as<int>(); c.omap = p.full_window ? nullptr : p.lmap.as<int>();
        } else {
            c.ox = p.kx; c.oy = p.ky; c.bx = p.lx; c.by = p.ly;
            c.imap = p.full_window ? nullptr : p.lmap.as<int>(); c.omap = p.full_k ? nullptr : p.kmap.as<int>();
        }
        c.in = in; c.ldi = ldi; c.out = out; c.ldo = ldo; c.k = k;
        const size_t need = tc_pack_bytes(c.bx, c.by, k);
        if (need > p.tc_bpk_bytes) { p.tc_bpk.alloc(need, p.st); p.tc_bpk_bytes = need; }
        c.bpk = p.tc_bpk.as<float>(); c.bpk_bytes = p.tc_bpk_bytes;
        c.ws = p.ws_corr.as<float>(); c.ws_bytes = p.ws_corr_bytes;
        tc_corr(c, p.st);
    } else {
        (void)p; (void)xv; (void)in; (void)ldi; (void)out; (void)ldo; (void)k;
        throw Error(SSA_ERR_ARG, "tensor-core path is fp32 only");
    }
}

template <typename T>
void op_xtu(PlanImpl &p, const T *U, int64_t ldu, T *V, int64_t ldv, int k, const double *cs) {
    if (p.path_xtu == SSA_PATH_FFT && p.fft) { fft_xtu<T>(p, U, ldu, V, ldv, k, cs); return; }
    if (p.path_xtu == SSA_PATH_TC) {
        tc_dispatch<T>(p, false, U, ldu, V, ldv, k);
        if (cs) scale_columns<T>(p.K, V, ldv, k, cs, p.st);
        return;
    }
    CorrParams<T> c = base_corr<T>(p);
    c.ox = p.kx; c.oy = p.ky; c.dx = p.lx; c.dy = p.ly;
    c.W = U; c.ldw = ldu; c.wmap = p.full_window ? nullptr : p.lmap.as<int>();
    c.out = V; c.ldo = ldv; c.omap = p.full_k ? nullptr : p.kmap.as<int>();
    c.k = k;
    corr_direct<T>(c, p.ws_corr.as<T>(), p.ws_corr_bytes, p.st);
    if (cs) scale_columns<T>(p.K, V, ldv, k, cs, p.st);
}

template <typename T>
void op_xv(PlanImpl &p, const T *V, int64_t ldv, T *U, int64_t ldu, int k) {
    if (p.path_xv == SSA_PATH_FFT && p.fft) {
        fft_xv<T>(p, V, ldv, U, ldu, k);
    } else if (p.path_xv == SSA_PATH_TC) {
        tc_dispatch<T>(p, true, V, ldv, U, ldu, k);
    } else {
        CorrParams<T> c = base_corr<T>(p);
        c.ox = p.lx; c.oy = p.ly; c.dx = p.kx; c.dy = p.ky;
        c.W = V; c.ldw = ldv; c.wmap = p.full_k ? nullptr : p.kmap.as<int>();
        c.out = U; c.ldo = ldu; c.omap = p.full_window ? nullptr : p.lmap.as<int>();
        c.k = k;
        corr_direct<T>(c, p.ws_corr.as<T>(), p.ws_corr_bytes, p.st);
    }
    // window-position band partition: sum the L x k partials
    if (p.has_comm && p.comm.world > 1) {
        // one allreduce over the k columns as stored (ldu >= L; rows L..ldu-1 between the
        // columns are the solver's zero padding, identical on every rank, or caller scratch)
        if (ldu < p.L) throw Error(SSA_ERR_ARG, "X·V output leading dimension below L");
        if (p.comm.allreduce_sum(p.comm.user, U, ldu * (int64_t)(k - 1) + p.L, p.dt, p.st) != 0)
            throw Error(SSA_ERR_COMM, "allreduce of X·V partials failed");
    }
}
template void op_xtu<float>(PlanImpl &, const float *, int64_t, float *, int64_t, int, const double *);
template void op_xtu<double>(PlanImpl &, const double *, int64_t, double *, int64_t, int, const double *);
template void op_xv<float>(PlanImpl &, const float *, int64_t, float *, int64_t, int);
template void op_xv<double>(PlanImpl &, const double *, int64_t, double *, int64_t, int);

// ---------------------------------------------------------------- path choice
// Candidates per product: FFT correlation (fft_supported), tensor-core 3xTF32
// implicit GEMM (fp32, output box rows >= 96) and the CUDA-core direct kernel.
// AUTO prunes by a cost model and times the survivors on the plan's stream (one
// block of k vectors, best of 3 after a warm-up); the decision is cached per shape
// for the process.  An explicit opts.path is honoured where the product supports it.
struct PathKey {
    int nx, ny, lx, ly, kx, ky; int64_t L, K; int dt, k, xv, fw, fk;
    bool operator<(const PathKey &o) const {
        return std::tie(nx, ny, lx, ly, kx, ky, L, K, dt, k, xv, fw, fk) <
               std::tie(o.nx, o.ny, o.lx, o.ly, o.kx, o.ky, o.L, o.K, o.dt, o.k, o.xv, o.fw, o.fk);
    }
};

template <typename T>
static double time_product(PlanImpl &p, bool xv, int path, int k, T *in, T *out) {
    const int save_xv = p.path_xv, save_xtu = p.path_xtu;
    const bool save_comm = p.has_comm;
    p.has_comm = false;   // time the local product only: no collective during the choice
    (xv ? p.path_xv : p.path_xtu) = path;
    cudaEvent_t e0, e1;
    SSA_CUDA(cudaEventCreate(&e0)); SSA_CUDA(cudaEventCreate(&e1));
    float best = 1e30f;
    for (int rep = 0; rep < 4; ++rep) {
        SSA_CUDA(cudaEventRecord(e0, p.st));
        if (xv) op_xv<T>(p, in, p.K, out, p.L, k);
        else op_xtu<T>(p, in, p.L, out, p.K, k);
        SSA_CUDA(cudaEventRecord(e1, p.st));
        SSA_CUDA(cudaEventSynchronize(e1));
        float ms = 0.f;
        SSA_CUDA(cudaEventElapsedTime(&ms, e0, e1));
        if (rep > 0) best = std::min(best, ms);
    }
    cudaEventDestroy(e0); cudaEventDestroy(e1);
    p.path_xv = save_xv; p.path_xtu = save_xtu;
    p.has_comm = save_comm;
    return best;
}

template <typename T>
static void choose_paths(PlanImpl &p) {
    const bool fft_ok = fft_supported(p);
    if (fft_ok && (p.path == SSA_PATH_FFT || p.path == SSA_PATH_AUTO)) fft_build(p);
    const int k = std::max(1, std::min<int>(p.block_k, 64));
    const bool is32 = sizeof(T) == 4;
    const bool tc_xv = is32 && tc_corr_supported(p.lx, p.ly, p.kx, p.ky, k);
    const bool tc_xtu = is32 && tc_corr_supported(p.kx, p.ky, p.lx, p.ly, k);
    auto fallback = [&](bool tc_ok) { return tc_ok ? SSA_PATH_TC : SSA_PATH_DIRECT; };
    if (p.path == SSA_PATH_FFT) {
        if (!fft_ok) throw Error(SSA_ERR_ARG, "FFT path not available for this shape");
        p.path_xv = p.path_xtu = SSA_PATH_FFT;
        return;
    }
    if (p.path == SSA_PATH_DIRECT) { p.path_xv = p.path_xtu = SSA_PATH_DIRECT; return; }
    if (p.path == SSA_PATH_TC) {
        if (!is32) throw Error(SSA_ERR_ARG, "tensor-core path is fp32 only");
        // products whose output box is too narrow for M = 128 tiles use the FFT / direct path
        p.path_xv = tc_xv ? SSA_PATH_TC : (fft_ok ? SSA_PATH_FFT : SSA_PATH_DIRECT);
        p.path_xtu = tc_xtu ? SSA_PATH_TC : (fft_ok ? SSA_PATH_FFT : SSA_PATH_DIRECT);
        if (!p.fft && fft_ok && (p.path_xv == SSA_PATH_FFT || p.path_xtu == SSA_PATH_FFT)) fft_build(p);
        return;
    }
    // AUTO
    static std::mutex mu;
    static std::map<PathKey, int> cache;
    const double flops = 2.0 * (double)p.L * (double)p.K * k;
    for (int xv = 0; xv < 2; ++xv) {
        const bool tc_ok = xv ? tc_xv : tc_xtu;
        PathKey key{p.nx, p.ny, p.lx, p.ly, p.kx, p.ky, p.L, p.K, (int)p.dt, k, xv, (int)p.full_window, (int)p.full_k};
        int choice = -1;
        {
            std::lock_guard<std::mutex> g(mu);
            auto itc = cache.find(key);
            if (itc != cache.end()) choice = itc->second;
        }
        if (choice < 0) {
            // cost model (µs) to prune hopeless candidates before timing
            std::vector<std::pair<int, double>> cand;
            const double t_direct = flops / (is32 ? 30e6 : 15e6);
            const double t_tc = flops / 150e6;
            if (fft_ok) cand.push_back({SSA_PATH_FFT, 0.0});
            if (tc_ok) cand.push_back({SSA_PATH_TC, t_tc});
            cand.push_back({SSA_PATH_DIRECT, t_direct});
            if (cand.size() == 1 || (!fft_ok && !tc_ok)) {
                choice = SSA_PATH_DIRECT;
            } else {
                DevBuf bin, bout;
                bin.alloc(sizeof(T) * (size_t)std::max(p.L, p.K) * k, p.st);
                bout.alloc(sizeof(T) * (size_t)std::max(p.L, p.K) * k, p.st);
                SSA_CUDA(cudaMemsetAsync(bin.p, 0, bin.bytes, p.st));
                double best = 1e300;
                for (auto &c : cand) {
                    // never time a candidate predicted > 20 ms or > 8x the best measured
                    if (c.second > 2e4 || c.second > 3.0 * best * 1e3) continue;
                    const double ms = time_product<T>(p, xv, c.first, k, bin.as<T>(), bout.as<T>());
                    if (ms < best) { best = ms; choice = c.first; }
                }
                if (choice < 0) choice = fft_ok ? SSA_PATH_FFT : fallback(tc_ok);
            }
            std::lock_guard<std::mutex> g(mu);
            cache[key] = choice;
        }
        (xv ? p.path_xv : p.path_xtu) = choice;
    }
    if (!fft_ok || (p.path_xv != SSA_PATH_FFT && p.path_xtu != SSA_PATH_FFT)) {
        // keep the spectrum only if a product or the averaging uses it
        (void)0;
    }
    p.path = p.path_xv;
}

// ---------------------------------------------------------------- plan creation
template <typename T>
static void build_plan(PlanImpl &p, const ssa_array *x, const uint8_t *mask_host) {
    cudaStream_t st = p.st;
    const int64_t nxy = (int64_t)p.nx * p.ny;
    // a1: image and 𝔑
    DevBuf stage, dmask;
    const int64_t ld = x->ld > 0 ? x->ld : x->nx;
    const T *src = nullptr;
    if (x->on_device) {
        if ((x->dtype == SSA_F64) == (sizeof(T) == 8)) {
            src = static_cast<const T *>(x->data);
        } else {
            stage.alloc(sizeof(T) * ld * p.ny, st);
            cast_copy<T>(x->data, x->dtype == SSA_F64, stage.as<T>(), ld * p.ny, st);
            src = stage.as<T>();
        }
    } else {
        const size_t esz = x->dtype == SSA_F64 ? 8 : 4;
        DevBuf raw;
        raw.alloc(esz * ld * p.ny, st);
        SSA_CUDA(cudaMemcpyAsync(raw.p, x->data, esz * ld * p.ny, cudaMemcpyHostToDevice, st));
        stage.alloc(sizeof(T) * ld * p.ny, st);
        cast_copy<T>(raw.p, x->dtype == SSA_F64, stage.as<T>(), ld * p.ny, st);
        SSA_CUDA(cudaStreamSynchronize(st));
        src = stage.as<T>();
    }
    if (mask_host) {
        dmask.alloc(nxy, st);
        SSA_CUDA(cudaMemcpyAsync(dmask.p, mask_host, nxy, cudaMemcpyHostToDevice, st));
    }
    p.img.alloc(sizeof(T) * nxy, st);
    p.nmask.alloc(nxy, st);
    prep_image<T>(src, ld, p.nx, p.ny, mask_host ? dmask.as<uint8_t>() : nullptr, p.img.as<T>(),
                  p.nmask.as<uint8_t>(), st);
    // |𝔑| counted on the device (a host copy and loop over the 16.7M cells of c5 cost ~6 ms of the plan)
    p.n_valid = count_device(p, p.nmask.as<uint8_t>(), nullptr, nxy);

    // 𝔏 map
    if (!p.full_window) {
        p.lmap.alloc(sizeof(int32_t) * p.lx * p.ly, st);
        SSA_CUDA(cudaMemcpyAsync(p.lmap.p, p.lmap_host.data(), sizeof(int32_t) * p.lx * p.ly,
                                 cudaMemcpyHostToDevice, st));
    }
    // a2: 𝔎 by Alg. 6: v = 𝒯ᵀ(I^𝔑)·1_𝔏 ;  𝔎 = {v = |𝔏|}
    const int64_t nk = (int64_t)p.kx * p.ky;
    p.kmask.alloc(nk, st);
    const bool trivial = (p.n_valid == nxy) && p.full_window;
    if (trivial) {
        SSA_CUDA(cudaMemsetAsync(p.kmask.p, 1, nk, st));
        p.full_k = true;
        p.K = nk;
    } else if (p.full_window) {
        // rectangular window: 𝔎 by separable box sums of 1_𝔑 (exact int32; same set as the
        // correlation below, without an L·K-flop kernel)
        DevBuf tmp;
        tmp.alloc(sizeof(int32_t) * (size_t)p.kx * p.ny, st);
        box_kmask(p.nmask.as<uint8_t>(), p.nx, p.ny, p.lx, p.ly, p.kmask.as<uint8_t>(), tmp.as<int32_t>(), st);
        DevBuf cc;
        cc.alloc(sizeof(int32_t) * (p.ky + 1), st);
        column_counts(p.kmask.as<uint8_t>(), p.kx, p.ky, cc.as<int32_t>(), st);
        std::vector<int32_t> h(p.ky + 1, 0);
        SSA_CUDA(cudaMemcpyAsync(h.data(), cc.p, sizeof(int32_t) * p.ky, cudaMemcpyDeviceToHost, st));
        SSA_CUDA(cudaStreamSynchronize(st));
        int64_t tot = 0;
        for (int j = 0; j < p.ky; ++j) { const int32_t c0 = h[j]; h[j] = (int32_t)tot; tot += c0; }
        p.K = tot;
        p.full_k = (tot == nk);
        if (!p.full_k) {
            SSA_CUDA(cudaMemcpyAsync(cc.p, h.data(), sizeof(int32_t) * p.ky, cudaMemcpyHostToDevice, st));
            p.kmap.alloc(sizeof(int32_t) * nk, st);
            compact_map(p.kmask.as<uint8_t>(), p.kx, p.ky, cc.as<int32_t>(), p.kmap.as<int32_t>(), nullptr, p.nx, st);
        }
        SSA_CUDA(cudaStreamSynchronize(st));
    } else {
        DevBuf ind, ones, cnt, ws;
        ind.alloc(sizeof(T) * nxy, st);
        u8_to_T_kernel<T><<<(unsigned)std::min<int64_t>(cdiv(nxy, 256), 16 * num_sms()), 256, 0, st>>>(
            p.nmask.as<uint8_t>(), nxy, ind.as<T>());
        after_launch("u8_to_T");
        std::vector<T> one(p.L, T(1));
        ones.alloc(sizeof(T) * p.L, st);
        SSA_CUDA(cudaMemcpyAsync(ones.p, one.data(), sizeof(T) * p.L, cudaMemcpyHostToDevice, st));
        cnt.alloc(sizeof(T) * nk, st);
        CorrParams<T> c{};
        c.x = ind.as<T>(); c.ldx = p.nx; c.nx = p.nx; c.ny = p.ny;
        c.ox = p.kx; c.oy = p.ky; c.dx = p.lx; c.dy = p.ly;
        c.W = ones.as<T>(); c.ldw = p.L; c.wmap = p.full_window ? nullptr : p.lmap.as<int>();
        c.out = cnt.as<T>(); c.ldo = nk; c.omap = nullptr; c.k = 1;
        const size_t wsb = sizeof(T) * nk * 64;
        ws.alloc(wsb, st);
        corr_direct<T>(c, ws.as<T>(), wsb, st);
        threshold_eq<T>(cnt.as<T>(), nk, (double)p.L, p.kmask.as<uint8_t>(), st);
        // compaction map box -> 𝔎 index (lex order)
        DevBuf cc;
        cc.alloc(sizeof(int32_t) * (p.ky + 1), st);
        column_counts(p.kmask.as<uint8_t>(), p.kx, p.ky, cc.as<int32_t>(), st);
        std::vector<int32_t> h(p.ky + 1, 0);
        SSA_CUDA(cudaMemcpyAsync(h.data(), cc.p, sizeof(int32_t) * p.ky, cudaMemcpyDeviceToHost, st));
        SSA_CUDA(cudaStreamSynchronize(st));
        int64_t tot = 0;
        for (int j = 0; j < p.ky; ++j) { const int32_t c0 = h[j]; h[j] = (int32_t)tot; tot += c0; }
        p.K = tot;
        p.full_k = (tot == nk);
        if (!p.full_k) {
            SSA_CUDA(cudaMemcpyAsync(cc.p, h.data(), sizeof(int32_t) * p.ky, cudaMemcpyHostToDevice, st));
            p.kmap.alloc(sizeof(int32_t) * nk, st);
            compact_map(p.kmask.as<uint8_t>(), p.kx, p.ky, cc.as<int32_t>(), p.kmap.as<int32_t>(), nullptr, p.nx, st);
        }
        SSA_CUDA(cudaStreamSynchronize(st));
    }
    if (p.K == 0) throw Error(SSA_ERR_EMPTY_KSHAPE, "no window position fits inside the shape (K-shape is empty)");

    // a3: weights 𝕎 = diagsums(1_𝔏, 1_𝔎) (Alg. 4 step 1)
    p.weights.alloc(sizeof(int32_t) * nxy, st);
    if (p.full_window && p.full_k) {
        weights_rect(p.nx, p.ny, p.lx, p.ly, p.weights.as<int32_t>(), st);
        p.n_excluded = p.n_valid - nxy;   // all cells valid in this case -> 0
        if (p.n_excluded < 0) p.n_excluded = 0;
    } else if (p.full_window) {
        // 𝕎 = box sum of 1_𝔎 over the window (exact int32)
        DevBuf tmp;
        tmp.alloc(sizeof(int32_t) * (size_t)p.nx * p.ky, st);
        box_weights(p.kmask.as<uint8_t>(), p.nx, p.ny, p.lx, p.ly, p.weights.as<int32_t>(), tmp.as<int32_t>(), st);
        const int64_t np = count_device(p, nullptr, p.weights.as<int32_t>(), nxy);   // |𝔑′|
        p.n_excluded = p.n_valid - np;   // band plans: cells of the band's sub-image
    } else {
        DevBuf num, go, gi;
        num.alloc(sizeof(T) * nxy, st);
        int32_t hoff[2] = {0, 1}, hidx[1] = {0};
        go.alloc(sizeof(hoff), st); gi.alloc(sizeof(hidx), st);
        SSA_CUDA(cudaMemcpyAsync(go.p, hoff, sizeof(hoff), cudaMemcpyHostToDevice, st));
        SSA_CUDA(cudaMemcpyAsync(gi.p, hidx, sizeof(hidx), cudaMemcpyHostToDevice, st));
        AvgParams<T> a{};
        a.nx = p.nx; a.ny = p.ny;
        a.lx = p.lx; a.ly = p.ly; a.lmap = p.full_window ? nullptr : p.lmap.as<int>();
        a.kx = p.kx; a.ky = p.ky; a.kmap = p.full_k ? nullptr : p.kmap.as<int>();
        a.U = nullptr; a.V = nullptr; a.coef = nullptr;
        a.grp_off = go.as<int>(); a.grp_idx = gi.as<int>(); a.ngroups = 1;
        a.w = nullptr; a.out = num.as<T>(); a.ldout = p.nx; a.out_stride = nxy;
        diagsums_direct<T>(a, st);
        box_ones_to_int<T>(num.as<T>(), nxy, p.weights.as<int32_t>(), st);
        const int64_t np = count_device(p, nullptr, p.weights.as<int32_t>(), nxy);   // |𝔑′|
        p.n_excluded = p.n_valid - np;   // band plans: cells of the band's sub-image
    }
    // workspaces
    const int kmax = std::max(64, p.block_k);
    p.ws_corr_bytes = std::min<size_t>((size_t)256 << 20,
                                       (size_t)64 * p.lx * p.ly * (size_t)kmax * sizeof(T));
    p.ws_corr_bytes = std::max(p.ws_corr_bytes, (size_t)p.lx * p.ly * (size_t)kmax * sizeof(T) * 2);
    p.ws_corr.alloc(p.ws_corr_bytes, st);
    p.ws_gram.alloc(gram_partial_bytes(std::max<int64_t>({p.L, p.K, nxy}), 512, 64), st);
    // product path (per product; SURVEY north star: "the choice made per shape from measurement")
    choose_paths<T>(p);
    SSA_CUDA(cudaStreamSynchronize(st));
}

// V_i = Xᵀu_i / σ_i, computed on demand: all r columns (ssa_get_v), or only the columns a
// reconstruction references (c5: 6 of 50 — one Xᵀ·U block of 6 instead of 50 vectors)
template <typename T>
static void get_v(PlanImpl &p, const std::vector<int> *need = nullptr) {
    if (p.v_valid) return;
    if ((int)p.v_have.size() != p.r) {
        p.v_have.assign(p.r, 0);
        p.V.alloc(sizeof(T) * p.K * std::max(p.r, 1), p.st);
    }
    std::vector<int> miss;
    for (int i = 0; i < p.r; ++i)
        if (!p.v_have[i] && (!need || std::find(need->begin(), need->end(), i) != need->end())) miss.push_back(i);
    if (!miss.empty()) {
        const int nm = (int)miss.size();
        std::vector<double> inv(nm);
        for (int t = 0; t < nm; ++t) inv[t] = p.sigma[miss[t]] > 0 ? 1.0 / p.sigma[miss[t]] : 0.0;
        double *d = small_dev(p, std::max(nm, 1));
        SSA_CUDA(cudaMemcpyAsync(d, inv.data(), sizeof(double) * nm, cudaMemcpyHostToDevice, p.st));
        if (nm == p.r) {
            op_xtu<T>(p, p.U.as<T>(), p.L, p.V.as<T>(), p.K, p.r, d);   // ÷σ inside the product
        } else {
            DevBuf ut, vt;
            ut.alloc(sizeof(T) * p.L * nm, p.st);
            vt.alloc(sizeof(T) * p.K * nm, p.st);
            for (int t = 0; t < nm; ++t)
                SSA_CUDA(cudaMemcpyAsync(ut.as<T>() + p.L * t, p.U.as<T>() + p.L * miss[t], sizeof(T) * p.L,
                                         cudaMemcpyDeviceToDevice, p.st));
            op_xtu<T>(p, ut.as<T>(), p.L, vt.as<T>(), p.K, nm, d);
            for (int t = 0; t < nm; ++t)
                SSA_CUDA(cudaMemcpyAsync(p.V.as<T>() + p.K * miss[t], vt.as<T>() + p.K * t, sizeof(T) * p.K,
                                         cudaMemcpyDeviceToDevice, p.st));
        }
        SSA_CUDA(cudaStreamSynchronize(p.st));
        for (int i : miss) p.v_have[i] = 1;
    }
    if (std::all_of(p.v_have.begin(), p.v_have.end(), [](char c) { return c != 0; })) p.v_valid = true;
}

template <typename T> void get_v_cols(PlanImpl &p, const std::vector<int> &need) { get_v<T>(p, &need); }
template void get_v_cols<float>(PlanImpl &, const std::vector<int> &);
template void get_v_cols<double>(PlanImpl &, const std::vector<int> &);

template <typename T>
static void reconstruct_impl(PlanImpl &p, const int32_t *off, const int32_t *idx, int ng, int add_rest, T *out_dev,
                             const int32_t *wdiv = nullptr) {
    if (!wdiv) wdiv = p.weights.as<int32_t>();
    {
        std::vector<int> need(idx, idx + off[ng]);
        get_v<T>(p, &need);
    }
    const int64_t nxy = (int64_t)p.nx * p.ny;
    DevBuf go, gi, sig;
    const int nidx = off[ng];
    go.alloc(sizeof(int32_t) * (ng + 1), p.st);
    gi.alloc(sizeof(int32_t) * std::max(nidx, 1), p.st);
    sig.alloc(sizeof(double) * p.r, p.st);
    SSA_CUDA(cudaMemcpyAsync(go.p, off, sizeof(int32_t) * (ng + 1), cudaMemcpyHostToDevice, p.st));
    if (nidx) SSA_CUDA(cudaMemcpyAsync(gi.p, idx, sizeof(int32_t) * nidx, cudaMemcpyHostToDevice, p.st));
    SSA_CUDA(cudaMemcpyAsync(sig.p, p.sigma.data(), sizeof(double) * p.r, cudaMemcpyHostToDevice, p.st));
    if (ng > 0 && p.fft) {
        // eigentriples referenced by the groups, and their slot in the batched spectra
        std::vector<int> used, slot(p.r, -1);
        for (int t = 0; t < nidx; ++t)
            if (slot[idx[t]] < 0) { slot[idx[t]] = (int)used.size(); used.push_back(idx[t]); }
        DevBuf ds;
        ds.alloc(sizeof(int) * p.r, p.st);
        SSA_CUDA(cudaMemcpyAsync(ds.p, slot.data(), sizeof(int) * p.r, cudaMemcpyHostToDevice, p.st));
        fft_diagsums<T>(p, p.U.as<T>(), p.V.as<T>(), sig.as<double>(), go.as<int>(), gi.as<int>(), ng, used,
                        ds.as<int>(), out_dev, wdiv);
    } else if (ng > 0) {
        AvgParams<T> a{};
        a.nx = p.nx; a.ny = p.ny;
        a.lx = p.lx; a.ly = p.ly; a.lmap = p.full_window ? nullptr : p.lmap.as<int>();
        a.kx = p.kx; a.ky = p.ky; a.kmap = p.full_k ? nullptr : p.kmap.as<int>();
        a.U = p.U.as<T>(); a.ldu = p.L; a.V = p.V.as<T>(); a.ldv = p.K; a.coef = sig.as<double>();
        a.grp_off = go.as<int>(); a.grp_idx = gi.as<int>(); a.ngroups = ng;
        a.w = wdiv; a.out = out_dev; a.ldout = p.nx; a.out_stride = nxy;
        diagsums_direct<T>(a, p.st);
    }
    if (add_rest)
        rest_group<T>(p.img.as<T>(), wdiv, out_dev, ng, nxy, nxy, out_dev + (int64_t)ng * nxy, p.st);
    SSA_CUDA(cudaStreamSynchronize(p.st));
}

// Band plans: the reconstruction of the global image from the ranks' bands.  Each
// rank forms the diagonal-averaging NUMERATORS of its sub-image (its own window positions only),
// places them at the band's global columns and the ranks sum them (one all-reduce per output; the
// (Ly−1)-column halos overlap with the next band); the global hit counts are the sum of the bands'
// (𝕎 counts (ℓ, κ) pairs and the κ are partitioned), so Alg. 4's division then gives the global
// X̃_g on every rank.  With want_img the global image (0 outside 𝔑) is assembled into out[ng]
// (owned columns only: a rank contributes [y0, y1), the last one also its halo).  w_global (int32,
// nx x ny_global) receives the global hit counts when non-null.
template <typename T>
static void band_reconstruct(PlanImpl &p, const int32_t *off, const int32_t *idx, int ng, bool want_img, T *out,
                             int32_t *w_global) {
    const int64_t nxy = (int64_t)p.nx * p.ny, nxg = (int64_t)p.nx * p.ny_global;
    const unsigned grid = (unsigned)std::min<int64_t>(cdiv(nxg * std::max(ng, 1), 256), 16 * num_sms());
    auto allreduce = [&](T *buf, int64_t n) {
        if (p.comm.allreduce_sum(p.comm.user, buf, n, p.dt, p.st) != 0)
            throw Error(SSA_ERR_COMM, "allreduce of the band reconstructions failed");
    };
    DevBuf ones, num, wl, wg;
    ones.alloc(sizeof(int32_t) * nxy, p.st);
    {
        std::vector<int32_t> h(nxy, 1);
        SSA_CUDA(cudaMemcpyAsync(ones.p, h.data(), sizeof(int32_t) * nxy, cudaMemcpyHostToDevice, p.st));
        if (ng > 0) {
            num.alloc(sizeof(T) * nxy * ng, p.st);
            reconstruct_impl<T>(p, off, idx, ng, 0, num.as<T>(), ones.as<int32_t>());   // raw numerators
        }
        SSA_CUDA(cudaStreamSynchronize(p.st));
    }
    if (ng > 0) {
        place_band_kernel<T><<<grid, 256, 0, p.st>>>(num.as<T>(), p.nx, p.ny, p.ny, out, (int)p.ny_global, p.band_y0, ng);
        after_launch("place_band");
        allreduce(out, nxg * ng);
    }
    wl.alloc(sizeof(T) * nxy, p.st);
    wg.alloc(sizeof(T) * nxg, p.st);
    int_to_T_kernel<T><<<grid, 256, 0, p.st>>>(p.weights.as<int32_t>(), nxy, wl.as<T>());
    after_launch("int_to_T");
    place_band_kernel<T><<<grid, 256, 0, p.st>>>(wl.as<T>(), p.nx, p.ny, p.ny, wg.as<T>(), (int)p.ny_global, p.band_y0, 1);
    after_launch("place_band");
    allreduce(wg.as<T>(), nxg);   // exact: integer counts < 2^24
    if (ng > 0) {
        divide_weights_kernel<T><<<grid, 256, 0, p.st>>>(out, wg.as<T>(), nxg, ng);
        after_launch("divide_weights");
    }
    if (want_img) {
        const bool last = p.band_y1 + p.ly - 1 == p.ny_global;
        place_band_kernel<T><<<grid, 256, 0, p.st>>>(p.img.as<T>(), p.nx, p.ny, last ? p.ny : p.band_y1 - p.band_y0,
                                                     out + nxg * ng, (int)p.ny_global, p.band_y0, 1);
        after_launch("place_band");
        allreduce(out + nxg * ng, nxg);
    }
    if (w_global) box_ones_to_int<T>(wg.as<T>(), nxg, w_global, p.st);
    SSA_CUDA(cudaStreamSynchronize(p.st));
}

}  // namespace ssa

// =====================================================================================
using namespace ssa;

struct ssa_plan_s {
    PlanImpl impl;
};

namespace ssa {
PlanImpl &ssa_plan_impl(ssa_plan p) {
    if (p->impl.broken) throw Error(SSA_ERR_CUDA, "plan is in a failed state (earlier CUDA/comm error); destroy it");
    return p->impl;
}
}  // namespace ssa

#define SSA_API_BEGIN try {
#define SSA_API_END                                                          \
    }                                                                        \
    catch (const Error &e) {                                                 \
        g_err = e.what();                                                    \
        if (p && (e.code == SSA_ERR_CUDA || e.code == SSA_ERR_COMM)) p->impl.broken = true; \
        return e.code;                                                       \
    }                                                                        \
    catch (const std::exception &e) {                                        \
        g_err = e.what();                                                    \
        return SSA_ERR_ARG;                                                  \
    }

static ssa_status check_plan(ssa_plan p) {
    if (!p) { g_err = "null plan"; return SSA_ERR_ARG; }
    if (p->impl.broken) { g_err = "plan is in a failed state (earlier CUDA/comm error); destroy it"; return SSA_ERR_CUDA; }
    return SSA_OK;
}

extern "C" {

ssa_status ssa_release_workspace(void) {
    ssa::release_workspace();
    if (cudaDeviceSynchronize() != cudaSuccess) cudaGetLastError();   // the frees are stream-ordered
    return SSA_OK;
}

const char *ssa_last_error(void) { return g_err.c_str(); }
const char *ssa_version(void) { return "ssa_b200 0.1 (sm_100a)"; }
int64_t ssa_launch_count(int reset) {
    const int64_t n = g_launches;
    if (reset) g_launches = 0;
    return n;
}

ssa_status ssa_plan_create(const ssa_array *x, const ssa_window *w, const uint8_t *mask, const ssa_opts *opts,
                           ssa_plan *out) {
    ssa_plan p = nullptr;
    SSA_API_BEGIN
    if (!x || !w || !out || !x->data) throw Error(SSA_ERR_ARG, "null argument");
    *out = nullptr;
    if (x->dtype != SSA_F32 && x->dtype != SSA_F64) throw Error(SSA_ERR_ARG, "dtype must be SSA_F32 or SSA_F64");
    if (x->nx < 1 || x->ny < 1 || x->nx > (1 << 24) || x->ny > (1 << 24) || x->nx * x->ny > ((int64_t)1 << 31))
        throw Error(SSA_ERR_ARG, "array size out of range");
    if (x->ld != 0 && x->ld < x->nx) throw Error(SSA_ERR_ARG, "ld < nx");
    // window bounds
    if (w->lx < 1 || w->ly < 1 || w->lx > x->nx || w->ly > x->ny || (int64_t)w->lx * w->ly <= 1 ||
        (int64_t)w->lx * w->ly >= x->nx * x->ny)
        throw Error(SSA_ERR_WINDOW, "window must satisfy 1<=Lx<=Nx, 1<=Ly<=Ny, 1<Lx*Ly<Nx*Ny");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        throw Error(SSA_ERR_CUDA, "no CUDA device: libssa_b200 has no CPU fallback");
    }
    p = new ssa_plan_s();
    PlanImpl &P = p->impl;
    P.nx = (int)x->nx; P.ny = (int)x->ny; P.lx = w->lx; P.ly = w->ly;
    P.kx = P.nx - P.lx + 1; P.ky = P.ny - P.ly + 1;
    ssa_opts o{};
    if (opts) o = *opts;
    // arithmetic type of the plan: the input's dtype unless opts.precision asks for another
    // (the input is cast once at plan creation)
    if (o.precision < 0 || o.precision > 2) throw Error(SSA_ERR_ARG, "precision must be 0 (input), 1 (fp32) or 2 (fp64)");
    P.dt = o.precision == 0 ? x->dtype : (o.precision == 1 ? SSA_F32 : SSA_F64);
    P.st = (cudaStream_t)o.stream;
    P.path = o.path;
    P.block_k = o.block_k > 0 ? o.block_k : (P.dt == SSA_F64 ? 16 : 32);
    if (o.svd_method != SSA_SVD_LANCZOS && o.svd_method != SSA_SVD_EIGEN) throw Error(SSA_ERR_ARG, "bad svd_method");
    P.svd_method = o.svd_method;
    P.tol = o.tol; P.max_products = o.max_products; P.seed = o.seed ? o.seed : 0x1309505000ull;
    if (o.comm && o.comm->world > 1) {
        // window-position band partition: x is this rank's sub-image, the global image
        // columns [band_y0, band_y1 + Ly − 1) (its origin band plus the (Ly−1)-column halo), so the
        // sub-image's own 𝔎 is exactly the band of the global 𝔎 (eq. P:3004-3005 only looks inside
        // the window span of each origin)
        P.comm = *o.comm; P.has_comm = true;
        P.band_y0 = o.band_y0; P.band_y1 = o.band_y1;
        P.ny_global = o.ny_global;
        if (P.band_y0 < 0 || P.band_y0 >= P.band_y1 || P.band_y1 - P.band_y0 != P.ky ||
            P.ny_global < P.band_y1 + P.ly - 1)
            throw Error(SSA_ERR_ARG, "band plan: x must be the global columns [band_y0, band_y1 + Ly - 1) "
                                     "and ny_global >= band_y1 + Ly - 1");
    }
    // 𝔏 (window shape) on the host: box index -> lex index
    P.lmap_host.assign((size_t)P.lx * P.ly, -1);
    int64_t L = 0;
    for (int64_t t = 0; t < (int64_t)P.lx * P.ly; ++t)
        if (!w->wmask || w->wmask[t]) P.lmap_host[t] = (int32_t)L++;
    if (L == 0) throw Error(SSA_ERR_WINDOW, "empty window shape");
    P.L = L;
    P.full_window = (L == (int64_t)P.lx * P.ly);
    try {
        if (P.dt == SSA_F64) build_plan<double>(P, x, mask);
        else build_plan<float>(P, x, mask);
    } catch (...) {
        delete p;
        throw;
    }
    *out = p;
    return SSA_OK;
    SSA_API_END
}

void ssa_plan_destroy(ssa_plan p) {
    if (!p) return;
    if (p->impl.st) cudaStreamSynchronize(p->impl.st);
    delete p;
}

ssa_status ssa_plan_info(ssa_plan p, ssa_plan_info_t *info) {
    if (ssa_status s = check_plan(p)) return s;
    if (!info) { g_err = "null info"; return SSA_ERR_ARG; }
    const PlanImpl &P = p->impl;
    info->nx = P.nx; info->ny = P.ny; info->lx = P.lx; info->ly = P.ly; info->kx = P.kx; info->ky = P.ky;
    info->L = P.L; info->K = P.K; info->n_valid = P.n_valid; info->n_excluded = P.n_excluded;
    info->path = P.path; info->dtype = P.dt;
    info->full_window = P.full_window; info->full_kshape = P.full_k;
    info->path_xv = P.path_xv; info->path_xtu = P.path_xtu;
    return SSA_OK;
}

static void copy_out(PlanImpl &P, void *dst, const void *src, size_t bytes, int on_device) {
    SSA_CUDA(cudaMemcpyAsync(dst, src, bytes, on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, P.st));
    SSA_CUDA(cudaStreamSynchronize(P.st));
}

ssa_status ssa_get_weights(ssa_plan p, int32_t *w, int on_device) {
    if (ssa_status s = check_plan(p)) return s;
    SSA_API_BEGIN
    if (!w) throw Error(SSA_ERR_ARG, "null output");
    copy_out(p->impl, w, p->impl.weights.p, sizeof(int32_t) * p->impl.nx * p->impl.ny, on_device);
    return SSA_OK;
    SSA_API_END
}

ssa_status ssa_get_kmask(ssa_plan p, uint8_t *km, int on_device) {
    if (ssa_status s = check_plan(p)) return s;
    SSA_API_BEGIN
    if (!km) throw Error(SSA_ERR_ARG, "null output");
    copy_out(p->impl, km, p->impl.kmask.p, (size_t)p->impl.kx * p->impl.ky, on_device);
    return SSA_OK;
    SSA_API_END
}

ssa_status ssa_matmul(ssa_plan p, int transpose, const void *in, int64_t ldin, void *out, int64_t ldout, int64_t k,
                      int on_device) {
    if (ssa_status s = check_plan(p)) return s;
    SSA_API_BEGIN
    PlanImpl &P = p->impl;
    if (!in || !out || k < 1 || k > (1 << 20)) throw Error(SSA_ERR_ARG, "bad matmul arguments");
    const int64_t nin = transpose ? P.L : P.K, nout = transpose ? P.K : P.L;
    if (ldin == 0) ldin = nin;
    if (ldout == 0) ldout = nout;
    if (ldin < nin || ldout < nout) throw Error(SSA_ERR_ARG, "leading dimension too small");
    const size_t es = P.elem();
    const void *din = in;
    void *dout = out;
    DevBuf bi, bo;
    if (!on_device) {
        bi.alloc(es * ldin * k, P.st);
        bo.alloc(es * ldout * k, P.st);
        SSA_CUDA(cudaMemcpyAsync(bi.p, in, es * ldin * k, cudaMemcpyHostToDevice, P.st));
        din = bi.p; dout = bo.p;
    }
    if (P.dt == SSA_F64) {
        if (transpose) op_xtu<double>(P, (const double *)din, ldin, (double *)dout, ldout, (int)k);
        else op_xv<double>(P, (const double *)din, ldin, (double *)dout, ldout, (int)k);
    } else {
        if (transpose) op_xtu<float>(P, (const float *)din, ldin, (float *)dout, ldout, (int)k);
        else op_xv<float>(P, (const float *)din, ldin, (float *)dout, ldout, (int)k);
    }
    if (!on_device) {
        SSA_CUDA(cudaMemcpyAsync(out, bo.p, es * ldout * k, cudaMemcpyDeviceToHost, P.st));
        SSA_CUDA(cudaStreamSynchronize(P.st));
    }
    return SSA_OK;
    SSA_API_END
}

ssa_status ssa_decompose(ssa_plan p, int32_t r, ssa_decomp_info *info) {
    if (ssa_status s = check_plan(p)) return s;
    SSA_API_BEGIN
    PlanImpl &P = p->impl;
    if (r < 1 || r > std::min(P.L, P.K)) throw Error(SSA_ERR_RANK, "r must satisfy 1 <= r <= min(L, K)");
    ssa_decomp_info tmp{};
    ssa_decomp_info *inf = info ? info : &tmp;
    std::memset(inf, 0, sizeof(*inf));
    const auto t0 = std::chrono::steady_clock::now();
    ssa_status st = SSA_OK;
    try {
        if (P.svd_method == SSA_SVD_EIGEN) {
            if (P.dt == SSA_F64) decompose_eigen<double>(P, r, inf);
            else decompose_eigen<float>(P, r, inf);
        } else if (P.dt == SSA_F64) {
            decompose<double>(P, r, inf);
        } else {
            decompose<float>(P, r, inf);
        }
    } catch (const Error &e) {
        if (e.code != SSA_ERR_NOT_CONVERGED) throw;
        g_err = e.what();
        st = e.code;
    }
    inf->ms_total = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    P.last_info = *inf;
    return st;
    SSA_API_END
}

ssa_status ssa_get_rank(ssa_plan p, int32_t *r) {
    if (ssa_status s = check_plan(p)) return s;
    if (!r) { g_err = "null output"; return SSA_ERR_ARG; }
    *r = p->impl.r;
    return SSA_OK;
}

ssa_status ssa_get_sigma(ssa_plan p, double *sigma) {
    if (ssa_status s = check_plan(p)) return s;
    if (!sigma) { g_err = "null output"; return SSA_ERR_ARG; }
    if (p->impl.r == 0) { g_err = "no decomposition"; return SSA_ERR_STATE; }
    std::memcpy(sigma, p->impl.sigma.data(), sizeof(double) * p->impl.r);
    return SSA_OK;
}

ssa_status ssa_get_residuals(ssa_plan p, double *res) {
    if (ssa_status s = check_plan(p)) return s;
    if (!res) { g_err = "null output"; return SSA_ERR_ARG; }
    if (p->impl.r == 0) { g_err = "no decomposition"; return SSA_ERR_STATE; }
    const PlanImpl &P = p->impl;
    for (int i = 0; i < P.r; ++i) res[i] = i < (int)P.residuals.size() ? P.residuals[i] : NAN;
    return SSA_OK;
}

ssa_status ssa_get_u(ssa_plan p, void *U, int on_device) {
    if (ssa_status s = check_plan(p)) return s;
    SSA_API_BEGIN
    PlanImpl &P = p->impl;
    if (P.r == 0) throw Error(SSA_ERR_STATE, "no decomposition");
    if (!U) throw Error(SSA_ERR_ARG, "null output");
    copy_out(P, U, P.U.p, P.elem() * P.L * P.r, on_device);
    return SSA_OK;
    SSA_API_END
}

ssa_status ssa_get_v(ssa_plan p, void *V, int on_device) {
    if (ssa_status s = check_plan(p)) return s;
    SSA_API_BEGIN
    PlanImpl &P = p->impl;
    if (P.r == 0) throw Error(SSA_ERR_STATE, "no decomposition");
    if (!V) throw Error(SSA_ERR_ARG, "null output");
    if (P.dt == SSA_F64) get_v<double>(P); else get_v<float>(P);
    copy_out(P, V, P.V.p, P.elem() * P.K * P.r, on_device);
    return SSA_OK;
    SSA_API_END
}

ssa_status ssa_set_triples(ssa_plan p, int32_t r, const double *sigma, const void *U, const void *V, int on_device) {
    if (ssa_status s = check_plan(p)) return s;
    SSA_API_BEGIN
    PlanImpl &P = p->impl;
    if (r < 1 || r > std::min(P.L, P.K)) throw Error(SSA_ERR_RANK, "bad r");
    if (!sigma || !U) throw Error(SSA_ERR_ARG, "null sigma/U");
    const size_t es = P.elem();
    P.U.alloc(es * P.L * r, P.st);
    SSA_CUDA(cudaMemcpyAsync(P.U.p, U, es * P.L * r, on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, P.st));
    P.sigma.assign(sigma, sigma + r);
    P.r = r;
    P.v_valid = false;
    P.v_have.clear();
    if (V) {
        P.V.alloc(es * P.K * r, P.st);
        SSA_CUDA(cudaMemcpyAsync(P.V.p, V, es * P.K * r, on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, P.st));
        P.v_valid = true;
    }
    SSA_CUDA(cudaStreamSynchronize(P.st));
    return SSA_OK;
    SSA_API_END
}

// Group validation.  A group index beyond the computed triples continues the decomposition
// automatically ("if 10 eigentriples were calculated while decomposing, then the user could still
// perform reconstruction by the first 15 components, since the decomposition will be automatically
// continued"): decompose(max index + 1), warm-started from the stored eigenvectors.
static void check_groups(PlanImpl &P, const int32_t *off, const int32_t *idx, int32_t ng) {
    if (ng < 0 || (ng > 0 && (!off || !idx))) throw Error(SSA_ERR_ARG, "bad group arrays");
    if (ng == 0) return;
    if (off[0] != 0) throw Error(SSA_ERR_ARG, "grp_off[0] must be 0");
    for (int g = 0; g < ng; ++g)
        if (off[g + 1] < off[g]) throw Error(SSA_ERR_ARG, "grp_off must be non-decreasing");
    int need = 0;
    for (int t = 0; t < off[ng]; ++t) {
        if (idx[t] < 0) throw Error(SSA_ERR_RANK, "negative group index");
        need = std::max(need, idx[t] + 1);
    }
    if (need > P.r) {
        if (need > std::min(P.L, P.K)) throw Error(SSA_ERR_RANK, "group index >= min(L, K)");
        ssa_decomp_info inf{};
        if (P.dt == SSA_F64) decompose<double>(P, need, &inf);
        else decompose<float>(P, need, &inf);
        P.last_info = inf;
    }
}

ssa_status ssa_reconstruct(ssa_plan p, const int32_t *off, const int32_t *idx, int32_t ng, int add_rest, void *out,
                           int on_device) {
    if (ssa_status s = check_plan(p)) return s;
    SSA_API_BEGIN
    PlanImpl &P = p->impl;
    if (P.r == 0) throw Error(SSA_ERR_STATE, "reconstruct before decompose");
    if (!out) throw Error(SSA_ERR_ARG, "null output");
    check_groups(P, off, idx, ng);
    const bool band = P.has_comm && P.comm.world > 1;
    const int64_t nxy = (int64_t)P.nx * (band ? P.ny_global : P.ny);   // band plans return the global image
    const int nout = ng + (add_rest ? 1 : 0);
    const int32_t zero_off = 0;
    if (ng == 0) off = &zero_off;
    DevBuf tmp;
    void *dout = out;
    if (!on_device) {
        tmp.alloc(P.elem() * nxy * std::max(nout, 1), P.st);
        dout = tmp.p;
    }
    if (band) {
        DevBuf wgi;
        if (add_rest) wgi.alloc(sizeof(int32_t) * nxy, P.st);
        if (P.dt == SSA_F64) {
            band_reconstruct<double>(P, off, idx, ng, add_rest, (double *)dout, add_rest ? wgi.as<int32_t>() : nullptr);
            if (add_rest) {   // rest = image − Σ_g X̃_g on the global 𝔑′ (the image was assembled into out[ng])
                DevBuf xg;
                xg.alloc(sizeof(double) * nxy, P.st);
                SSA_CUDA(cudaMemcpyAsync(xg.p, (double *)dout + nxy * ng, sizeof(double) * nxy, cudaMemcpyDeviceToDevice, P.st));
                rest_group<double>(xg.as<double>(), wgi.as<int32_t>(), (double *)dout, ng, nxy, nxy, (double *)dout + nxy * ng, P.st);
            }
        } else {
            band_reconstruct<float>(P, off, idx, ng, add_rest, (float *)dout, add_rest ? wgi.as<int32_t>() : nullptr);
            if (add_rest) {
                DevBuf xg;
                xg.alloc(sizeof(float) * nxy, P.st);
                SSA_CUDA(cudaMemcpyAsync(xg.p, (float *)dout + nxy * ng, sizeof(float) * nxy, cudaMemcpyDeviceToDevice, P.st));
                rest_group<float>(xg.as<float>(), wgi.as<int32_t>(), (float *)dout, ng, nxy, nxy, (float *)dout + nxy * ng, P.st);
            }
        }
        SSA_CUDA(cudaStreamSynchronize(P.st));
    } else if (P.dt == SSA_F64) {
        reconstruct_impl<double>(P, off, idx, ng, add_rest, (double *)dout);
    } else {
        reconstruct_impl<float>(P, off, idx, ng, add_rest, (float *)dout);
    }
    if (!on_device) copy_out(P, out, dout, P.elem() * nxy * nout, 0);
    return SSA_OK;
    SSA_API_END
}

ssa_status ssa_wcor(ssa_plan p, const int32_t *off, const int32_t *idx, int32_t ng, double *rho, double *contrib) {
    if (ssa_status s = check_plan(p)) return s;
    SSA_API_BEGIN
    PlanImpl &P = p->impl;
    if (P.r == 0) throw Error(SSA_ERR_STATE, "wcor before decompose");
    if (!rho || ng < 1 || ng > 63) throw Error(SSA_ERR_ARG, "wcor: 1..63 groups");
    check_groups(P, off, idx, ng);
    const bool band = P.has_comm && P.comm.world > 1;
    const int64_t nxy = (int64_t)P.nx * (band ? P.ny_global : P.ny);
    // columns: the ng reconstructions, then the image itself (its weighted norm is the denominator
    // of the contributions); each scaled by sqrt(w_n) so that one Gram gives (Y, Z)_w.
    // Band plans work on the assembled global reconstructions, image and hit counts.
    const int nc = ng + 1;
    DevBuf rec, wgl;
    rec.alloc(P.elem() * nxy * nc, P.st);
    const int32_t *wts = P.weights.as<int32_t>();
    if (band) {
        wgl.alloc(sizeof(int32_t) * nxy, P.st);
        wts = wgl.as<int32_t>();
    }
    std::vector<double> G((size_t)nc * nc);
    double *Gd = small_dev(P, 64 * 64);
    if (P.dt == SSA_F64) {
        if (band) {
            band_reconstruct<double>(P, off, idx, ng, true, rec.as<double>(), wgl.as<int32_t>());
        } else {
            reconstruct_impl<double>(P, off, idx, ng, 0, rec.as<double>());
            SSA_CUDA(cudaMemcpyAsync(rec.as<double>() + nxy * ng, P.img.p, sizeof(double) * nxy, cudaMemcpyDeviceToDevice, P.st));
        }
        weighted_sqrt_kernel<double><<<(unsigned)std::min<int64_t>(cdiv(nxy * nc, 256), 16 * num_sms()), 256, 0, P.st>>>(
            rec.as<double>(), wts, nxy, nc);
        after_launch("weighted_sqrt");
        gram_tn<double>(nxy, rec.as<double>(), nxy, nc, rec.as<double>(), nxy, nc, Gd, P.ws_gram.as<double>(), P.ws_gram.bytes, P.st);
    } else {
        if (band) {
            band_reconstruct<float>(P, off, idx, ng, true, rec.as<float>(), wgl.as<int32_t>());
        } else {
            reconstruct_impl<float>(P, off, idx, ng, 0, rec.as<float>());
            SSA_CUDA(cudaMemcpyAsync(rec.as<float>() + nxy * ng, P.img.p, sizeof(float) * nxy, cudaMemcpyDeviceToDevice, P.st));
        }
        weighted_sqrt_kernel<float><<<(unsigned)std::min<int64_t>(cdiv(nxy * nc, 256), 16 * num_sms()), 256, 0, P.st>>>(
            rec.as<float>(), wts, nxy, nc);
        after_launch("weighted_sqrt");
        gram_tn<float>(nxy, rec.as<float>(), nxy, nc, rec.as<float>(), nxy, nc, Gd, P.ws_gram.as<double>(), P.ws_gram.bytes, P.st);
    }
    SSA_CUDA(cudaMemcpyAsync(G.data(), Gd, sizeof(double) * nc * nc, cudaMemcpyDeviceToHost, P.st));
    SSA_CUDA(cudaStreamSynchronize(P.st));
    for (int b = 0; b < ng; ++b)
        for (int a = 0; a < ng; ++a) {
            const double d = std::sqrt(G[a + (size_t)nc * a] * G[b + (size_t)nc * b]);
            rho[a + (size_t)ng * b] = d > 0 ? G[a + (size_t)nc * b] / d : 0.0;
        }
    if (contrib) {
        const double xx = G[ng + (size_t)nc * ng];
        for (int g = 0; g < ng; ++g) contrib[g] = xx > 0 ? G[g + (size_t)nc * g] / xx : 0.0;
    }
    return SSA_OK;
    SSA_API_END
}

}  // extern "C"
