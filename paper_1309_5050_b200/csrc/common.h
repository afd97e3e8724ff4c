// Internal helpers shared by the CUDA translation units of libssa_b200.so.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/ssa_b200.h"

namespace ssa {

// Error carried from deep inside the library to the ABI boundary, where it is
// turned into an ssa_status plus the thread-local message (no exception ever
// crosses the C ABI).
struct Error : std::runtime_error {
    ssa_status code;
    Error(ssa_status c, const std::string &m) : std::runtime_error(m), code(c) {}
};

#define SSA_CUDA(call)                                                                   \
    do {                                                                                 \
        cudaError_t e_ = (call);                                                         \
        if (e_ != cudaSuccess)                                                           \
            throw ::ssa::Error(e_ == cudaErrorMemoryAllocation ? SSA_ERR_OOM : SSA_ERR_CUDA, \
                               std::string(#call) + ": " + cudaGetErrorString(e_));      \
    } while (0)

#define SSA_REQUIRE(cond, code, msg)                      \
    do {                                                  \
        if (!(cond)) throw ::ssa::Error((code), (msg));   \
    } while (0)

// Count of kernels launched through this library on the calling thread.
void count_launch(int n = 1);
// Check the last launch and count it.
void after_launch(const char *what);

// Owning device buffer from the stream-ordered pool allocator (cudaMallocAsync on the
// plan's stream; the device's default pool keeps freed blocks cached, so creating and
// destroying plans does not pay cudaMalloc/cudaFree each time).
void pool_init();
// Large blocks (>= 8 MB) are kept, when freed, in a per-host-thread cache keyed by their exact size and
// handed back to the next allocation of that size (any stream: the new stream waits on an event recorded
// at the free).  A plan's large buffers have the same sizes in every plan of a shape, so steady-state plans
// never return to the pool allocator: freed to the pool, the multi-GB buffers of plan, decomposition and
// reconstruction were re-carved differently from step to step and the pool had to map new memory now and
// then (host stalls of 15-700 ms inside ssa_reconstruct / ssa_decompose, gpurun r1-r4).  The cache holds
// at most 64 GB (oldest blocks go back to the pool first); ssa_release_workspace empties it.
void *big_take(size_t n, cudaStream_t st);
bool big_give(void *p, size_t n, cudaStream_t st);
void big_release_all();
constexpr size_t kBigBlock = (size_t)8 << 20;
struct DevBuf {
    void *p = nullptr;
    size_t bytes = 0;
    cudaStream_t s = nullptr;
    DevBuf() = default;
    DevBuf(const DevBuf &) = delete;
    DevBuf &operator=(const DevBuf &) = delete;
    DevBuf(DevBuf &&o) noexcept { *this = std::move(o); }
    DevBuf &operator=(DevBuf &&o) noexcept {
        if (this != &o) { release(); p = o.p; bytes = o.bytes; s = o.s; o.p = nullptr; o.bytes = 0; }
        return *this;
    }
    ~DevBuf() { release(); }
    void alloc(size_t n, cudaStream_t st) {
        if (n <= bytes && p) return;
        release();
        pool_init();
        s = st;
        if (n >= kBigBlock) p = big_take(n, st);
        if (!p) SSA_CUDA(cudaMallocAsync(&p, n ? n : 16, st));
        bytes = n;
    }
    void release() {
        if (p) {
            if (bytes < kBigBlock || !big_give(p, bytes, s)) cudaFreeAsync(p, s);
            p = nullptr; bytes = 0;
        }
    }
    template <class T> T *as() const { return static_cast<T *>(p); }
};

inline int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }
inline int64_t rup(int64_t a, int64_t b) { return cdiv(a, b) * b; }

int num_sms();
// Raise a kernel's dynamic shared-memory cap to the sm_100 maximum once per function (the
// attribute call costs host time on every launch otherwise; the launch's own size still decides
// the carve-out).
void set_max_smem_impl(const void *fn);
template <typename F> inline void set_max_smem(F *fn) { set_max_smem_impl(reinterpret_cast<const void *>(fn)); }
// set the thread-local message returned by ssa_last_error()
void ssa_set_error(const std::string &msg);

}  // namespace ssa
