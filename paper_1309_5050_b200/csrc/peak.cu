// Measured tensor-core peak for the roofline of the tcgen05 product and Gram kernels (VERDICT r1:
// "commit a measured tcgen05 kind::tf32 peak"): every CTA (one per SM) issues a long run of
// back-to-back `tcgen05.mma.cta_group::1.kind::tf32` M = 128, N = 256, K = 8 from one elected
// thread, operands resident in shared memory (128-B swizzled K-major tiles, contents irrelevant
// for the rate), alternating between two TMEM accumulators; one commit + mbarrier wait at the end.
// The rate is 2·128·256·8 flops per MMA over the kernel's device time.
#include <cstdlib>

#include "common.h"
#include "tc_common.h"

namespace ssa {

// N (accumulator width) and TS (A operand from tensor memory, as the Gram / update kernels issue it)
// are measurement variants: SSA_MMA_N = 64 / 128 / 256 (default 256), SSA_MMA_TS = 1
template <int N, bool TS>
__global__ void __launch_bounds__(128, 1) mma_peak_kernel(int iters, int *sink) {
    using namespace tc;
    extern __shared__ unsigned char smem_raw[];
    unsigned char *smem = smem_align1024(smem_raw);
    uint64_t *bar = reinterpret_cast<uint64_t *>(smem + 48 * 1024);
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bar + 1);
    const int warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < 48 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t *>(smem)[i] = 0;
    if (threadIdx.x == 0) mbar_init(smem_u32(bar), 1);
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)), "n"(512)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    fence_proxy_async();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    if (threadIdx.x == 32) {
        const uint64_t adesc = make_desc(smem_u32(smem));               // A: 128 rows x 128 B
        const uint64_t bdesc = make_desc(smem_u32(smem + 16 * 1024));   // B: 256 rows x 128 B
        constexpr uint32_t idesc = make_idesc(128, N);
        if constexpr (TS) {
            // A (128 lanes x 8 tf32) from tensor-memory columns [256, 264); accumulators alternate in [0, 256)
            for (int i = 0; i < iters; ++i)
                mma_tf32_ts(tmem + (uint32_t)((i & 1) * (N <= 128 ? N : 0)), tmem + 256u, bdesc, idesc, i > 1);
        } else {
            for (int i = 0; i < iters; ++i) mma_tf32(tmem + (uint32_t)((i & 1) * 256), adesc, bdesc, idesc, i > 1);
        }
        mma_commit(smem_u32(bar));
    }
    __syncwarp();
    if (warp == 1) mbar_wait(smem_u32(bar), 0);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 0) {
        float v[32];
        tmem_ld32(tmem, v);   // keep the MMAs observable (warp 0: lanes 0-31)
        if (v[0] == 12345.f) sink[0] = 1;
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(512) : "memory");
    }
}

}  // namespace ssa

extern "C" ssa_status ssa_bench_mma(int32_t iters, int32_t ctas, double *ms, double *tflops) {
    using namespace ssa;
    try {
        if (iters < 1 || ctas < 0) throw Error(SSA_ERR_ARG, "ssa_bench_mma: bad arguments");
        if (ctas == 0) ctas = num_sms();
        DevBuf sink;
        sink.alloc(16, nullptr);
        const size_t smem = 48 * 1024 + 1024 + 64;
        static const int nvar = [] { const char *e = std::getenv("SSA_MMA_N"); return e ? std::atoi(e) : 256; }();
        static const int ts = [] { const char *e = std::getenv("SSA_MMA_TS"); return e ? std::atoi(e) : 0; }();
        auto kern = mma_peak_kernel<256, false>;
        if (nvar == 64) kern = ts ? mma_peak_kernel<64, true> : mma_peak_kernel<64, false>;
        else if (nvar == 128) kern = ts ? mma_peak_kernel<128, true> : mma_peak_kernel<128, false>;
        else if (ts) kern = mma_peak_kernel<256, true>;
        const int nmma = (nvar == 64 || nvar == 128) ? nvar : 256;
        set_max_smem(kern);
        kern<<<ctas, 128, smem>>>(8, sink.as<int>());   // warm-up
        after_launch("mma_peak");
        cudaEvent_t e0, e1;
        SSA_CUDA(cudaEventCreate(&e0));
        SSA_CUDA(cudaEventCreate(&e1));
        SSA_CUDA(cudaEventRecord(e0, nullptr));
        kern<<<ctas, 128, smem>>>(iters, sink.as<int>());
        after_launch("mma_peak");
        SSA_CUDA(cudaEventRecord(e1, nullptr));
        SSA_CUDA(cudaEventSynchronize(e1));
        float t = 0.f;
        SSA_CUDA(cudaEventElapsedTime(&t, e0, e1));
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        if (ms) *ms = t;
        if (tflops) *tflops = 2.0 * 128 * nmma * 8 * (double)iters * ctas / (t * 1e-3) / 1e12;
        return SSA_OK;
    } catch (const Error &e) {
        ssa_set_error(e.what());
        return e.code;
    }
}
