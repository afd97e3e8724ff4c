// Plan-time kernels: shape ingestion, 𝔎 selection,
// compaction maps, rectangular weights, and small elementwise epilogues.
#include <mutex>
#include <set>

#include "common.h"
#include "kernels.h"

namespace ssa {

void set_max_smem_impl(const void *fn) {
    static std::mutex mu;
    static std::set<const void *> done;
    std::lock_guard<std::mutex> lk(mu);
    if (done.count(fn)) return;
    // opt-in per-block maximum minus the kernel's static shared memory
    static int optin = [] {
        int dev = 0, v = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
        return v;
    }();
    cudaFuncAttributes fa{};
    SSA_CUDA(cudaFuncGetAttributes(&fa, fn));
    SSA_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, optin - (int)fa.sharedSizeBytes));
    done.insert(fn);
}

// a1: 𝔑 = {finite cells} ∩ mask; cells outside 𝔑 are set to 0
// (they never enter 𝒯(𝕏) because every κ ∈ 𝔎 keeps its window inside 𝔑).
template <typename T>
__global__ void prep_image_kernel(const T *src, int64_t ld_src, int nx, int ny, const uint8_t *mask,
                                  T *dst, uint8_t *nmask) {
    const int64_t n = (int64_t)nx * ny;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = t % nx, j = t / nx;
        const T v = src[i + ld_src * j];
        const bool in = isfinite((double)v) && (mask == nullptr || mask[t] != 0);
        dst[t] = in ? v : T(0);
        nmask[t] = in ? 1 : 0;
    }
}

template <typename T>
void prep_image(const T *src, int64_t ld_src, int nx, int ny, const uint8_t *mask, T *dst, uint8_t *nmask,
                cudaStream_t st) {
    const int64_t n = (int64_t)nx * ny;
    prep_image_kernel<T><<<(unsigned)std::min<int64_t>(cdiv(n, 256), 16 * num_sms()), 256, 0, st>>>(
        src, ld_src, nx, ny, mask, dst, nmask);
    after_launch("prep_image");
}
template void prep_image<float>(const float *, int64_t, int, int, const uint8_t *, float *, uint8_t *, cudaStream_t);
template void prep_image<double>(const double *, int64_t, int, int, const uint8_t *, double *, uint8_t *, cudaStream_t);

// a2 (Alg. 6 step 3): 𝔎 = {κ : v_κ = |𝔏|}, v = 𝒯ᵀ(I^𝔑)·1_𝔏 (exact integers).
template <typename T>
__global__ void threshold_eq_kernel(const T *c, int64_t n, double value, uint8_t *out) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x)
        out[t] = ((double)c[t] == value) ? 1 : 0;
}
template <typename T>
void threshold_eq(const T *counts, int64_t n, double value, uint8_t *out, cudaStream_t st) {
    threshold_eq_kernel<T><<<(unsigned)std::min<int64_t>(cdiv(n, 256), 16 * num_sms()), 256, 0, st>>>(
        counts, n, value, out);
    after_launch("threshold_eq");
}
template void threshold_eq<float>(const float *, int64_t, double, uint8_t *, cudaStream_t);
template void threshold_eq<double>(const double *, int64_t, double, uint8_t *, cudaStream_t);

template <typename T>
__global__ void to_int_kernel(const T *s, int64_t n, int32_t *d) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x)
        d[t] = (int32_t)llrint((double)s[t]);
}
template <typename T>
void box_ones_to_int(const T *src, int64_t n, int32_t *dst, cudaStream_t st) {
    to_int_kernel<T><<<(unsigned)std::min<int64_t>(cdiv(n, 256), 16 * num_sms()), 256, 0, st>>>(src, n, dst);
    after_launch("to_int");
}
template void box_ones_to_int<float>(const float *, int64_t, int32_t *, cudaStream_t);
template void box_ones_to_int<double>(const double *, int64_t, int32_t *, cudaStream_t);

// Compaction of a (bx x by) mask in lexicographic (x-fastest) order:
// one warp per column counts its cells, the host scans the column counts,
// then one warp per column assigns ranks with ballots.
__global__ void column_counts_kernel(const uint8_t *m, int bx, int by, int32_t *counts) {
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) / 32, lane = threadIdx.x % 32;
    if (warp >= by) return;
    int c = 0;
    for (int i = lane; i < bx; i += 32) c += m[i + (int64_t)bx * warp] ? 1 : 0;
    for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if (lane == 0) counts[warp] = c;
}
void column_counts(const uint8_t *m, int bx, int by, int32_t *counts, cudaStream_t st) {
    column_counts_kernel<<<(unsigned)cdiv((int64_t)by * 32, 256), 256, 0, st>>>(m, bx, by, counts);
    after_launch("column_counts");
}

__global__ void compact_map_kernel(const uint8_t *m, int bx, int by, const int32_t *col_start, int32_t *map,
                                   int32_t *pos, int64_t ld_img) {
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) / 32, lane = threadIdx.x % 32;
    if (warp >= by) return;
    int base = col_start[warp];
    for (int i0 = 0; i0 < bx; i0 += 32) {
        const int i = i0 + lane;
        const bool v = (i < bx) && m[i + (int64_t)bx * warp];
        const unsigned b = __ballot_sync(0xffffffffu, v);
        const int rank = __popc(b & ((1u << lane) - 1u));
        if (i < bx) {
            map[i + (int64_t)bx * warp] = v ? base + rank : -1;
            if (v && pos) pos[base + rank] = (int32_t)(i + ld_img * warp);
        }
        base += __popc(b);
    }
}
void compact_map(const uint8_t *m, int bx, int by, const int32_t *col_start, int32_t *map, int32_t *pos,
                 int64_t ld_img, cudaStream_t st) {
    compact_map_kernel<<<(unsigned)cdiv((int64_t)by * 32, 256), 256, 0, st>>>(m, bx, by, col_start, map, pos, ld_img);
    after_launch("compact_map");
}

// a3 for full rectangles: 𝕎 = w_x ⊗ w_y with w = (1, 2, .., L*, .., L*, .., 2, 1)
// (Alg. 2 step 2; the 2-D weights factor because 𝒯 is separable).
__global__ void weights_rect_kernel(int nx, int ny, int lx, int ly, int32_t *w) {
    const int64_t n = (int64_t)nx * ny;
    const int kx = nx - lx + 1, ky = ny - ly + 1;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
        const int i = (int)(t % nx), j = (int)(t / nx);
        const int wx = min(min(i + 1, nx - i), min(lx, kx));
        const int wy = min(min(j + 1, ny - j), min(ly, ky));
        w[t] = wx * wy;
    }
}
void weights_rect(int nx, int ny, int lx, int ly, int32_t *w, cudaStream_t st) {
    const int64_t n = (int64_t)nx * ny;
    weights_rect_kernel<<<(unsigned)std::min<int64_t>(cdiv(n, 256), 16 * num_sms()), 256, 0, st>>>(nx, ny, lx, ly, w);
    after_launch("weights_rect");
}

// Separable box sums for full rectangular windows (a2/a3 without a correlation kernel):
// 𝔎 = {κ : Σ_{d ∈ 𝔏} 1_𝔑(κ + d) = |𝔏|} (Alg. 6) and 𝕎(p) = #{κ ∈ 𝔎 : p − κ ∈ 𝔏}
// (Alg. 4 step 1) are 2-D box filters of 0/1 images; each pass is a sliding-window sum along one
// axis (one thread per line, exact int32).
// forward window: out[i, j] = Σ_{d < w} in[i + d, j] for i < no   (lines along the fast axis)
__global__ void box_fwd_x_kernel(const uint8_t *__restrict__ in, int nin, int ny, int w, int no, int32_t *__restrict__ out) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= ny) return;
    const uint8_t *r = in + (int64_t)nin * j;
    int32_t s = 0;
    for (int d = 0; d < w - 1 && d < nin; ++d) s += r[d];
    for (int i = 0; i < no; ++i) {
        s += r[i + w - 1];
        out[i + (int64_t)no * j] = s;
        s -= r[i];
    }
}
// forward window along the slow axis, thresholded: mask[i, j] = (Σ_{d < w} in[i, j + d] == full)
__global__ void box_fwd_y_kernel(const int32_t *__restrict__ in, int nx, int w, int no, int32_t full, uint8_t *__restrict__ mask) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nx) return;
    int32_t s = 0;
    for (int d = 0; d < w - 1; ++d) s += in[i + (int64_t)nx * d];
    for (int j = 0; j < no; ++j) {
        s += in[i + (int64_t)nx * (j + w - 1)];
        mask[i + (int64_t)nx * j] = (s == full) ? 1 : 0;
        s -= in[i + (int64_t)nx * j];
    }
}
// backward window along the fast axis: out[x, j] = Σ_{d < w, 0 <= x - d < nin} in[x - d, j], x < nout
__global__ void box_bwd_x_kernel(const uint8_t *__restrict__ in, int nin, int ny, int w, int nout, int32_t *__restrict__ out) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= ny) return;
    const uint8_t *r = in + (int64_t)nin * j;
    int32_t s = 0;
    for (int x = 0; x < nout; ++x) {
        if (x < nin) s += r[x];
        if (x - w >= 0 && x - w < nin) s -= r[x - w];
        out[x + (int64_t)nout * j] = s;
    }
}
// backward window along the slow axis: out[x, y] = Σ_{d < w, 0 <= y - d < nin} in[x, y - d], y < nout
__global__ void box_bwd_y_kernel(const int32_t *__restrict__ in, int nx, int nin, int w, int nout, int32_t *__restrict__ out) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    if (x >= nx) return;
    int32_t s = 0;
    for (int y = 0; y < nout; ++y) {
        if (y < nin) s += in[x + (int64_t)nx * y];
        if (y - w >= 0 && y - w < nin) s -= in[x + (int64_t)nx * (y - w)];
        out[x + (int64_t)nx * y] = s;
    }
}

void box_kmask(const uint8_t *nmask, int nx, int ny, int lx, int ly, uint8_t *kmask, int32_t *tmp, cudaStream_t st) {
    const int kx = nx - lx + 1, ky = ny - ly + 1;
    box_fwd_x_kernel<<<(unsigned)cdiv(ny, 128), 128, 0, st>>>(nmask, nx, ny, lx, kx, tmp);
    after_launch("box_fwd_x");
    box_fwd_y_kernel<<<(unsigned)cdiv(kx, 128), 128, 0, st>>>(tmp, kx, ly, ky, lx * ly, kmask);
    after_launch("box_fwd_y");
}

void box_weights(const uint8_t *kmask, int nx, int ny, int lx, int ly, int32_t *w, int32_t *tmp, cudaStream_t st) {
    const int kx = nx - lx + 1, ky = ny - ly + 1;
    box_bwd_x_kernel<<<(unsigned)cdiv(ky, 128), 128, 0, st>>>(kmask, kx, ky, lx, nx, tmp);
    after_launch("box_bwd_x");
    box_bwd_y_kernel<<<(unsigned)cdiv(nx, 128), 128, 0, st>>>(tmp, nx, ky, ly, ny, w);
    after_launch("box_bwd_y");
}

// "rest" group of eq. P:440-443: 𝕏 − Σ_g X̃_g on 𝔑′ (NaN elsewhere).
template <typename T>
__global__ void rest_kernel(const T *x, const int32_t *w, const T *groups, int ng, int64_t stride, int64_t n, T *rest) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
        if (w[t] <= 0) { rest[t] = (T)NAN; continue; }
        T s = x[t];
        for (int g = 0; g < ng; ++g) s -= groups[g * stride + t];
        rest[t] = s;
    }
}
template <typename T>
void rest_group(const T *x, const int32_t *w, const T *groups, int ngroups, int64_t stride, int64_t n, T *rest,
                cudaStream_t st) {
    rest_kernel<T><<<(unsigned)std::min<int64_t>(cdiv(n, 256), 16 * num_sms()), 256, 0, st>>>(
        x, w, groups, ngroups, stride, n, rest);
    after_launch("rest_group");
}
template void rest_group<float>(const float *, const int32_t *, const float *, int, int64_t, int64_t, float *, cudaStream_t);
template void rest_group<double>(const double *, const int32_t *, const double *, int, int64_t, int64_t, double *, cudaStream_t);

template <typename T>
__global__ void cast_kernel(const void *src, int is_double, T *dst, int64_t n) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x)
        dst[t] = is_double ? (T)((const double *)src)[t] : (T)((const float *)src)[t];
}
template <typename T>
void cast_copy(const void *src, int src_is_double, T *dst, int64_t n, cudaStream_t st) {
    if (n <= 0) return;
    cast_kernel<T><<<(unsigned)std::min<int64_t>(cdiv(n, 256), 16 * num_sms()), 256, 0, st>>>(src, src_is_double, dst, n);
    after_launch("cast_copy");
}
template void cast_copy<float>(const void *, int, float *, int64_t, cudaStream_t);
template void cast_copy<double>(const void *, int, double *, int64_t, cudaStream_t);

}  // namespace ssa
