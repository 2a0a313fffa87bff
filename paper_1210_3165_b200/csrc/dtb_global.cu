// dtb_global.cu -- Otsu global threshold + apply_global, device-resident end to end
// (SURVEY.md §8 row f3).
//
// Reference: /root/reference/pkg/src/docthresh/threshold.py
//   55-88  otsu_threshold: 256-bin histogram, then a 256-step scan maximising
//          wb*wf*(mb-mf)^2 with strict `>` (ties -> smallest t); a one-value image returns
//          that value; the result is t+1 (strict `<` convention)
//   91-96  apply_global: pixel < T -> 0 else 255
//
// Three stream-ordered launches, no host round trip: a shared-memory histogram (16 pixels
// per thread per step, warp-private bins), a one-warp scan that replays the reference's
// Python arithmetic in IEEE fp64 (int/int true division and int->float conversion are
// both correctly rounded in Python, so __ddiv_rn / __ull2double_rn reproduce them bit for
// bit), and the apply kernel that reads T from device memory.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "docthresh_b200.h"
#include "dtb_common.cuh"

namespace dtb {

constexpr int HIST_NT = 256;

// Histogram with one 256-bin copy per warp in shared memory (fewer same-address atomics on
// document pages, where most pixels share a few background levels).
__global__ void __launch_bounds__(HIST_NT) hist_kernel(const uint8_t* __restrict__ in, int64_t pitch,
                                                       int rows, int cols,
                                                       unsigned long long* __restrict__ hist) {
    __shared__ uint32_t bins[HIST_NT / 32][256];
    for (int i = threadIdx.x; i < (HIST_NT / 32) * 256; i += HIST_NT) (&bins[0][0])[i] = 0;
    __syncthreads();
    uint32_t* mine = bins[threadIdx.x >> 5];
    const int64_t vec_per_row = cols >> 4;  // 16-byte groups when the row base is aligned
    const bool aligned = ((reinterpret_cast<uintptr_t>(in) | (uintptr_t)pitch) & 15) == 0;
    const int64_t stride = (int64_t)gridDim.x * HIST_NT;
    if (aligned) {
        const int64_t nvec = (int64_t)rows * vec_per_row;
        for (int64_t v = blockIdx.x * (int64_t)HIST_NT + threadIdx.x; v < nvec; v += stride) {
            const int64_t y = v / vec_per_row, xv = v - y * vec_per_row;
            const uint4 q = __ldg(reinterpret_cast<const uint4*>(in + y * pitch) + xv);
            const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
                for (int b = 0; b < 4; ++b) atomicAdd(&mine[(w[a] >> (8 * b)) & 255u], 1u);
        }
        // ragged right edge
        const int tail = cols - (int)(vec_per_row << 4);
        const int64_t ntail = (int64_t)rows * tail;
        for (int64_t t = blockIdx.x * (int64_t)HIST_NT + threadIdx.x; t < ntail; t += stride) {
            const int64_t y = t / tail;
            atomicAdd(&mine[in[y * pitch + (vec_per_row << 4) + (t - y * tail)]], 1u);
        }
    } else {
        const int64_t n = (int64_t)rows * cols;
        for (int64_t i = blockIdx.x * (int64_t)HIST_NT + threadIdx.x; i < n; i += stride) {
            const int64_t y = i / cols;
            atomicAdd(&mine[in[y * pitch + (i - y * cols)]], 1u);
        }
    }
    __syncthreads();
    for (int b = threadIdx.x; b < 256; b += HIST_NT) {
        uint32_t s = 0;
#pragma unroll
        for (int w = 0; w < HIST_NT / 32; ++w) s += bins[w][b];
        if (s) atomicAdd(&hist[b], (unsigned long long)s);
    }
}

// threshold.py:62-88, one thread.  hist: 256 counts; first: the image's first pixel.
__global__ void otsu_select_kernel(const unsigned long long* __restrict__ hist,
                                   const uint8_t* __restrict__ first, int32_t* __restrict__ t_out) {
    if (threadIdx.x != 0) return;
    unsigned long long total = 0, sum_all = 0;
    for (int t = 0; t < 256; ++t) {
        total += hist[t];
        sum_all += (unsigned long long)t * hist[t];
    }
    int best_t = -1;
    double best_var = -1.0;
    unsigned long long wb = 0, sumb = 0;
    for (int t = 0; t < 256; ++t) {
        wb += hist[t];
        sumb += (unsigned long long)t * hist[t];
        if (wb == 0) continue;
        const unsigned long long wf = total - wb;
        if (wf == 0) break;
        // sums < 2^53 (255 * 2^36 pixels at most), so the int -> double casts are exact and
        // __ddiv_rn is Python's correctly rounded int / int
        const double mb = __ddiv_rn((double)sumb, (double)wb);
        const double mf = __ddiv_rn((double)(sum_all - sumb), (double)wf);
        const double d = __dsub_rn(mb, mf);
        // Python: (wb*wf) is an exact int, then int * float rounds it to the nearest double
        const double var = __dmul_rn(__ull2double_rn(wb * wf), __dmul_rn(d, d));
        if (var > best_var) {
            best_var = var;
            best_t = t;
        }
    }
    *t_out = best_t < 0 ? (int32_t)first[0] : best_t + 1;
}

// threshold.py:91-96 with T read from device memory; optional tmap filled with T
// (threshold.py:124-127 returns a constant map for Otsu).
__global__ void apply_dev_kernel(const uint8_t* __restrict__ in, int64_t pitch, int rows, int cols,
                                 const int32_t* __restrict__ t_dev, uint8_t* __restrict__ out,
                                 int64_t out_pitch, double* __restrict__ tmap) {
    const int t = *t_dev;
    const int64_t n = (int64_t)rows * cols;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t y = i / cols, x = i - y * cols;
        out[y * out_pitch + x] = (int)in[y * pitch + x] < t ? 0 : 255;
        if (tmap) tmap[i] = (double)t;
    }
}

}  // namespace dtb

using namespace dtb;

extern "C" {

int dtb_otsu(const uint8_t* gray, int64_t pitch, int32_t rows, int32_t cols, uint64_t* hist256,
             int32_t* t_out, void* stream) {
    if (!gray || !hist256 || !t_out) return fail(DTB_E_INVALID, "null pointer");
    if (rows <= 0 || cols <= 0) return fail(DTB_E_INVALID, "image is empty");
    if (pitch < cols) return fail(DTB_E_INVALID, "pitch smaller than the row width");
    cudaStream_t st = (cudaStream_t)stream;
    cudaError_t e = cudaMemsetAsync(hist256, 0, 256 * sizeof(uint64_t), st);
    if (e != cudaSuccess) return cuda_fail(e, "dtb_otsu memset");
    const int64_t n16 = ((int64_t)rows * cols + 15) / 16;
    const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>((n16 + HIST_NT - 1) / HIST_NT,
                                                                   (int64_t)num_sms() * 4));
    auto* h = reinterpret_cast<unsigned long long*>(hist256);
    hist_kernel<<<blocks, HIST_NT, 0, st>>>(gray, pitch, rows, cols, h);
    otsu_select_kernel<<<1, 32, 0, st>>>(h, gray, t_out);
    e = cudaGetLastError();
    return e == cudaSuccess ? DTB_OK : cuda_fail(e, "otsu kernels launch");
}

int dtb_apply_global_dev(const uint8_t* gray, int64_t pitch, int32_t rows, int32_t cols,
                         const int32_t* t_dev, uint8_t* out, int64_t out_pitch, double* tmap,
                         void* stream) {
    if (!gray || !t_dev || !out) return fail(DTB_E_INVALID, "null pointer");
    if (rows <= 0 || cols <= 0) return fail(DTB_E_INVALID, "image is empty");
    if (pitch < cols || out_pitch < cols) return fail(DTB_E_INVALID, "pitch smaller than the row width");
    const int64_t n = (int64_t)rows * cols;
    const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, (int64_t)num_sms() * 16));
    apply_dev_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(gray, pitch, rows, cols, t_dev, out,
                                                               out_pitch, tmap);
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? DTB_OK : cuda_fail(e, "apply_dev_kernel launch");
}

}  // extern "C"
