// dtb_metrics.cu -- scoring kernels for the (W, k) sweep.
//
// Reference: /root/reference/pkg/src/docthresh/metrics.py
//   42-61   evaluate: foreground (value 0) is the positive class; TP/FP/FN/TN counts
//   83-136  sweep: stats once per W, then for every k the Sauvola/Niblack map, the strict
//           `img < tmap` prediction, and evaluate()'s counts
//   validation.py:31-40 as_binary_image: every pixel 0 or 255, first offender reported
//
// The GPU never materialises a prediction image for the sweep: one pass per W reads the
// page, the ground truth and the fp64 (mean, std) of that W, evaluates every k of the grid
// per pixel with the reference's fp64 operation sequence (threshold_exact), and keeps only
// two integers per k -- predicted-foreground and true-positive counts.  FP, FN and TN follow
// on the host from those and the ground-truth foreground count, and the F-measure is
// formed there with the reference's own float expressions (bit-identical ratios).
//
// Bytes per pixel per W: 1 (page) + 1 (gt) + 16 (mean, std); the k loop is ALU work on
// registers.  Counters: per-thread uint32 registers -> warp __reduce_add_sync -> shared
// uint64 -> one global atomicAdd per counter per CTA.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "docthresh_b200.h"
#include "dtb_common.cuh"

namespace dtb {

constexpr int SWEEP_KC = 8;  // k values per CTA row (grid.y walks the k grid in chunks)

struct SweepKs {
    double k[DTB_SWEEP_MAX_K];
    int n;
};

// Warp-sum `v` into a shared 64-bit slot.  Every lane of the warp must call it.
__device__ __forceinline__ void block_add(uint32_t v, unsigned long long* smem_slot) {
    const uint32_t w = __reduce_add_sync(0xffffffffu, v);
    if ((threadIdx.x & 31) == 0 && w) atomicAdd(smem_slot, (unsigned long long)w);
}

// evaluate() counts + as_binary_image() checks.  Either image may be NULL (validation and
// foreground count of the other one only).  out: [0] TP, [1] pred fg, [2] gt fg,
// [3] first non-binary linear index in pred, [4] same for gt (UINT64_MAX = none).
__global__ void __launch_bounds__(256) confusion_kernel(const uint8_t* __restrict__ pred,
                                                        int64_t pp,
                                                        const uint8_t* __restrict__ gt,
                                                        int64_t gp, int rows, int cols,
                                                        unsigned long long* out) {
    __shared__ unsigned long long acc[3];
    __shared__ unsigned long long bad[2];
    if (threadIdx.x < 3) acc[threadIdx.x] = 0;
    if (threadIdx.x < 2) bad[threadIdx.x] = ~0ull;
    __syncthreads();
    uint32_t tp = 0, pf = 0, gf = 0;
    unsigned long long bp = ~0ull, bg = ~0ull;
    const int64_t n = (int64_t)rows * cols;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int y = (int)(i / cols), x = (int)(i - (int64_t)y * cols);
        uint32_t p = 255, g = 255;
        if (pred) {
            p = pred[(int64_t)y * pp + x];
            if (p != 0 && p != 255 && bp == ~0ull) bp = (unsigned long long)i;
        }
        if (gt) {
            g = gt[(int64_t)y * gp + x];
            if (g != 0 && g != 255 && bg == ~0ull) bg = (unsigned long long)i;
        }
        pf += p == 0;
        gf += g == 0;
        tp += (p == 0) & (g == 0);
    }
    block_add(tp, &acc[0]);
    block_add(pf, &acc[1]);
    block_add(gf, &acc[2]);
    if (bp != ~0ull) atomicMin(&bad[0], bp);
    if (bg != ~0ull) atomicMin(&bad[1], bg);
    __syncthreads();
    if (threadIdx.x < 3 && acc[threadIdx.x]) atomicAdd(&out[threadIdx.x], acc[threadIdx.x]);
    if (threadIdx.x < 2 && bad[threadIdx.x] != ~0ull) atomicMin(&out[3 + threadIdx.x], bad[threadIdx.x]);
}

// One W of the sweep: for the k values [blockIdx.y*KC, +KC) count predicted-foreground
// pixels (img < t) and true positives (also gt == 0).  out[2*j] = pred fg, out[2*j+1] = TP.
__global__ void __launch_bounds__(256) sweep_counts_kernel(
    const uint8_t* __restrict__ img, int64_t ip, const uint8_t* __restrict__ gt, int64_t gp,
    int rows, int cols, const double* __restrict__ mean, const double* __restrict__ sd,
    int64_t sp, SweepKs ks, int method, double r, unsigned long long* out) {
    __shared__ unsigned long long acc[2 * SWEEP_KC];
    if (threadIdx.x < 2 * SWEEP_KC) acc[threadIdx.x] = 0;
    __syncthreads();
    const int j0 = blockIdx.y * SWEEP_KC;
    const int nk = min(SWEEP_KC, ks.n - j0);
    double kk[SWEEP_KC];
#pragma unroll
    for (int j = 0; j < SWEEP_KC; ++j) kk[j] = j < nk ? ks.k[j0 + j] : 0.0;
    uint32_t pf[SWEEP_KC], tp[SWEEP_KC];
#pragma unroll
    for (int j = 0; j < SWEEP_KC; ++j) pf[j] = tp[j] = 0;
    const int64_t n = (int64_t)rows * cols;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int y = (int)(i / cols), x = (int)(i - (int64_t)y * cols);
        const double f = (double)img[(int64_t)y * ip + x];
        const uint32_t gfg = gt[(int64_t)y * gp + x] == 0;
        const double m = mean[(int64_t)y * sp + x], s = sd[(int64_t)y * sp + x];
#pragma unroll
        for (int j = 0; j < SWEEP_KC; ++j) {
            if (j < nk) {
                const uint32_t black = f < threshold_exact(m, s, method, kk[j], r);
                pf[j] += black;
                tp[j] += black & gfg;
            }
        }
    }
#pragma unroll
    for (int j = 0; j < SWEEP_KC; ++j) {
        block_add(pf[j], &acc[2 * j]);
        block_add(tp[j], &acc[2 * j + 1]);
    }
    __syncthreads();
    if (threadIdx.x < 2 * nk && acc[threadIdx.x])
        atomicAdd(&out[2 * j0 + threadIdx.x], acc[threadIdx.x]);
}

static int grid_for(int64_t n, int per_sm) {
    return (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, (int64_t)num_sms() * per_sm));
}

}  // namespace dtb

using namespace dtb;

extern "C" {

int dtb_confusion(const uint8_t* pred, int64_t pred_pitch, const uint8_t* gt, int64_t gt_pitch,
                  int32_t rows, int32_t cols, uint64_t* counts5, void* stream) {
    if (!counts5 || (!pred && !gt)) return fail(DTB_E_INVALID, "null pointer");
    if (rows <= 0 || cols <= 0) return fail(DTB_E_INVALID, "image is empty");
    if ((pred && pred_pitch < cols) || (gt && gt_pitch < cols))
        return fail(DTB_E_INVALID, "pitch smaller than the row width");
    cudaStream_t st = (cudaStream_t)stream;
    cudaError_t e = cudaMemsetAsync(counts5, 0, 3 * sizeof(uint64_t), st);
    if (e == cudaSuccess) e = cudaMemsetAsync(counts5 + 3, 0xff, 2 * sizeof(uint64_t), st);
    if (e != cudaSuccess) return cuda_fail(e, "dtb_confusion memset");
    confusion_kernel<<<grid_for((int64_t)rows * cols, 8), 256, 0, st>>>(
        pred, pred_pitch, gt, gt_pitch, rows, cols, reinterpret_cast<unsigned long long*>(counts5));
    e = cudaGetLastError();
    return e == cudaSuccess ? DTB_OK : cuda_fail(e, "confusion_kernel launch");
}

int dtb_sweep_counts(const uint8_t* gray, int64_t gray_pitch, const uint8_t* gt, int64_t gt_pitch,
                     int32_t rows, int32_t cols, const double* mean, const double* std_,
                     int64_t stat_pitch, const double* ks, int32_t n_k, int32_t method, double r,
                     uint64_t* counts, void* stream) {
    if (!gray || !gt || !mean || !std_ || !ks || !counts) return fail(DTB_E_INVALID, "null pointer");
    if (rows <= 0 || cols <= 0) return fail(DTB_E_INVALID, "image is empty");
    if (n_k <= 0 || n_k > DTB_SWEEP_MAX_K)
        return fail(DTB_E_INVALID, "k grid: expected 1..%d values, got %d", DTB_SWEEP_MAX_K, n_k);
    if (method != DTB_METHOD_SAUVOLA && method != DTB_METHOD_NIBLACK)
        return fail(DTB_E_INVALID, "method: unknown code %d", method);
    if (gray_pitch < cols || gt_pitch < cols || stat_pitch < cols)
        return fail(DTB_E_INVALID, "pitch smaller than the row width");
    SweepKs p{};
    for (int j = 0; j < n_k; ++j) p.k[j] = ks[j];
    p.n = n_k;
    cudaStream_t st = (cudaStream_t)stream;
    cudaError_t e = cudaMemsetAsync(counts, 0, 2 * (size_t)n_k * sizeof(uint64_t), st);
    if (e != cudaSuccess) return cuda_fail(e, "dtb_sweep_counts memset");
    const dim3 grid(grid_for((int64_t)rows * cols, 8), (n_k + SWEEP_KC - 1) / SWEEP_KC);
    sweep_counts_kernel<<<grid, 256, 0, st>>>(gray, gray_pitch, gt, gt_pitch, rows, cols, mean,
                                              std_, stat_pitch, p, method, r,
                                              reinterpret_cast<unsigned long long*>(counts));
    e = cudaGetLastError();
    return e == cudaSuccess ? DTB_OK : cuda_fail(e, "sweep_counts_kernel launch");
}

}  // extern "C"
