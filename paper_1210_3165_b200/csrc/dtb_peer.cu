// dtb_peer.cu -- segmented (multi-buffer) band binarization and CUDA IPC helpers for reading
// a neighbour GPU's halo rows in place (SURVEY.md §8 row e).
//
// Row-band sharding (C4 at G GPUs): rank i owns rows [H*i/G, H*(i+1)/G) and needs r = W//2
// rows from each neighbour.  Instead of copying those rows into a local halo buffer first
// (the NCCL send/recv path in distributed.py), dtb_binarize_segments reads them where they
// live: the kernel's row staging (cp.async.bulk / loads in dtb_slide.cu, row_at()) takes
// each global row from one of up to three segments -- the upper neighbour's tail, the local
// band, the lower neighbour's head -- so the exchange is fused into the kernel's own reads
// over NVLink and there is no separate copy step to order or wait for.
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <string.h>

#include <algorithm>

#include "docthresh_b200.h"
#include "dtb_common.cuh"
#include "dtb_slide.cuh"

namespace dtb {
cudaError_t launch_slide(SlideParams p, int n_images, int num_sms, cudaStream_t st);
bool slide_ok(int r, int cols, int rows, const void* base, int64_t pitch, int64_t stride);
cudaError_t set_fp32_audit(unsigned long long* counters);
}  // namespace dtb

using namespace dtb;

extern "C" {

int dtb_binarize_segments(const uint8_t* const* seg_ptr, const int64_t* seg_pitch,
                          const int32_t* seg_rows, int32_t n_seg, int32_t row0_global,
                          int32_t rows_global, int32_t cols, int32_t out_row_begin,
                          int32_t out_row_end, uint8_t* binary, int64_t binary_pitch, int32_t win,
                          int32_t method, double k, double r, void* stream) {
    if (win < 3 || win % 2 == 0) return fail(DTB_E_INVALID, "window: must be an odd integer >= 3, got %d", win);
    if (method != DTB_METHOD_SAUVOLA && method != DTB_METHOD_NIBLACK)
        return fail(DTB_E_INVALID, "method: unknown code %d", method);
    if (method == DTB_METHOD_SAUVOLA && !(k > 0.0)) return fail(DTB_E_INVALID, "k_sauvola: must be > 0, got %g", k);
    if (!(r > 0.0)) return fail(DTB_E_INVALID, "r: must be > 0, got %g", r);
    if (!seg_ptr || !seg_pitch || !seg_rows || !binary) return fail(DTB_E_INVALID, "null pointer");
    if (n_seg < 1 || n_seg > 3) return fail(DTB_E_INVALID, "n_seg: expected 1..3, got %d", n_seg);
    if (cols <= 0 || rows_global <= 0) return fail(DTB_E_INVALID, "image is empty");
    if (out_row_begin < 0 || out_row_end > rows_global || out_row_begin > out_row_end)
        return fail(DTB_E_INVALID, "rows: output rows [%d,%d) outside image of %d rows",
                    out_row_begin, out_row_end, rows_global);
    SlideParams q{};
    int lo = row0_global, total = 0;
    for (int i = 0; i < 3; ++i) {
        const int rows_i = i < n_seg ? seg_rows[i] : 0;
        if (rows_i < 0) return fail(DTB_E_INVALID, "seg_rows[%d]: negative", i);
        if (rows_i > 0 && (!seg_ptr[i] || seg_pitch[i] < cols))
            return fail(DTB_E_INVALID, "segment %d: null pointer or pitch < cols", i);
        q.seg_ptr[i] = rows_i > 0 ? seg_ptr[i] : nullptr;
        q.seg_pitch[i] = rows_i > 0 ? seg_pitch[i] : 0;
        q.seg_lo[i] = lo;
        lo += rows_i;
        total += rows_i;
    }
    // empty segments: make the lookup skip them (a row never maps to a zero-row segment)
    if (q.seg_ptr[2] == nullptr) q.seg_lo[2] = 0x7fffffff;
    if (q.seg_ptr[1] == nullptr) q.seg_lo[1] = q.seg_lo[2];
    const int rad = win / 2;
    const int need0 = std::max(out_row_begin - rad, 0);
    const int need1 = std::min(out_row_end + rad, (int)rows_global);
    if (out_row_end > out_row_begin && (need0 < row0_global || need1 > row0_global + total))
        return fail(DTB_E_INVALID, "rows: band needs global rows [%d,%d) but segments hold [%d,%d)",
                    need0, need1, row0_global, row0_global + total);
    for (int i = 0; i < 3; ++i)
        if (q.seg_ptr[i] && !slide_ok(rad, cols, rows_global, q.seg_ptr[i], q.seg_pitch[i], 0))
            return fail(DTB_E_UNSUPPORTED,
                        "segment %d: needs 16-byte aligned base and pitch (and W within the fast "
                        "kernel's range); stage the rows into one buffer and use dtb_binarize", i);
    if (out_row_end <= out_row_begin) return DTB_OK;
    q.nseg = 3;
    q.in = q.seg_ptr[0] ? q.seg_ptr[0] : (q.seg_ptr[1] ? q.seg_ptr[1] : q.seg_ptr[2]);
    q.pitch = q.seg_ptr[0] ? q.seg_pitch[0] : (q.seg_ptr[1] ? q.seg_pitch[1] : q.seg_pitch[2]);
    q.cols = cols;
    q.row0 = row0_global;
    q.H = rows_global;
    q.in_rows = total;
    q.out_begin = out_row_begin;
    q.out_end = out_row_end;
    q.r = rad;
    q.rx = std::min(rad, cols - 1);
    q.bin = binary;
    q.bin_pitch = binary_pitch;
    q.method = method;
    q.k = k;
    q.rr = r;
    const cudaError_t e = launch_slide(q, 1, num_sms(), (cudaStream_t)stream);
    return e == cudaSuccess ? DTB_OK : cuda_fail(e, "slide kernel launch (segments)");
}

const char* dtb_last_kernel(void) { return dtb::last_kernel(); }

int dtb_debug_bb_times(uint64_t* device_buf, int32_t cap) {
    const cudaError_t e = dtb::bb_set_times(reinterpret_cast<unsigned long long*>(device_buf), device_buf ? cap : 0);
    return e == cudaSuccess ? DTB_OK : cuda_fail(e, "dtb_debug_bb_times");
}

// sqrt_rn_pos vs __dsqrt_rn, bit for bit: `count` values per class -- uniform bit patterns with
// exponents in [-70, 17], and variances formed like the epilogue's (Q/n - (S/n)^2 from integers)
__global__ void sqrt_selftest_kernel(unsigned long long seed, unsigned long long count,
                                     unsigned long long* mismatches) {
    unsigned long long x = seed ^ (0x9E3779B97F4A7C15ull * (blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x + 1));
    unsigned long long bad = 0;
    const unsigned long long per = (count + (unsigned long long)gridDim.x * blockDim.x - 1) /
                                   ((unsigned long long)gridDim.x * blockDim.x);
    for (unsigned long long i = 0; i < per; ++i) {
        x ^= x << 13; x ^= x >> 7; x ^= x << 17;  // xorshift64
        const int e = 1023 - 70 + (int)((x >> 52) % 88);
        const double a = __longlong_as_double(((long long)e << 52) | (long long)(x & 0xFFFFFFFFFFFFFull));
        if (__double_as_longlong(dtb::sqrt_rn_pos(a)) != __double_as_longlong(__dsqrt_rn(a))) ++bad;
        x ^= x << 13; x ^= x >> 7; x ^= x << 17;
        const unsigned n = 9 + (unsigned)(x % 65017);               // window counts 9 .. 255^2
        const unsigned f0 = (unsigned)((x >> 20) & 255), sp = (unsigned)((x >> 28) & 63);
        const unsigned long long S = (unsigned long long)n * f0 + ((x >> 34) % (1 + (unsigned long long)n * min(sp, 255u - f0)));
        const unsigned long long Q = S * f0 + ((x >> 40) % (1 + S * (sp + 1)));
        const double nd = (double)n, mean = __ddiv_rn((double)S, nd);
        const double var = __dsub_rn(__ddiv_rn((double)Q, nd), __dmul_rn(mean, mean));
        if (var > 0.0 && __double_as_longlong(dtb::sqrt_rn_pos(var)) != __double_as_longlong(__dsqrt_rn(var))) ++bad;
    }
    if (bad) atomicAdd(mismatches, bad);
}

int dtb_debug_sqrt_selftest(uint64_t seed, uint64_t count, uint64_t* mismatches) {
    if (!mismatches) return fail(DTB_E_INVALID, "dtb_debug_sqrt_selftest: mismatches is NULL");
    unsigned long long* d = nullptr;
    cudaError_t e = cudaMalloc(&d, sizeof(*d));
    if (e == cudaSuccess) e = cudaMemset(d, 0, sizeof(*d));
    if (e == cudaSuccess) {
        sqrt_selftest_kernel<<<1184, 256>>>(seed, count, d);
        e = cudaGetLastError();
    }
    unsigned long long h = 0;
    if (e == cudaSuccess) e = cudaMemcpy(&h, d, sizeof(h), cudaMemcpyDeviceToHost);
    if (d) cudaFree(d);
    *mismatches = h;
    return e == cudaSuccess ? DTB_OK : cuda_fail(e, "dtb_debug_sqrt_selftest");
}

int dtb_debug_bb_exact(uint64_t* count, int32_t reset) {
    if (!count) return fail(DTB_E_INVALID, "null pointer");
    unsigned long long v = 0;
    const cudaError_t e = dtb::bb_exact_count(&v, reset != 0);
    *count = v;
    return e == cudaSuccess ? DTB_OK : cuda_fail(e, "dtb_debug_bb_exact");
}

int dtb_set_fp32_audit(uint64_t* counters3) {
    const cudaError_t e = set_fp32_audit(reinterpret_cast<unsigned long long*>(counters3));
    return e == cudaSuccess ? DTB_OK : cuda_fail(e, "dtb_set_fp32_audit");
}

int dtb_ipc_export(const void* ptr, uint8_t* handle64, int64_t* offset) {
    if (!ptr || !handle64 || !offset) return fail(DTB_E_INVALID, "null pointer");
    // driver entry point through the runtime: the library must load on hosts without libcuda
    using GetRange = CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr);
    static GetRange get_range = nullptr;
    if (!get_range) {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        const cudaError_t ge = cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q);
        if (ge != cudaSuccess || !fn) return cuda_fail(ge, "cudaGetDriverEntryPoint(cuMemGetAddressRange)");
        get_range = reinterpret_cast<GetRange>(fn);
    }
    CUdeviceptr base = 0;
    size_t size = 0;
    const CUresult cr = get_range(&base, &size, (CUdeviceptr)ptr);
    if (cr != CUDA_SUCCESS) return fail(DTB_E_CUDA, "cuMemGetAddressRange failed (%d)", (int)cr);
    cudaIpcMemHandle_t h;
    const cudaError_t e = cudaIpcGetMemHandle(&h, (void*)base);
    if (e != cudaSuccess) return cuda_fail(e, "cudaIpcGetMemHandle");
    static_assert(sizeof(h) == 64, "CUDA IPC handles are 64 bytes");
    memcpy(handle64, &h, 64);
    *offset = (int64_t)((CUdeviceptr)ptr - base);
    return DTB_OK;
}

int dtb_ipc_import(const uint8_t* handle64, void** base) {
    if (!handle64 || !base) return fail(DTB_E_INVALID, "null pointer");
    cudaIpcMemHandle_t h;
    memcpy(&h, handle64, 64);
    const cudaError_t e = cudaIpcOpenMemHandle(base, h, cudaIpcMemLazyEnablePeerAccess);
    return e == cudaSuccess ? DTB_OK : cuda_fail(e, "cudaIpcOpenMemHandle");
}

int dtb_ipc_close(void* base) {
    if (!base) return fail(DTB_E_INVALID, "null pointer");
    const cudaError_t e = cudaIpcCloseMemHandle(base);
    return e == cudaSuccess ? DTB_OK : cuda_fail(e, "cudaIpcCloseMemHandle");
}

}  // extern "C"
