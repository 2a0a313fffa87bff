// dtb_kernels.cu -- libdocthresh_b200: B200 (sm_100a) kernels for windowed-statistics
// binarization + the extern "C" ABI declared in include/docthresh_b200.h.
//
// Reference hot path (/root/reference/pkg/src/docthresh):
//   threshold.py:121-148 binarize -> threshold.py:113-118 _mean_std
//     -> stats.py:166-191 mean_std_{naive,integral} -> stats.py:50-54 _finish_arrays
//     -> threshold.py:143-147 Sauvola / Niblack epilogue, strict `<`
//   pnm.py:18-38 to_gray
//
// v1 structure ("strip" kernel): one CTA owns a strip of TW = NC - 2*rx output columns
// and a band of output rows.  Each thread keeps exact running vertical column sums
// (sum f, sum f^2) for CPT input columns in registers and slides them down the band
// (add row y+r, subtract row y-r-1: the O(1)-per-pixel sliding formulation).  Per output
// row the CTA forms the horizontal prefix of the column sums in shared memory and each
// output reads two prefix entries.  Sums are exact integers (uint32 mod 2^32 is exact
// because every true window sum is < 2^32 for the supported range; otherwise the
// 64-bit instantiation is used).  The epilogue replays the reference fp64 sequence.
#include <cuda_runtime.h>
#include <stdarg.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>

#include "docthresh_b200.h"
#include "dtb_common.cuh"
#include "dtb_slide.cuh"

namespace dtb {

static thread_local char g_err[512] = "";

int fail(int code, const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
    return code;
}

int cuda_fail(cudaError_t e, const char* where) {
    return fail(DTB_E_CUDA, "%s: %s", where, cudaGetErrorString(e));
}

struct StripParams {
    const uint8_t* in;
    int64_t pitch;
    int64_t img_stride;  // batch stride (bytes) between images
    int cols;
    int row0;      // global row index of in[0]
    int H;         // global rows
    int out_begin, out_end;
    int r;         // win / 2
    int rx;        // min(r, cols - 1): horizontal radius actually needed
    int TH;        // output rows per CTA band
    // binarize outputs
    uint8_t* bin;
    int64_t bin_pitch;
    int64_t out_stride;
    double* tmap;
    int64_t tmap_pitch;
    int method;
    double k, rr;
    // statistics outputs (dense, pitch = cols elements)
    int64_t* S;
    int64_t* Q;
    int32_t* cnt;
    double* mean;
    double* std;
};

enum { MODE_BINARIZE = 0, MODE_STATS = 1 };

template <int NT, int CPT, typename SumT, int MODE>
__global__ void __launch_bounds__(NT) strip_kernel(StripParams p) {
    constexpr int NC = NT * CPT;
    constexpr int NW = NT / 32;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    SumT* PS = reinterpret_cast<SumT*>(smem_raw);
    SumT* PQ = PS + (NC + 1);
    SumT* wS = PQ + (NC + 1);
    SumT* wQ = wS + NW;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint8_t* in = p.in + (int64_t)blockIdx.z * p.img_stride;
    const int TW = NC - 2 * p.rx;
    const int xo0 = blockIdx.x * TW;   // first output column of this strip
    const int xc0 = xo0 - p.rx;        // image column held at prefix index 0
    const int ya = p.out_begin + blockIdx.y * p.TH;
    const int yb = min(ya + p.TH, p.out_end);
    if (ya >= yb) return;

    uint32_t colS[CPT];
    SumT colQ[CPT];
#pragma unroll
    for (int j = 0; j < CPT; ++j) { colS[j] = 0; colQ[j] = 0; }

    auto row_ptr = [&](int g) { return in + (int64_t)(g - p.row0) * p.pitch; };
    auto add_row = [&](int g) {
        const uint8_t* rp = row_ptr(g);
#pragma unroll
        for (int j = 0; j < CPT; ++j) {
            const int c = xc0 + tid * CPT + j;
            if (c >= 0 && c < p.cols) {
                const uint32_t v = rp[c];
                colS[j] += v;
                colQ[j] += (SumT)(v * v);
            }
        }
    };
    auto sub_row = [&](int g) {
        const uint8_t* rp = row_ptr(g);
#pragma unroll
        for (int j = 0; j < CPT; ++j) {
            const int c = xc0 + tid * CPT + j;
            if (c >= 0 && c < p.cols) {
                const uint32_t v = rp[c];
                colS[j] -= v;
                colQ[j] -= (SumT)(v * v);
            }
        }
    };

    // Warm-up: vertical window of the first output row, clipped to the image.
    {
        const int g0 = max(ya - p.r, 0), g1 = min(ya + p.r, p.H - 1);
        for (int g = g0; g <= g1; ++g) add_row(g);
    }

    if (tid == 0) { PS[0] = 0; PQ[0] = 0; }
    for (int y = ya; y < yb; ++y) {
        if (y > ya) {
            const int gi = y + p.r, go = y - p.r - 1;
            if (gi < p.H) add_row(gi);
            if (go >= 0) sub_row(go);
        }
        // Block-wide inclusive prefix of the column sums (exact mod 2^bits(SumT)).
        SumT ls[CPT], lq[CPT];
        ls[0] = colS[0];
        lq[0] = colQ[0];
#pragma unroll
        for (int j = 1; j < CPT; ++j) { ls[j] = ls[j - 1] + colS[j]; lq[j] = lq[j - 1] + colQ[j]; }
        SumT ts = ls[CPT - 1], tq = lq[CPT - 1];
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const SumT vs = __shfl_up_sync(0xffffffffu, ts, off);
            const SumT vq = __shfl_up_sync(0xffffffffu, tq, off);
            if (lane >= off) { ts += vs; tq += vq; }
        }
        if (lane == 31) { wS[warp] = ts; wQ[warp] = tq; }
        __syncthreads();
        SumT bs = ts - ls[CPT - 1], bq = tq - lq[CPT - 1];
#pragma unroll
        for (int w = 0; w < NW; ++w)
            if (w < warp) { bs += wS[w]; bq += wQ[w]; }
#pragma unroll
        for (int j = 0; j < CPT; ++j) {
            PS[tid * CPT + j + 1] = bs + ls[j];
            PQ[tid * CPT + j + 1] = bq + lq[j];
        }
        __syncthreads();

        const int ny = min(y + p.r, p.H - 1) - max(y - p.r, 0) + 1;
        const uint8_t* rp = row_ptr(y);
        for (int o = tid; o < TW; o += NT) {
            const int x = xo0 + o;
            if (x >= p.cols) break;
            const SumT S = PS[o + 2 * p.rx + 1] - PS[o];
            const SumT Q = PQ[o + 2 * p.rx + 1] - PQ[o];
            const int nx = min(x + p.r, p.cols - 1) - max(x - p.r, 0) + 1;
            const double n = (double)ny * (double)nx;
            double mean, sd;
            finish_exact((double)S, (double)Q, n, mean, sd);
            if constexpr (MODE == MODE_BINARIZE) {
                const double t = threshold_exact(mean, sd, p.method, p.k, p.rr);
                const int yo = y - p.out_begin;
                uint8_t* bp = p.bin + (int64_t)blockIdx.z * p.out_stride + (int64_t)yo * p.bin_pitch;
                bp[x] = ((double)rp[x] < t) ? 0 : 255;
                if (p.tmap) {
                    double* tp = (double*)((char*)p.tmap + (int64_t)yo * p.tmap_pitch);
                    tp[x] = t;
                }
            } else {
                const int64_t idx = (int64_t)y * p.cols + x;
                if (p.S) p.S[idx] = (int64_t)S;
                if (p.Q) p.Q[idx] = (int64_t)Q;
                if (p.cnt) p.cnt[idx] = ny * nx;
                if (p.mean) p.mean[idx] = mean;
                if (p.std) p.std[idx] = sd;
            }
        }
    }
}

// to_gray (pnm.py:18-38), 16 pixels per thread: 3 x 16-byte loads of interleaved RGB, integer
// 299r+587g+114b with the fp64 re-evaluation only at exact .5 ties (gray_fast), one 16-byte
// store.  Rows are processed by a grid-stride loop over (row, 16-pixel chunk); ragged row
// tails and unaligned rows fall back to per-pixel code.
__global__ void to_gray_kernel(const uint8_t* rgb, int64_t rgb_pitch, uint8_t* gray,
                               int64_t gray_pitch, int rows, int cols) {
    const int chunks = (cols + 15) / 16;
    const int64_t n = (int64_t)rows * chunks;
    const bool vec = ((reinterpret_cast<uintptr_t>(rgb) | (uintptr_t)rgb_pitch |
                       reinterpret_cast<uintptr_t>(gray) | (uintptr_t)gray_pitch) & 15) == 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int y = (int)(i / chunks), x0 = 16 * (int)(i % chunks);
        const uint8_t* src = rgb + (int64_t)y * rgb_pitch + 3 * (int64_t)x0;
        uint8_t* dst = gray + (int64_t)y * gray_pitch + x0;
        if (vec && x0 + 16 <= cols) {
            uint32_t w[12];
            const uint4* s4 = reinterpret_cast<const uint4*>(src);
#pragma unroll
            for (int q = 0; q < 3; ++q) {
                const uint4 v = __ldg(s4 + q);
                w[4 * q] = v.x; w[4 * q + 1] = v.y; w[4 * q + 2] = v.z; w[4 * q + 3] = v.w;
            }
            uint32_t o[4] = {0, 0, 0, 0};
#pragma unroll
            for (int j = 0; j < 16; ++j) {
                const int b = 3 * j;
                const uint32_t r = (w[b >> 2] >> (8 * (b & 3))) & 0xFF;
                const uint32_t g = (w[(b + 1) >> 2] >> (8 * ((b + 1) & 3))) & 0xFF;
                const uint32_t bl = (w[(b + 2) >> 2] >> (8 * ((b + 2) & 3))) & 0xFF;
                o[j >> 2] |= gray_fast(r, g, bl) << (8 * (j & 3));
            }
            *reinterpret_cast<uint4*>(dst) = make_uint4(o[0], o[1], o[2], o[3]);
        } else {
            for (int j = 0; j < 16 && x0 + j < cols; ++j)
                dst[j] = (uint8_t)gray_fast(src[3 * j], src[3 * j + 1], src[3 * j + 2]);
        }
    }
}

// Mask-restricted statistics: the reference's `sampled` engine (stats.py:133-163) for an
// arbitrary offset set (masks.py GS-1..GS-6).  One thread per pixel, O(|mask|) exact
// integer sums, in-bounds count, then the shared fp64 finish + epilogue.
__global__ void sampled_kernel(const uint8_t* in, int64_t pitch, int rows, int cols,
                               const int2* offs, int n_offs, double* mean_o, double* std_o,
                               int32_t* cnt_o, uint8_t* bin, double* tmap, int method, double k,
                               double rr) {
    extern __shared__ int2 soffs[];
    for (int i = threadIdx.x; i < n_offs; i += blockDim.x) soffs[i] = offs[i];
    __syncthreads();
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    const int y = blockIdx.y;
    if (x >= cols) return;
    uint64_t S = 0, Q = 0;
    uint32_t n = 0;
    for (int i = 0; i < n_offs; ++i) {
        const int sx = x + soffs[i].x, sy = y + soffs[i].y;
        if (sx >= 0 && sx < cols && sy >= 0 && sy < rows) {
            const uint32_t v = in[(int64_t)sy * pitch + sx];
            S += v;
            Q += v * v;
            ++n;
        }
    }
    double mean, sd;
    finish_exact((double)S, (double)Q, (double)n, mean, sd);
    const int64_t idx = (int64_t)y * cols + x;
    if (mean_o) mean_o[idx] = mean;
    if (std_o) std_o[idx] = sd;
    if (cnt_o) cnt_o[idx] = (int32_t)n;
    if (bin) {
        const double t = threshold_exact(mean, sd, method, k, rr);
        bin[idx] = ((double)in[(int64_t)y * pitch + x] < t) ? 0 : 255;
        if (tmap) tmap[idx] = t;
    }
}

// 256-bin histogram (threshold.py:63 np.bincount) with per-CTA shared-memory bins.
__global__ void histogram_kernel(const uint8_t* in, int64_t pitch, int rows, int cols,
                                 unsigned long long* hist) {
    __shared__ uint32_t bins[256];
    for (int i = threadIdx.x; i < 256; i += blockDim.x) bins[i] = 0;
    __syncthreads();
    const int64_t n = (int64_t)rows * cols;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int y = (int)(i / cols), x = (int)(i % cols);
        atomicAdd(&bins[in[(int64_t)y * pitch + x]], 1u);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < 256; i += blockDim.x)
        if (bins[i]) atomicAdd(&hist[i], (unsigned long long)bins[i]);
}

// apply_global (threshold.py:91-96): pixel < t -> 0 else 255.
__global__ void apply_global_kernel(const uint8_t* in, int64_t pitch, int rows, int cols, int t,
                                    uint8_t* out, int64_t out_pitch) {
    const int64_t n = (int64_t)rows * cols;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int y = (int)(i / cols), x = (int)(i % cols);
        out[(int64_t)y * out_pitch + x] = (int)in[(int64_t)y * pitch + x] < t ? 0 : 255;
    }
}

// Summed-area tables (stats.py:82-91 build_integral): pass 1 row prefixes, pass 2 column
// accumulation, int64, zero top row / left column.  Off the hot path (16 B/px).
__global__ void sat_rows_kernel(const uint8_t* in, int64_t pitch, int rows, int cols,
                                int64_t* s, int64_t* sq) {
    const int64_t tw = (int64_t)cols + 1;
    for (int y = blockIdx.x * blockDim.x + threadIdx.x; y <= rows; y += gridDim.x * blockDim.x) {
        int64_t* srow = s + (int64_t)y * tw;
        int64_t* qrow = sq + (int64_t)y * tw;
        srow[0] = 0;
        qrow[0] = 0;
        if (y == 0) {
            for (int x = 1; x <= cols; ++x) { srow[x] = 0; qrow[x] = 0; }
            continue;
        }
        const uint8_t* rp = in + (int64_t)(y - 1) * pitch;
        int64_t a = 0, b = 0;
        for (int x = 0; x < cols; ++x) {
            const int64_t v = rp[x];
            a += v;
            b += v * v;
            srow[x + 1] = a;
            qrow[x + 1] = b;
        }
    }
}

__global__ void sat_cols_kernel(int rows, int cols, int64_t* s, int64_t* sq) {
    const int64_t tw = (int64_t)cols + 1;
    for (int x = blockIdx.x * blockDim.x + threadIdx.x; x <= cols; x += gridDim.x * blockDim.x) {
        int64_t a = 0, b = 0;
        for (int y = 1; y <= rows; ++y) {
            a += s[(int64_t)y * tw + x];
            b += sq[(int64_t)y * tw + x];
            s[(int64_t)y * tw + x] = a;
            sq[(int64_t)y * tw + x] = b;
        }
    }
}

static int g_num_sms = 0;

int num_sms() {
    if (g_num_sms == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
        if (g_num_sms <= 0) g_num_sms = 148;
    }
    return g_num_sms;
}

template <int NT, int CPT, typename SumT, int MODE>
static cudaError_t run_strip(dim3 grid, const StripParams& p, cudaStream_t st) {
    constexpr int NC = NT * CPT;
    const size_t smem = sizeof(SumT) * (2 * (NC + 1) + 2 * (NT / 32));
    auto kern = strip_kernel<NT, CPT, SumT, MODE>;
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
    }
    kern<<<grid, NT, smem, st>>>(p);
    return cudaSuccess;
}

template <int MODE>
static int launch_strip(StripParams p, int n_images, cudaStream_t st) {
    if (MODE == MODE_BINARIZE) set_last_kernel("strip_kernel");
    constexpr int NT = 256;
    const int rows_out = p.out_end - p.out_begin;
    if (rows_out <= 0 || p.cols <= 0 || n_images <= 0) return DTB_OK;
    p.rx = std::min(p.r, p.cols - 1);
    const int ry = std::min(p.r, p.H - 1);
    // Widest true sums: S <= 255*n, Q <= 65025*n with n <= (2ry+1)(2rx+1).
    const double nmax = (2.0 * ry + 1.0) * (2.0 * p.rx + 1.0);
    const bool wide = 65025.0 * nmax >= 4294967296.0;
    int NC;
    if (2 * p.rx + 64 <= NT * 4) NC = NT * 4;
    else if (2 * p.rx + 64 <= NT * 16) NC = NT * 16;
    else return fail(DTB_E_UNSUPPORTED, "window: horizontal radius %d exceeds this build's strip (max 2016)", p.rx);
    const int TW = NC - 2 * p.rx;
    const int nstrips = (p.cols + TW - 1) / TW;
    const int target = num_sms() * 4;
    int nbands = (target + nstrips * n_images - 1) / (nstrips * n_images);
    nbands = std::max(1, std::min(nbands, (rows_out + 31) / 32));
    p.TH = (rows_out + nbands - 1) / nbands;
    dim3 grid(nstrips, (rows_out + p.TH - 1) / p.TH, n_images);
    cudaError_t e;
    if (NC == NT * 4) {
        e = wide ? run_strip<NT, 4, uint64_t, MODE>(grid, p, st)
                 : run_strip<NT, 4, uint32_t, MODE>(grid, p, st);
    } else {
        e = wide ? run_strip<NT, 16, uint64_t, MODE>(grid, p, st)
                 : run_strip<NT, 16, uint32_t, MODE>(grid, p, st);
    }
    if (e == cudaSuccess) e = cudaGetLastError();
    return e == cudaSuccess ? DTB_OK : cuda_fail(e, "strip_kernel launch");
}

// The fast kernel keeps 32-bit sums: every window sum must stay < 2^32, and the strip
// (<= 8 warps = 8192 columns) must hold a window plus 32 outputs.
bool slide_ok(int r, int cols, int rows, const void* base, int64_t pitch,
                     int64_t stride) {
    // rows are staged with 16-byte bulk copies
    if (((uintptr_t)base | (uintptr_t)pitch | (uintptr_t)stride) & 15) return false;
    const double rx = std::min(r, cols - 1), ry = std::min(r, rows - 1);
    const double nmax = (2.0 * rx + 1.0) * (2.0 * ry + 1.0);
    return 65025.0 * nmax < 4294967296.0 && 2 * rx + 16 + 32 <= 8192;
}

static int check_window(int win) {
    if (win < 3 || (win % 2) == 0)
        return fail(DTB_E_INVALID, "window: must be an odd integer >= 3, got %d", win);
    return DTB_OK;
}

static int check_method(int method, double k, double r) {
    if (method != DTB_METHOD_SAUVOLA && method != DTB_METHOD_NIBLACK)
        return fail(DTB_E_INVALID, "method: expected sauvola(%d) or niblack(%d), got %d",
                    DTB_METHOD_SAUVOLA, DTB_METHOD_NIBLACK, method);
    if (method == DTB_METHOD_SAUVOLA && !(k > 0.0))
        return fail(DTB_E_INVALID, "k_sauvola: must be > 0, got %g", k);
    if (!(r > 0.0)) return fail(DTB_E_INVALID, "r: must be > 0, got %g", r);
    return DTB_OK;
}

}  // namespace dtb

using namespace dtb;

extern "C" {

int dtb_abi_version(void) { return DTB_ABI_VERSION; }

const char* dtb_last_error(void) { return g_err; }

int dtb_to_gray(const uint8_t* rgb, int64_t rgb_pitch, uint8_t* gray, int64_t gray_pitch,
                int32_t rows, int32_t cols, void* stream) {
    if (rows < 0 || cols < 0) return fail(DTB_E_INVALID, "shape: negative size %dx%d", rows, cols);
    if (!rgb || !gray) return fail(DTB_E_INVALID, "null image pointer");
    if (rows == 0 || cols == 0) return DTB_OK;
    const int64_t n = (int64_t)rows * ((cols + 15) / 16);
    const int threads = 256;
    const int64_t blocks = std::min<int64_t>((n + threads - 1) / threads, (int64_t)num_sms() * 16);
    to_gray_kernel<<<(unsigned)blocks, threads, 0, (cudaStream_t)stream>>>(rgb, rgb_pitch, gray,
                                                                         gray_pitch, rows, cols);
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? DTB_OK : cuda_fail(e, "to_gray_kernel launch");
}

int dtb_binarize(const uint8_t* gray, int64_t pitch, int32_t in_rows, int32_t cols,
                 int32_t row0_global, int32_t rows_global, int32_t out_row_begin,
                 int32_t out_row_end, uint8_t* binary, int64_t binary_pitch, double* tmap,
                 int64_t tmap_pitch, int32_t win, int32_t method, double k, double r,
                 void* stream) {
    int rc;
    if ((rc = check_window(win))) return rc;
    if ((rc = check_method(method, k, r))) return rc;
    if (!gray || !binary) return fail(DTB_E_INVALID, "null image pointer");
    if (cols <= 0 || rows_global <= 0) return fail(DTB_E_INVALID, "image is empty");
    if (out_row_begin < 0 || out_row_end > rows_global || out_row_begin > out_row_end)
        return fail(DTB_E_INVALID, "rows: output rows [%d,%d) outside image of %d rows",
                    out_row_begin, out_row_end, rows_global);
    const int rad = win / 2;
    const int need0 = std::max(out_row_begin - rad, 0);
    const int need1 = std::min(out_row_end + rad, (int)rows_global);
    if (out_row_end > out_row_begin && (need0 < row0_global || need1 > row0_global + in_rows))
        return fail(DTB_E_INVALID,
                    "rows: band needs global rows [%d,%d) but buffer holds [%d,%d)", need0,
                    need1, row0_global, row0_global + in_rows);
    if (slide_ok(rad, cols, rows_global, gray, pitch, 0) &&
        (!tmap || (((uintptr_t)tmap | (uintptr_t)tmap_pitch) & 15) == 0)) {
        SlideParams q{};
        q.in = gray; q.pitch = pitch; q.cols = cols; q.row0 = row0_global; q.H = rows_global;
        q.in_rows = in_rows;
        q.out_begin = out_row_begin; q.out_end = out_row_end; q.r = rad;
        q.rx = std::min(rad, cols - 1);
        q.bin = binary; q.bin_pitch = binary_pitch; q.method = method; q.k = k; q.rr = r;
        q.tmap = tmap; q.tmap_pitch = tmap_pitch;  // tmap rows = output rows [out_begin, out_end)
        if (out_row_end <= out_row_begin) return DTB_OK;
        const cudaError_t e = launch_slide(q, 1, num_sms(), (cudaStream_t)stream);
        return e == cudaSuccess ? DTB_OK : cuda_fail(e, "slide_kernel launch");
    }
    StripParams p{};
    p.in = gray; p.pitch = pitch; p.cols = cols; p.row0 = row0_global; p.H = rows_global;
    p.out_begin = out_row_begin; p.out_end = out_row_end; p.r = rad;
    p.bin = binary; p.bin_pitch = binary_pitch; p.tmap = tmap; p.tmap_pitch = tmap_pitch;
    p.method = method; p.k = k; p.rr = r;
    return launch_strip<MODE_BINARIZE>(p, 1, (cudaStream_t)stream);
}

int dtb_binarize_batch(const uint8_t* gray, int64_t image_stride, int32_t n_images,
                       int32_t rows, int32_t cols, uint8_t* binary, int64_t out_stride,
                       int32_t win, int32_t method, double k, double r, void* stream) {
    int rc;
    if ((rc = check_window(win))) return rc;
    if ((rc = check_method(method, k, r))) return rc;
    if (!gray || !binary) return fail(DTB_E_INVALID, "null image pointer");
    if (rows <= 0 || cols <= 0) return fail(DTB_E_INVALID, "image is empty");
    if (n_images < 0) return fail(DTB_E_INVALID, "n_images: negative");
    if (n_images > 65535) return fail(DTB_E_UNSUPPORTED, "n_images: at most 65535 per call");
    if (slide_ok(win / 2, cols, rows, gray, cols, image_stride)) {
        SlideParams q{};
        q.in = gray; q.pitch = cols; q.img_stride = image_stride; q.cols = cols; q.row0 = 0;
        q.H = rows; q.in_rows = rows; q.out_begin = 0; q.out_end = rows; q.r = win / 2;
        q.rx = std::min(win / 2, cols - 1);
        q.bin = binary; q.bin_pitch = cols; q.out_stride = out_stride;
        q.method = method; q.k = k; q.rr = r;
        if (n_images == 0) return DTB_OK;
        const cudaError_t e = launch_slide(q, n_images, num_sms(), (cudaStream_t)stream);
        return e == cudaSuccess ? DTB_OK : cuda_fail(e, "slide_kernel launch");
    }
    StripParams p{};
    p.in = gray; p.pitch = cols; p.img_stride = image_stride; p.cols = cols; p.row0 = 0;
    p.H = rows; p.out_begin = 0; p.out_end = rows; p.r = win / 2;
    p.bin = binary; p.bin_pitch = cols; p.out_stride = out_stride;
    p.method = method; p.k = k; p.rr = r;
    return launch_strip<MODE_BINARIZE>(p, n_images, (cudaStream_t)stream);
}

int dtb_rgb_binarize(const uint8_t* rgb, int64_t rgb_pitch, int32_t rows, int32_t cols,
                     uint8_t* binary, int64_t binary_pitch, uint8_t* gray_out,
                     int64_t gray_pitch, int32_t win, int32_t method, double k, double r,
                     void* stream) {
    if (!gray_out)
        return fail(DTB_E_UNSUPPORTED, "gray_out: this build stages the gray page; pass a buffer");
    int rc = dtb_to_gray(rgb, rgb_pitch, gray_out, gray_pitch, rows, cols, stream);
    if (rc) return rc;
    return dtb_binarize(gray_out, gray_pitch, rows, cols, 0, rows, 0, rows, binary,
                        binary_pitch, nullptr, 0, win, method, k, r, stream);
}

int dtb_window_stats(const uint8_t* gray, int64_t pitch, int32_t rows, int32_t cols,
                     int32_t win, int64_t* S, int64_t* Q, int32_t* count, double* mean,
                     double* std, void* stream) {
    int rc;
    if ((rc = check_window(win))) return rc;
    if (!gray) return fail(DTB_E_INVALID, "null image pointer");
    if (rows <= 0 || cols <= 0) return fail(DTB_E_INVALID, "image is empty");
    StripParams p{};
    p.in = gray; p.pitch = pitch; p.cols = cols; p.row0 = 0; p.H = rows;
    p.out_begin = 0; p.out_end = rows; p.r = win / 2;
    p.S = S; p.Q = Q; p.cnt = count; p.mean = mean; p.std = std;
    return launch_strip<MODE_STATS>(p, 1, (cudaStream_t)stream);
}

int dtb_sampled_stats(const uint8_t* gray, int64_t pitch, int32_t rows, int32_t cols,
                      const int32_t* offsets_xy, int32_t n_offsets, double* mean, double* std,
                      int32_t* count, uint8_t* binary, double* tmap, int32_t method, double k,
                      double r, void* stream) {
    if (!gray || !offsets_xy) return fail(DTB_E_INVALID, "null pointer");
    if (rows <= 0 || cols <= 0) return fail(DTB_E_INVALID, "image is empty");
    if (n_offsets <= 0) return fail(DTB_E_INVALID, "mask: empty offset set");
    if (binary) {
        int rc = check_method(method, k, r);
        if (rc) return rc;
    }
    const size_t smem = sizeof(int2) * (size_t)n_offsets;
    if (smem > 200 * 1024) return fail(DTB_E_UNSUPPORTED, "mask: %d offsets exceed shared memory", n_offsets);
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(sampled_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return cuda_fail(e, "sampled_kernel attribute");
    }
    dim3 grid((cols + 127) / 128, rows);
    sampled_kernel<<<grid, 128, smem, (cudaStream_t)stream>>>(
        gray, pitch, rows, cols, reinterpret_cast<const int2*>(offsets_xy), n_offsets, mean, std,
        count, binary, tmap, method, k, r);
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? DTB_OK : cuda_fail(e, "sampled_kernel launch");
}

int dtb_histogram(const uint8_t* gray, int64_t pitch, int32_t rows, int32_t cols,
                  uint64_t* hist256, void* stream) {
    if (!gray || !hist256) return fail(DTB_E_INVALID, "null pointer");
    if (rows <= 0 || cols <= 0) return fail(DTB_E_INVALID, "image is empty");
    const int64_t n = (int64_t)rows * cols;
    const int64_t blocks = std::min<int64_t>((n + 255) / 256, (int64_t)num_sms() * 8);
    histogram_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(
        gray, pitch, rows, cols, reinterpret_cast<unsigned long long*>(hist256));
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? DTB_OK : cuda_fail(e, "histogram_kernel launch");
}

int dtb_apply_global(const uint8_t* gray, int64_t pitch, int32_t rows, int32_t cols, int32_t t,
                     uint8_t* out, int64_t out_pitch, void* stream) {
    if (!gray || !out) return fail(DTB_E_INVALID, "null pointer");
    if (t < 0 || t > 255) return fail(DTB_E_INVALID, "threshold: expected an integer in [0, 255], got %d", t);
    if (rows <= 0 || cols <= 0) return fail(DTB_E_INVALID, "image is empty");
    const int64_t n = (int64_t)rows * cols;
    const int64_t blocks = std::min<int64_t>((n + 255) / 256, (int64_t)num_sms() * 16);
    apply_global_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(gray, pitch, rows, cols,
                                                                           t, out, out_pitch);
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? DTB_OK : cuda_fail(e, "apply_global_kernel launch");
}

int dtb_integral_tables(const uint8_t* gray, int64_t pitch, int32_t rows, int32_t cols,
                        int64_t* sum_table, int64_t* sqsum_table, void* stream) {
    if (!gray || !sum_table || !sqsum_table) return fail(DTB_E_INVALID, "null pointer");
    if (rows <= 0 || cols <= 0) return fail(DTB_E_INVALID, "image is empty");
    cudaStream_t st = (cudaStream_t)stream;
    sat_rows_kernel<<<(rows + 1 + 127) / 128, 128, 0, st>>>(gray, pitch, rows, cols, sum_table, sqsum_table);
    sat_cols_kernel<<<(cols + 1 + 127) / 128, 128, 0, st>>>(rows, cols, sum_table, sqsum_table);
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? DTB_OK : cuda_fail(e, "sat kernels launch");
}

}  // extern "C"
