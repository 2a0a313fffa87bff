// dtb_gs.cu -- O(1)-per-pixel GS-mask ("sampled" engine) statistics and binarization
// (SURVEY.md §8 row f1).
//
// Reference: /root/reference/pkg/src/docthresh
//   masks.py:28-64    GS-1..GS-6 membership predicates over a W x W window (r = W // 2)
//   masks.py:98-114   make_mask: the offsets, row-major
//   stats.py:133-163  _accumulate + mean_std_sampled: sums over the IN-BOUNDS offsets,
//                     count = number of in-bounds offsets, then _finish_arrays
//   threshold.py:121-148 binarize(engine="sampled") = that + the Sauvola/Niblack epilogue
//
// Every GS structure is a union of straight segments through the window:
//   R0  centre row  (dx in [-r, r], dy = 0)         C0  centre column (dx = 0)
//   D+  main diagonal (dx = dy)                       D-  anti-diagonal (dx = -dy)
//   RT/RB ring top / bottom rows (dy = -r / +r, full width)
//   RL/RR ring left / right columns (dx = -r / +r, dy in [-r+1, r-1])
//   gs1 = R0 + C0 - c            gs2 = D+ + D- - c          gs3 = R0 + C0 + D+ + D- - 3c
//   gs4 = R0 + D+ + D- - 2c      gs5 = RT + RB + RL + RR + c
//   gs6 = R0 + C0 - c + RT + RB + RL + RR - {(0,-r), (0,r), (-r,0), (r,0)}
// (c = the centre pixel; the subtractions remove the points two segments share).
//
// One CTA owns a TY x TX output tile.  The tile plus an r-pixel halo is staged once in
// shared memory as bytes, zero outside the image, so a segment's in-bounds sum is just its
// sum over the padded tile.  Each segment family is then a 1-D sliding sum along its
// direction: a thread owns 16 consecutive outputs of one line, pays 2r+1 loads to start
// the line and 2 per further output -- O(1) per pixel in W.  Row and diagonal families
// accumulate into a shared (S, Q) array; column families accumulate in the registers of
// the thread that finishes those pixels.  Counts are closed-form clipped segment lengths.
// The epilogue is the reference's fp64 sequence (finish_exact / threshold_exact), so the
// output is bit-identical.  Sums are exact uint32 (|mask| * 255^2 < 2^32 for every W this
// kernel accepts).
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "docthresh_b200.h"
#include "dtb_common.cuh"

namespace dtb {

constexpr int GS_TY = 32;     // output rows per tile
constexpr int GS_TX = 128;    // output columns per tile
constexpr int GS_NT = 256;    // threads per CTA
constexpr int GS_SEG = 16;    // outputs per thread per segment family
constexpr int GS_ACC = GS_TX + 1;  // uint2 row stride of the accumulator (bank-conflict pad)
static_assert(GS_TY * GS_TX == GS_NT * GS_SEG, "one 16-output run per thread");

struct GsParams {
    const uint8_t* in;
    int64_t pitch;
    int rows, cols, r;
    int pw;  // shared-memory pitch of the padded tile (bytes, == 4 mod 8)
    double* mean;
    double* sd;
    int32_t* cnt;
    uint8_t* bin;
    int64_t bin_pitch;
    double* tmap;
    int method;
    double k, rr;
    int row0;       // global row held by buffer row 0 (row bands; 0 for a whole image)
    int in_rows;    // rows in the buffer
    int y0, y1;     // output rows [y0, y1) (global); outputs are stored from row y0
    int nmask;      // |mask| = the count of every unclipped window
    int fast;       // binary only (no tmap / stats): certified fp32 decision
    FastConsts fc;  // for the interior count |mask|
};

__device__ __forceinline__ int clip_len(int a, int b, int n) {
    return max(0, min(b, n - 1) - max(a, 0) + 1);
}

// Row family at tile row offset oy (0 = R0, -r = RT, +r = RB).  Thread: line i = lane,
// outputs j in [16*warp, +16).  Writes (FIRST) or adds into acc.
template <bool FIRST>
__device__ __forceinline__ void gs_rows(const uint8_t* tile, int pw, uint2* acc, int r, int oy) {
    const int i = threadIdx.x & 31, j0 = (threadIdx.x >> 5) * GS_SEG;
    const uint8_t* row = tile + (i + r + oy) * pw;
    uint32_t s = 0, q = 0;
    for (int c = j0; c <= j0 + 2 * r; ++c) {
        const uint32_t v = row[c];
        s += v;
        q += v * v;
    }
    uint2* a = acc + i * GS_ACC + j0;
#pragma unroll
    for (int u = 0; u < GS_SEG; ++u) {
        if (u) {
            const uint32_t e = row[j0 + u + 2 * r], l = row[j0 + u - 1];
            s += e - l;
            q += e * e - l * l;
        }
        if (FIRST) {
            a[u] = make_uint2(s, q);
        } else {
            uint2 o = a[u];
            o.x += s;
            o.y += q;
            a[u] = o;
        }
    }
}

// Diagonal families.  DIR = +1: D+ (tile points (i+d, j+d), d in [0, 2r]); DIR = -1: D-
// (points (i+2r-d, j+d)).  Thread: column j0 = tid & 127, rows [i0, i0+16); output u is
// (i0+u, (j0 + DIR*u) mod 128), so consecutive outputs of a thread lie on one line except
// where the column wraps -- there the line restarts from edge[] (precomputed start sums).
template <int DIR, bool FIRST>
__device__ __forceinline__ void gs_diag(const uint8_t* tile, int pw, uint2* acc, const uint2* edge,
                                        int r) {
    const int j0 = threadIdx.x & (GS_TX - 1), i0 = (threadIdx.x >> 7) * GS_SEG;
    uint32_t s = 0, q = 0;
    for (int d = 0; d <= 2 * r; ++d) {
        const uint32_t v = DIR > 0 ? tile[(i0 + d) * pw + j0 + d] : tile[(i0 + 2 * r - d) * pw + j0 + d];
        s += v;
        q += v * v;
    }
#pragma unroll
    for (int u = 0; u < GS_SEG; ++u) {
        const int i = i0 + u, j = (j0 + DIR * u) & (GS_TX - 1);
        if (u) {
            if (j == (DIR > 0 ? 0 : GS_TX - 1)) {
                const uint2 e = edge[i];
                s = e.x;
                q = e.y;
            } else {
                uint32_t e, l;
                if (DIR > 0) {
                    e = tile[(i + 2 * r) * pw + j + 2 * r];
                    l = tile[(i - 1) * pw + j - 1];
                } else {
                    e = tile[(i + 2 * r) * pw + j];
                    l = tile[(i - 1) * pw + j + 2 * r + 1];
                }
                s += e - l;
                q += e * e - l * l;
            }
        }
        uint2* a = acc + i * GS_ACC + j;
        if (FIRST) {
            *a = make_uint2(s, q);
        } else {
            uint2 o = *a;
            o.x += s;
            o.y += q;
            *a = o;
        }
    }
}

// Column family at tile column offset ox with half-length h (C0: ox = 0, h = r; RL/RR:
// ox = -r/+r, h = r-1).  Thread: column j, rows [i0, i0+16) -- the finishing layout, so the
// sums stay in registers.
__device__ __forceinline__ void gs_cols(const uint8_t* tile, int pw, int r, int ox, int h, int j,
                                        int i0, uint32_t (&vs)[GS_SEG], uint32_t (&vq)[GS_SEG]) {
    const uint8_t* col = tile + j + r + ox;
    uint32_t s = 0, q = 0;
    for (int d = i0 + r - h; d <= i0 + r + h; ++d) {
        const uint32_t v = col[d * pw];
        s += v;
        q += v * v;
    }
#pragma unroll
    for (int u = 0; u < GS_SEG; ++u) {
        if (u) {
            const uint32_t e = col[(i0 + u + r + h) * pw], l = col[(i0 + u - 1 + r - h) * pw];
            s += e - l;
            q += e * e - l * l;
        }
        vs[u] += s;
        vq[u] += q;
    }
}

// Remove the points two segments share from (S, Q) (out-of-image pixels are 0 in the tile).
template <int GS>
__device__ __forceinline__ void gs_overlaps(const uint8_t* tile, int pw, int r, int i, int j,
                                            uint32_t f, uint32_t& S, uint32_t& Q) {
    if (GS == 1 || GS == 2) { S -= f; Q -= f * f; }
    if (GS == 3) { S -= 3 * f; Q -= 3 * f * f; }
    if (GS == 4) { S -= 2 * f; Q -= 2 * f * f; }
    if (GS == 5) { S += f; Q += f * f; }
    if (GS == 6) {
        const uint32_t t0 = tile[i * pw + j + r], t1 = tile[(i + 2 * r) * pw + j + r];
        const uint32_t t2 = tile[(i + r) * pw + j], t3 = tile[(i + r) * pw + j + 2 * r];
        S -= f + t0 + t1 + t2 + t3;
        Q -= f * f + t0 * t0 + t1 * t1 + t2 * t2 + t3 * t3;
    }
}

// Interior tile, binary only: every count is |mask|, so the per-launch fp32 constants apply
// to all 16 pixels; uncertain pixels replay the reference fp64 sequence (exact_white).
template <int GS, int METHOD>
__device__ __forceinline__ void gs_fast_interior(const GsParams& p, const uint8_t* tile,
                                                 const uint2* acc, const uint32_t (&vs)[GS_SEG],
                                                 const uint32_t (&vq)[GS_SEG], int i0, int j,
                                                 int tx0, int ty0) {
    const int r = p.r, pw = p.pw;
    uint8_t* out = p.bin + (int64_t)(ty0 + i0 - p.y0) * p.bin_pitch + tx0 + j;
#pragma unroll
    for (int u = 0; u < GS_SEG; ++u) {
        const int i = i0 + u;
        const uint2 a = acc[i * GS_ACC + j];
        uint32_t S = a.x + vs[u], Q = a.y + vq[u];
        const uint32_t f = tile[(i + r) * pw + j + r];
        gs_overlaps<GS>(tile, pw, r, i, j, f, S, Q);
        const float d = fast_diff<METHOD, false>(S, Q, f, p.fc.N, p.fc.cA, p.fc.cC, p.fc.a, p.fc.c);
        const uint32_t white = fabsf(d) >= p.fc.tol
                                   ? (d < 0.f ? 0u : 255u)
                                   : exact_white(S, Q, (double)p.fc.N, f, METHOD, p.k, p.rr);
        out[(int64_t)u * p.bin_pitch] = (uint8_t)white;
    }
}

template <int GS>
__global__ void __launch_bounds__(GS_NT) gs_kernel(GsParams p) {
    extern __shared__ __align__(16) uint8_t gs_smem[];
    const int r = p.r, pw = p.pw;
    const int PR = GS_TY + 2 * r, PC = GS_TX + 2 * r;
    uint2* acc = reinterpret_cast<uint2*>(gs_smem);
    uint2* edge_p = acc + GS_TY * GS_ACC;
    uint2* edge_m = edge_p + GS_TY;
    uint8_t* tile = reinterpret_cast<uint8_t*>(edge_m + GS_TY);

    const int ty0 = p.y0 + blockIdx.y * GS_TY, tx0 = blockIdx.x * GS_TX;
    const uint8_t* in0 = p.in - (int64_t)p.row0 * p.pitch;  // global row g at in0 + g * pitch
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    // Interior tile: every window of every output is unclipped (count = |mask|), and the
    // staged rows are followed by at least one more image row (the word loads below may run
    // up to 7 bytes past a staged row's end).
    const bool interior = ty0 >= r && ty0 + GS_TY + r <= p.rows &&
                          ty0 + GS_TY + r < p.row0 + p.in_rows && ty0 + GS_TY <= p.y1 &&
                          tx0 >= r && tx0 + GS_TX + r <= p.cols;
    // Stage the padded tile (zero outside the image).
    if (interior) {
        // aligned 4-byte loads, realigned with a funnel shift, 4-byte shared stores
        const int nw = (PC + 3) >> 2;
        for (int pr = warp; pr < PR; pr += GS_NT / 32) {
            const uintptr_t ad = reinterpret_cast<uintptr_t>(in0 + (int64_t)(ty0 - r + pr) * p.pitch +
                                                             (tx0 - r));
            const uint32_t* w = reinterpret_cast<const uint32_t*>(ad & ~(uintptr_t)3);
            const uint32_t sh = (uint32_t)(ad & 3) * 8u;
            for (int kw = lane; kw < nw; kw += 32) {
                const uint32_t lo = __ldg(w + kw), hi = __ldg(w + kw + 1);
                *reinterpret_cast<uint32_t*>(tile + pr * pw + 4 * kw) = __funnelshift_r(lo, hi, sh);
            }
        }
    } else {
        for (int pr = warp; pr < PR; pr += GS_NT / 32) {
            const int gy = ty0 - r + pr;
            const bool rowok = gy >= 0 && gy < p.rows;
            const uint8_t* src = in0 + (int64_t)gy * p.pitch;
            for (int pc = lane; pc < PC; pc += 32) {
                const int gx = tx0 - r + pc;
                tile[pr * pw + pc] = (rowok && gx >= 0 && gx < p.cols) ? __ldg(src + gx) : 0;
            }
        }
    }
    __syncthreads();

    constexpr bool HAS_DIAG = GS == 2 || GS == 3 || GS == 4;
    constexpr bool HAS_R0 = GS == 1 || GS == 3 || GS == 4 || GS == 6;
    constexpr bool HAS_RING = GS == 5 || GS == 6;
    if (HAS_DIAG && threadIdx.x < 2 * GS_TY) {
        // Line-start sums where a thread's diagonal run wraps: D+ at column 0, D- at 127.
        const int i = threadIdx.x & (GS_TY - 1);
        uint32_t s = 0, q = 0;
        if (threadIdx.x < GS_TY) {
            for (int d = 0; d <= 2 * r; ++d) {
                const uint32_t v = tile[(i + d) * pw + d];
                s += v;
                q += v * v;
            }
            edge_p[i] = make_uint2(s, q);
        } else {
            for (int d = 0; d <= 2 * r; ++d) {
                const uint32_t v = tile[(i + 2 * r - d) * pw + GS_TX - 1 + d];
                s += v;
                q += v * v;
            }
            edge_m[i] = make_uint2(s, q);
        }
    }
    if (HAS_R0) gs_rows<true>(tile, pw, acc, r, 0);
    if (HAS_RING) {
        if (HAS_R0) gs_rows<false>(tile, pw, acc, r, -r);
        else gs_rows<true>(tile, pw, acc, r, -r);
        gs_rows<false>(tile, pw, acc, r, r);
    }
    if (HAS_DIAG) {
        __syncthreads();  // edge sums visible
        if (HAS_R0) gs_diag<1, false>(tile, pw, acc, edge_p, r);
        else gs_diag<1, true>(tile, pw, acc, edge_p, r);
        __syncthreads();  // D+ and D- runs of different threads touch the same acc cells
        gs_diag<-1, false>(tile, pw, acc, edge_m, r);
    }
    const int j = threadIdx.x & (GS_TX - 1), i0 = (threadIdx.x >> 7) * GS_SEG;
    uint32_t vs[GS_SEG], vq[GS_SEG];
#pragma unroll
    for (int u = 0; u < GS_SEG; ++u) vs[u] = vq[u] = 0;
    if (GS == 1 || GS == 3 || GS == 6) gs_cols(tile, pw, r, 0, r, j, i0, vs, vq);
    if (HAS_RING) {
        gs_cols(tile, pw, r, -r, r - 1, j, i0, vs, vq);
        gs_cols(tile, pw, r, r, r - 1, j, i0, vs, vq);
    }
    __syncthreads();  // row / diagonal accumulators complete
    if (p.fast && interior) {  // the common case: unclipped windows, binary output only
        if (p.method == DTB_METHOD_SAUVOLA)
            gs_fast_interior<GS, DTB_METHOD_SAUVOLA>(p, tile, acc, vs, vq, i0, j, tx0, ty0);
        else
            gs_fast_interior<GS, DTB_METHOD_NIBLACK>(p, tile, acc, vs, vq, i0, j, tx0, ty0);
        return;
    }
    // Fold the column families into this thread's own accumulator cells.
#pragma unroll
    for (int u = 0; u < GS_SEG; ++u) {
        uint2* a = acc + (i0 + u) * GS_ACC + j;
        uint2 o = *a;
        o.x += vs[u];
        o.y += vq[u];
        *a = o;
    }

    const int x = tx0 + j;
    if (x >= p.cols) return;
#pragma unroll 1
    for (int u = 0; u < GS_SEG; ++u) {
        const int i = i0 + u, y = ty0 + i;
        if (y >= p.y1) break;
        const uint2 a = acc[i * GS_ACC + j];
        uint32_t S = a.x, Q = a.y;
        const uint32_t f = tile[(i + r) * pw + j + r];
        const int rows = p.rows, cols = p.cols;
        gs_overlaps<GS>(tile, pw, r, i, j, f, S, Q);
        int n = p.nmask;
        if (!interior) {  // closed-form clipped segment lengths
            const int cx = clip_len(x - r, x + r, cols), cy = clip_len(y - r, y + r, rows);
            n = 0;
            if (GS == 1 || GS == 3 || GS == 6) n += cx + cy;  // R0 + C0
            if (GS == 4) n += cx;
            if (HAS_DIAG) {
                const int dp = min(r, min(cols - 1 - x, rows - 1 - y)) - max(-r, max(-x, -y)) + 1;
                const int dm = min(r, min(cols - 1 - x, y)) - max(-r, max(-x, y - rows + 1)) + 1;
                n += dp + dm;
            }
            if (HAS_RING) {
                const int ch = clip_len(y - r + 1, y + r - 1, rows);
                n += (y - r >= 0 ? cx : 0) + (y + r < rows ? cx : 0) + (x - r >= 0 ? ch : 0) +
                     (x + r < cols ? ch : 0);
            }
            if (GS == 1 || GS == 2) n -= 1;
            if (GS == 3) n -= 3;
            if (GS == 4) n -= 2;
            if (GS == 5) n += 1;
            if (GS == 6)
                n -= 1 + (y - r >= 0) + (y + r < rows) + (x - r >= 0) + (x + r < cols);
        }
        if (p.fast) {
            // binary only: certified fp32 decision, fp64 replay for the uncertain pixels
            const uint32_t un = (uint32_t)n;
            float d;
            if (p.method == DTB_METHOD_SAUVOLA)
                d = un == p.fc.N ? fast_diff<DTB_METHOD_SAUVOLA, false>(S, Q, f, un, p.fc.cA, p.fc.cC, p.fc.a, p.fc.c)
                                 : fast_diff<DTB_METHOD_SAUVOLA, true>(S, Q, f, un, p.fc.cA, p.fc.cC, p.fc.a, p.fc.c);
            else
                d = un == p.fc.N ? fast_diff<DTB_METHOD_NIBLACK, false>(S, Q, f, un, p.fc.cA, p.fc.cC, p.fc.a, p.fc.c)
                                 : fast_diff<DTB_METHOD_NIBLACK, true>(S, Q, f, un, p.fc.cA, p.fc.cC, p.fc.a, p.fc.c);
            const uint32_t white = fabsf(d) >= p.fc.tol ? (d < 0.f ? 0u : 255u)
                                                        : exact_white(S, Q, (double)n, f, p.method, p.k, p.rr);
            p.bin[(int64_t)(y - p.y0) * p.bin_pitch + x] = (uint8_t)white;
            continue;
        }
        double mean, sd;
        finish_exact((double)S, (double)Q, (double)n, mean, sd);
        const int64_t idx = (int64_t)(y - p.y0) * cols + x;
        if (p.mean) p.mean[idx] = mean;
        if (p.sd) p.sd[idx] = sd;
        if (p.cnt) p.cnt[idx] = n;
        if (p.bin) {
            const double t = threshold_exact(mean, sd, p.method, p.k, p.rr);
            p.bin[(int64_t)(y - p.y0) * p.bin_pitch + x] = ((double)f < t) ? 0 : 255;
            if (p.tmap) p.tmap[idx] = t;
        }
    }
}

static int gs_pitch(int r) {
    const int pc = GS_TX + 2 * r;
    return ((pc + 7) & ~7) + 4;  // == 4 (mod 8): consecutive tile rows hit distinct banks
}

size_t gs_smem_bytes(int r) {
    return sizeof(uint2) * (GS_TY * GS_ACC + 2 * GS_TY) + (size_t)(GS_TY + 2 * r) * gs_pitch(r);
}

// Shared launcher: p has the image/band fields, outputs and method set.
static int gs_run(GsParams p, int structure, int win, void* stream) {
    if (structure < DTB_GS1 || structure > DTB_GS6)
        return fail(DTB_E_INVALID, "structure: expected DTB_GS1..DTB_GS6, got %d", structure);
    if (win < 3 || win % 2 == 0) return fail(DTB_E_INVALID, "window: must be an odd integer >= 3, got %d", win);
    if (p.bin && p.method != DTB_METHOD_SAUVOLA && p.method != DTB_METHOD_NIBLACK)
        return fail(DTB_E_INVALID, "method: unknown code %d", p.method);
    // the same parameter checks as dtb_binarize (threshold.py:40-52): k_sauvola > 0, r > 0
    if (p.bin && p.method == DTB_METHOD_SAUVOLA && !(p.k > 0.0))
        return fail(DTB_E_INVALID, "k_sauvola: must be > 0, got %g", p.k);
    if (p.bin && !(p.rr > 0.0)) return fail(DTB_E_INVALID, "r: must be > 0, got %g", p.rr);
    const int rad = win / 2;
    const size_t smem = gs_smem_bytes(rad);
    if (smem > DTB_GS_MAX_SMEM)
        return fail(DTB_E_UNSUPPORTED, "window %d too large for the tiled GS kernel", win);
    p.r = rad;
    p.pw = gs_pitch(rad);
    static const int mul[7] = {0, 2, 2, 4, 3, 4, 6};  // |mask| = mul*W - sub (masks.py:5-12)
    static const int sub[7] = {0, 1, 1, 3, 2, 3, 9};
    p.nmask = mul[structure] * win - sub[structure];
    if (p.bin && !p.tmap && !p.mean && !p.sd && !p.cnt) {
        p.fast = 1;
        p.fc = fast_constants(p.method, p.k, p.rr, (double)p.nmask);
    }
    if (p.y1 <= p.y0) return DTB_OK;
    const dim3 grid((p.cols + GS_TX - 1) / GS_TX, (p.y1 - p.y0 + GS_TY - 1) / GS_TY);
    cudaStream_t st = (cudaStream_t)stream;
    cudaError_t e = cudaSuccess;
#define DTB_GS_LAUNCH(G)                                                                      \
    case G: {                                                                                 \
        e = cudaFuncSetAttribute(gs_kernel<G>, cudaFuncAttributeMaxDynamicSharedMemorySize,  \
                                 (int)smem);                                                  \
        if (e == cudaSuccess) gs_kernel<G><<<grid, GS_NT, smem, st>>>(p);                     \
        break;                                                                                \
    }
    switch (structure) {
        DTB_GS_LAUNCH(1)
        DTB_GS_LAUNCH(2)
        DTB_GS_LAUNCH(3)
        DTB_GS_LAUNCH(4)
        DTB_GS_LAUNCH(5)
        DTB_GS_LAUNCH(6)
    }
#undef DTB_GS_LAUNCH
    if (e == cudaSuccess) e = cudaGetLastError();
    return e == cudaSuccess ? DTB_OK : cuda_fail(e, "gs_kernel launch");
}

}  // namespace dtb

using namespace dtb;

extern "C" {

int dtb_gs_stats(const uint8_t* gray, int64_t pitch, int32_t rows, int32_t cols, int32_t structure,
                 int32_t win, double* mean, double* std_, int32_t* count, uint8_t* binary,
                 int64_t binary_pitch, double* tmap, int32_t method, double k, double r,
                 void* stream) {
    if (!gray) return fail(DTB_E_INVALID, "null pointer");
    if (rows <= 0 || cols <= 0) return fail(DTB_E_INVALID, "image is empty");
    if (!binary && !mean && !std_ && !count) return fail(DTB_E_INVALID, "no output requested");
    if (pitch < cols || (binary && binary_pitch < cols))
        return fail(DTB_E_INVALID, "pitch smaller than the row width");
    GsParams p{};
    p.in = gray; p.pitch = pitch; p.rows = rows; p.cols = cols;
    p.row0 = 0; p.in_rows = rows; p.y0 = 0; p.y1 = rows;
    p.mean = mean; p.sd = std_; p.cnt = count; p.bin = binary; p.bin_pitch = binary_pitch;
    p.tmap = tmap; p.method = method; p.k = k; p.rr = r;
    return gs_run(p, structure, win, stream);
}

int dtb_gs_band(const uint8_t* gray, int64_t pitch, int32_t in_rows, int32_t cols,
                int32_t row0_global, int32_t rows_global, int32_t out_row_begin,
                int32_t out_row_end, int32_t structure, int32_t win, uint8_t* binary,
                int64_t binary_pitch, int32_t method, double k, double r, void* stream) {
    if (!gray || !binary) return fail(DTB_E_INVALID, "null image pointer");
    if (cols <= 0 || rows_global <= 0) return fail(DTB_E_INVALID, "image is empty");
    if (pitch < cols || binary_pitch < cols) return fail(DTB_E_INVALID, "pitch smaller than the row width");
    if (out_row_begin < 0 || out_row_end > rows_global || out_row_begin > out_row_end)
        return fail(DTB_E_INVALID, "rows: output rows [%d,%d) outside image of %d rows",
                    out_row_begin, out_row_end, rows_global);
    const int rad = win / 2;
    const int need0 = std::max(out_row_begin - rad, 0);
    const int need1 = std::min(out_row_end + rad, (int)rows_global);
    if (out_row_end > out_row_begin && (need0 < row0_global || need1 > row0_global + in_rows))
        return fail(DTB_E_INVALID, "rows: band needs global rows [%d,%d) but buffer holds [%d,%d)",
                    need0, need1, row0_global, row0_global + in_rows);
    GsParams p{};
    p.in = gray; p.pitch = pitch; p.rows = rows_global; p.cols = cols;
    p.row0 = row0_global; p.in_rows = in_rows; p.y0 = out_row_begin; p.y1 = out_row_end;
    p.bin = binary; p.bin_pitch = binary_pitch; p.method = method; p.k = k; p.rr = r;
    return gs_run(p, structure, win, stream);
}

}  // extern "C"
