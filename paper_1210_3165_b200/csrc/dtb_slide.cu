// dtb_slide.cu -- the fast fused sliding-sum binarization kernel (K2) for sm_100a.
//
// Replaces, for the binary output, threshold.py:121-148 -> stats.py:166-191 ->
// stats.py:50-54 -> threshold.py:143-147 of the reference, bit for bit.
//
// Layout.  One CTA owns a vertical strip and a band of output rows.  Strip s produces output
// columns [X0, X0+TW), X0 = s*TW (TW = 0 mod 32).  Its column index space i <-> image column
// xc0 + i with xc0 = X0 - rx - alpha = 0 mod 16 (alpha = (-rx) mod 16), i in [0, NC),
// NC = V*NT (V = 16 or 32 columns per thread).  Thread t owns columns [Vt, Vt+V): it keeps
// their exact running column sums
//   cS[j] = sum f, cQ[j] = sum f^2   over rows [y-r, y+r] (clipped)
// in registers and slides them down the band (+ row y+r, - row y-r-1, 2 LDG.128 each).
// Per output row the CTA forms the inclusive horizontal prefix P of the column sums in shared
// memory (uint32, exact mod 2^32 -- every true window sum is < 2^32 for W <= 255): per-thread
// totals -> warp shuffle scan -> cross-warp totals -> per-thread running prefix, stored as
// logical word k = P[k-1] (so each thread writes 8 aligned 16-byte chunks).  Shared memory is
// padded one 16-byte chunk per 8 (chunk L lives at L + L/8), which makes both the per-thread
// stores and the run loads bank-conflict free.  Output x = X0 + Vt + j has window indices
// [alpha+Vt+j, alpha+2rx+Vt+j]:  S = P[alpha+2rx+Vt+j] - P[alpha-1+Vt+j];
// the two runs are misaligned by (-rx) mod 4 and (rx+1) mod 4 words, resolved at compile time
// (RXM4 template) so both are read with LDS.128.
//
// Decision.  The threshold is formed in fp32 from the EXACT integer D = n*Q - S^2 (>= 0, no
// cancellation; n = N = W^2 for unclipped windows, n = ny*nx at image borders):
//   Sauvola  t = S * ((1-k)/n + k/(R n^2) * sqrt(D))        Niblack  t = S/n + k/n * sqrt(D)
// The host bounds |t_fp32 - t_reference| (fp32 error of this sequence + the reference's own
// fp64 rounding of var/std) by `tol`.  A pixel with |f - t_fp32| >= tol is decided by the sign;
// if any of a thread's 32 pixels is within tol (~1e-5 of pixels), the thread replays the
// reference fp64 sequence for those pixels (out of line, rare).
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <mutex>
#include <tuple>

#include "docthresh_b200.h"
#include "dtb_common.cuh"
#include "dtb_slide.cuh"
#include "dtb_async.cuh"

#ifndef DTB_WS_DEFAULT
#define DTB_WS_DEFAULT 2  // 0 classic, 1 always warp-specialized, 2 auto
#endif

namespace dtb {

// Guarded byte-wise load of 4 words (image edges / unaligned buffers); out of line.
__device__ __noinline__ uint4 ldg16_slow(const uint8_t* rowp, int c0, int cols) {
    uint32_t w[4];
    for (int q = 0; q < 4; ++q) {
        uint32_t v = 0;
        for (int b = 0; b < 4; ++b) {
            const int c = c0 + 4 * q + b;
            if (c >= 0 && c < cols) v |= (uint32_t)__ldg(rowp + c) << (8 * b);
        }
        w[q] = v;
    }
    return make_uint4(w[0], w[1], w[2], w[3]);
}

__device__ __forceinline__ uint4 ldg16(const uint8_t* rowp, int c0, int cols, bool vec) {
    // 16 bytes of one image row at columns [c0, c0+16), zeros outside [0, cols); c0 = 0 mod 16.
    if (c0 >= 0 && c0 + 16 <= cols) {
        if (vec) return __ldg(reinterpret_cast<const uint4*>(rowp + c0));
    } else if (c0 + 16 <= 0 || c0 >= cols) {
        return make_uint4(0, 0, 0, 0);
    }
    return ldg16_slow(rowp, c0, cols);
}

__device__ __forceinline__ void ldg32B(const uint8_t* rowp, int c0, int cols, bool vec,
                                       uint32_t (&w)[8]) {
    const uint4 a = ldg16(rowp, c0, cols, vec);
    const uint4 b = ldg16(rowp, c0 + 16, cols, vec);
    w[0] = a.x; w[1] = a.y; w[2] = a.z; w[3] = a.w;
    w[4] = b.x; w[5] = b.y; w[6] = b.z; w[7] = b.w;
}

template <int NW>
__device__ __forceinline__ uint32_t byte_at(const uint32_t (&w)[NW], int j) {
    return __byte_perm(w[j >> 2], 0u, 0x4440 | (j & 3));
}


// padded shared-memory position (in words) of logical chunk L
__device__ __forceinline__ int pchunk_word(int L) { return 4 * (L + (L >> 3)); }


// sqrt_ftz, rcp_ftz, fast_diff, exact_white: dtb_common.cuh


// fp32-epilogue audit (dtb_set_fp32_audit): when set, the replay path counts
// [0] pixels replayed in fp64 (|f - t32| < tol), [1] pixels whose plain fp32 sign would have
// flipped the reference's decision, [2] max |f - t_fp64| over those (float bits).
__device__ unsigned long long* g_fp32_audit = nullptr;

// Rare path, out of line: re-decide this thread's 32 pixels, the uncertain ones (|f - t32| < tol)
// with the reference fp64 sequence.  S/Q are read back from the shared prefix (valid until the next
// row's first barrier); corrected bytes are written after the vector stores (program order).
template <int METHOD>
__device__ __noinline__ void fix_uncertain(const uint32_t* sPS, const uint32_t* sPQ, int a_word,
                                           int b_word, const uint8_t* frow, uint8_t* orow,
                                           int xo, int nv, int cols, int ny, int r, uint32_t N,
                                           float cA, float cC, float a, float c, float tol,
                                           double k, double rr) {
    for (int j = 0; j < nv; ++j) {
        const int x = xo + j;
        if (x < 0 || x >= cols) continue;
        const int la = a_word + j, lb = b_word + j;  // logical words
        const int pa = pchunk_word(la >> 2) + (la & 3), pb = pchunk_word(lb >> 2) + (lb & 3);
        const uint32_t S = sPS[pb] - sPS[pa];
        const uint32_t Q = sPQ[pb] - sPQ[pa];
        const uint32_t f = frow[x];
        const int nx = min(x + r, cols - 1) - max(x - r, 0) + 1;
        const uint32_t n = (uint32_t)(ny * nx);
        const float d = (n == N) ? fast_diff<METHOD, false>(S, Q, f, n, cA, cC, a, c)
                                 : fast_diff<METHOD, true>(S, Q, f, n, cA, cC, a, c);
        // rewrite every pixel of the thread: the caller's decision may have used the other
        // (border) constant set, so its certified set can differ from this one's
        if (fabsf(d) >= tol) {
            orow[x] = d < 0.f ? 0 : 255;
            continue;
        }
        const uint32_t white = exact_white(S, Q, (double)n, f, METHOD, k, rr);
        orow[x] = (uint8_t)white;
        if (unsigned long long* audit = g_fp32_audit) {
            atomicAdd(&audit[0], 1ull);
            if (white != (d < 0.f ? 0u : 0xFFu)) {
                double mean, sd;
                finish_exact((double)S, (double)Q, (double)n, mean, sd);
                const float gap = (float)fabs((double)f - threshold_exact(mean, sd, METHOD, k, rr));
                atomicAdd(&audit[1], 1ull);
                atomicMax(&audit[2], (unsigned long long)__float_as_uint(gap));
            }
        }
    }
}

// One row of 32 outputs for this thread: S/Q from the shared prefix, f from global (row y),
// fp32 certified decision, 8-byte stores.  Returns whether any pixel was uncertain.
// aw/bw: shared-memory word addresses of the 9 chunks of the A and B runs (precomputed).
template <int V, int RXM4, int METHOD, bool BORDER>
__device__ __forceinline__ bool row_outputs(const uint32_t* sPS, const uint32_t* sPQ,
                                            const int (&aw)[V / 4 + 1], const int (&bw)[V / 4 + 1],
                                            const uint8_t* fsm, uint32_t (&ow)[V / 4], int xo,
                                            int cols, int ny, int r, const SlideParams& p) {
    constexpr int MA = (4 - RXM4) & 3;  // misalignment (words) of the A run
    constexpr int MB = (RXM4 + 1) & 3;  // misalignment (words) of the B run
    uint32_t fw[V / 4];  // row y pixel values of this thread's V outputs, from the shared stage
#pragma unroll
    for (int q = 0; q < V / 16; ++q) {
        const uint4 v = *reinterpret_cast<const uint4*>(fsm + 16 * q);
        fw[4 * q] = v.x; fw[4 * q + 1] = v.y; fw[4 * q + 2] = v.z; fw[4 * q + 3] = v.w;
    }
    float mind = 3.0e38f;
#pragma unroll
    for (int g = 0; g < V / 8; ++g) {  // groups of 8 outputs
        uint32_t S8[8], Q8[8];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const uint32_t* sp = h ? sPQ : sPS;
            uint32_t A[12], B[12];
#pragma unroll
            for (int q = 0; q < 3; ++q) {
                if (q < 2 || MA) {
                    DTB_CHECK(aw[2 * g + q] >= 0 && aw[2 * g + q] + 4 <= slide_padded_words(p.PL));
                    const uint4 v = *reinterpret_cast<const uint4*>(sp + aw[2 * g + q]);
                    A[4 * q] = v.x; A[4 * q + 1] = v.y; A[4 * q + 2] = v.z; A[4 * q + 3] = v.w;
                }
                if (q < 2 || MB) {
                    DTB_CHECK(bw[2 * g + q] >= 0 && bw[2 * g + q] + 4 <= slide_padded_words(p.PL));
                    const uint4 v = *reinterpret_cast<const uint4*>(sp + bw[2 * g + q]);
                    B[4 * q] = v.x; B[4 * q + 1] = v.y; B[4 * q + 2] = v.z; B[4 * q + 3] = v.w;
                }
            }
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const uint32_t v = B[MB + j] - A[MA + j];
                if (h) Q8[j] = v; else S8[j] = v;
            }
        }
        const uint32_t fa = fw[2 * g], fb = fw[2 * g + 1];
        float d[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const uint32_t f = __byte_perm(j < 4 ? fa : fb, 0u, 0x4440 | (j & 3));
            uint32_t n = p.N;
            if (BORDER) {
                const int x = xo + 8 * g + j;
                n = (uint32_t)(ny * (min(x + r, cols - 1) - max(x - r, 0) + 1));
            }
            d[j] = fast_diff<METHOD, BORDER>(S8[j], Q8[j], f, n, p.cA, p.cC, p.a, p.c);
            mind = fminf(mind, fabsf(d[j]));
        }
        // byte = 0x00 if f < t (diff negative) else 0xFF: sign-replicate the diff's top byte
        ow[2 * g] = ~prmt(prmt(__float_as_uint(d[0]), __float_as_uint(d[1]), 0xFBFB),
                          prmt(__float_as_uint(d[2]), __float_as_uint(d[3]), 0xFBFB), 0x5410);
        ow[2 * g + 1] = ~prmt(prmt(__float_as_uint(d[4]), __float_as_uint(d[5]), 0xFBFB),
                              prmt(__float_as_uint(d[6]), __float_as_uint(d[7]), 0xFBFB), 0x5410);
    }
    return mind < p.tol;
}



// TMAP variant of row_outputs: every pixel runs the reference fp64 epilogue (t_exact_fast,
// bit-exact), its threshold goes to the fp64 map row trow[0..V) and its byte to ow.
template <int V, int RXM4, int METHOD, bool BORDER, bool RP2>
__device__ __forceinline__ void row_outputs_tmap(const uint32_t* sPS, const uint32_t* sPQ,
                                                 const int (&aw)[V / 4 + 1], const int (&bw)[V / 4 + 1],
                                                 const uint8_t* fsm, uint32_t (&ow)[V / 4], double* trow,
                                                 int xo, int cols, int ny, int r, const SlideParams& p,
                                                 double rnN, double rinv) {
    constexpr int MA = (4 - RXM4) & 3;
    constexpr int MB = (RXM4 + 1) & 3;
    uint32_t fw[V / 4];
#pragma unroll
    for (int q = 0; q < V / 16; ++q) {
        const uint4 v = *reinterpret_cast<const uint4*>(fsm + 16 * q);
        fw[4 * q] = v.x; fw[4 * q + 1] = v.y; fw[4 * q + 2] = v.z; fw[4 * q + 3] = v.w;
    }
    const bool full = xo + V <= cols;
#pragma unroll
    for (int g = 0; g < V / 8; ++g) {
        uint32_t S8[8], Q8[8];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const uint32_t* sp = h ? sPQ : sPS;
            uint32_t A[12], B[12];
#pragma unroll
            for (int q = 0; q < 3; ++q) {
                if (q < 2 || MA) {
                    const uint4 v = *reinterpret_cast<const uint4*>(sp + aw[2 * g + q]);
                    A[4 * q] = v.x; A[4 * q + 1] = v.y; A[4 * q + 2] = v.z; A[4 * q + 3] = v.w;
                }
                if (q < 2 || MB) {
                    const uint4 v = *reinterpret_cast<const uint4*>(sp + bw[2 * g + q]);
                    B[4 * q] = v.x; B[4 * q + 1] = v.y; B[4 * q + 2] = v.z; B[4 * q + 3] = v.w;
                }
            }
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const uint32_t v = B[MB + j] - A[MA + j];
                if (h) Q8[j] = v; else S8[j] = v;
            }
        }
        uint32_t bytes[2] = {0u, 0u};
        double t8[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const uint32_t f = __byte_perm(fw[2 * g + (j >> 2)], 0u, 0x4440 | (j & 3));
            uint32_t n = p.N;
            double rn = rnN;
            if (BORDER) {
                const int x = xo + 8 * g + j;
                n = (uint32_t)(ny * (min(x + r, cols - 1) - max(x - r, 0) + 1));
                if (n != p.N) rn = __drcp_rn((double)n);
            }
            const double t = t_exact_fast<RP2>(S8[j], Q8[j], n, rn, METHOD, p.k, p.rr, rinv);
            t8[j] = t;
            if (!((double)f < t)) bytes[j >> 2] |= 0xFFu << (8 * (j & 3));
        }
        ow[2 * g] = bytes[0];
        ow[2 * g + 1] = bytes[1];
        if (full) {
#pragma unroll
            for (int j = 0; j < 8; j += 2)
                __stcs(reinterpret_cast<double2*>(trow + 8 * g + j), make_double2(t8[j], t8[j + 1]));
        } else {
#pragma unroll
            for (int j = 0; j < 8; ++j)
                if (xo + 8 * g + j < cols) trow[8 * g + j] = t8[j];
        }
    }
}

// register budget: V=16 fits 128 registers without spills (4 CTAs x 4 warps per SM)
// V = 16: 128 registers (4 CTAs x 4 warps per SM); the plain Niblack variant fits 96 without
// spills, which makes room for a fifth 4-warp CTA (C3 0.670 -> 0.640 ms; the Sauvola variants
// measured 1-2% slower at 96 / 104 / 112 on C5 and C2 and stay at 128)
#ifndef DTB_SLIDE_MAXREG16_NIBLACK
#define DTB_SLIDE_MAXREG16_NIBLACK 96
#endif

// MX = method code | 4 for the segmented-input variant (dtb_binarize_segments)
template <int V, int RXM4, int MX>
__global__ void __maxnreg__(V == 32 ? 255 : (MX == DTB_METHOD_NIBLACK ? DTB_SLIDE_MAXREG16_NIBLACK : 128))
slide_kernel(SlideParams p) {
    constexpr int METHOD = MX & 3;
    constexpr bool SEG = (MX & 4) != 0;
    constexpr bool TMAP = (MX & 8) != 0;  // also write the fp64 threshold map (exact per pixel)
    constexpr int MA = (4 - RXM4) & 3;
    constexpr int MB = (RXM4 + 1) & 3;
    constexpr int NS = SLIDE_STAGES;
    extern __shared__ __align__(128) uint32_t sm[];
    const int NCp = slide_padded_words(p.PL);
    uint32_t* sPS = sm;
    uint32_t* sPQ = sm + NCp;
    uint32_t* sWS = sm + 2 * NCp;  // per-warp totals (8 + 8 words)
    uint32_t* sWQ = sWS + 8;
    uint64_t* full = reinterpret_cast<uint64_t*>(sWS + 16);   // NS barriers
    uint64_t* empty = full + NS;                              // NS barriers
    uint8_t* ring = reinterpret_cast<uint8_t*>(empty + NS);   // NS stages x (E, O, F) x NC
    const int nwarps = (blockDim.x + 31) >> 5;

    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const uint8_t* in = p.in + (int64_t)blockIdx.z * p.img_stride;
    const int X0 = (int)blockIdx.x * p.TW;
    // word RA = alpha + (x - X0) of a prefix array holds P(x - rx - 1), word RA + 2rx + 1 holds
    // P(x + rx).  Halo layout: column index 0 is image column X0 - rx - alpha.  Edge-padded
    // layout (p.pad > 0, one strip): column index 0 is image column X0 = 0 and the column threads
    // write their prefix p.pad words further right.
    const int alpha = p.pad ? p.pad - p.rx : (16 - (p.rx & 15)) & 15;
    const int xc0 = p.pad ? X0 : X0 - p.rx - alpha;
    const int padc = p.pad >> 2;  // chunks
    const int ya = p.out_begin + (int)blockIdx.y * p.TH;
    const int yb = min(ya + p.TH, p.out_end);
    if (ya >= yb) return;
    const uint8_t* in0 = in - (int64_t)p.row0 * p.pitch;  // row g at in0 + g*pitch
    // bulk-copied column range of the strip, [c_lo, c_hi16) (16-byte multiples), + byte tail
    const int c_lo = max(xc0, 0);
    const int c_hi = min(xc0 + p.NC, p.cols);
    const int c_hi16 = c_lo + ((max(c_hi - c_lo, 0)) & ~15);
    const int f_hi = min(X0 + p.TW, p.cols);
    const int f_hi16 = X0 + ((max(f_hi - X0, 0)) & ~15);

    // warm-up items carry up to 3 warm-up rows each (E, O, F slots)
    Items it;
    it.g0 = max(ya - p.r, 0);
    const int nwr = min(ya + p.r, p.H - 1) - it.g0 + 1;  // warm-up rows
    it.nwarm = (nwr + 2) / 3;                             // warm-up items
    it.ya = ya;
    it.n = it.nwarm + (yb - ya);

    // ---- init: zero the ring (columns outside the image stay zero), barriers
    {
        uint4* r4 = reinterpret_cast<uint4*>(ring);
        const int n16 = NS * 3 * p.NC / 16;
        for (int i = t; i < n16; i += blockDim.x) r4[i] = make_uint4(0, 0, 0, 0);
        // edge-padded layout: P of the columns left of the image is zero
        for (int L = t; L < padc; L += blockDim.x) {
            *reinterpret_cast<uint4*>(&sPS[pchunk_word(L)]) = make_uint4(0, 0, 0, 0);
            *reinterpret_cast<uint4*>(&sPQ[pchunk_word(L)]) = make_uint4(0, 0, 0, 0);
        }
    }
    if (t == 0) {
        for (int s = 0; s < NS; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], nwarps);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    // producer (thread 0): stage item k.  Rows outside the image are not copied; consumers
    // treat them as zero.  The byte tail beyond the last 16-byte chunk is written by thread 0
    // with generic stores (visible to consumers after the barriers in between).
    const uint64_t pol_keep = make_policy(p.l2hint ? 2 : 0), pol_drop = make_policy(p.l2hint ? 1 : 0);
    // The byte tail of a ragged row is written with generic stores BEFORE the arrive that arms
    // the stage: the arrive (release) publishes them to the consumers that wait on the stage.
    auto issue = [&](int k) {
        const int s = k % NS;
        if (k >= NS) mbar_wait(&empty[s], ((k / NS) - 1) & 1);
        uint8_t* E = ring + (size_t)s * 3 * p.NC;
        uint8_t* O = E + p.NC;
        uint8_t* F = O + p.NC;
        const uint32_t rowb = (uint32_t)(c_hi16 - c_lo);
        if (k < it.nwarm) {
            // warm-up rows g0+3k .. g0+3k+2 into the E, O, F slots (full strip width each)
            const int g = it.g0 + 3 * k, cnt = min(3, it.g0 + nwr - g);
            for (int i = 0; i < cnt; ++i)
                for (int c = c_hi16; c < c_hi; ++c) E[i * p.NC + c - xc0] = row_at<SEG>(p, in0, g + i)[c];
            mbar_expect_tx(&full[s], (uint32_t)cnt * rowb);
            for (int i = 0; i < cnt; ++i)
                if (rowb) bulk_g2s(E + i * p.NC + (c_lo - xc0), row_at<SEG>(p, in0, g + i) + c_lo, rowb, &full[s], pol_keep);
            return;
        }
        const int y = it.ya + (k - it.nwarm);
        const int gf = y;
        int ge = (k == it.nwarm) ? -1 : y + p.r;
        const int go = (k == it.nwarm) ? -1 : y - p.r - 1;
        if (ge >= p.H) ge = -1;
        const uint32_t fb = (uint32_t)(f_hi16 - X0);
        for (int c = c_hi16; c < c_hi; ++c) {
            if (ge >= 0) E[c - xc0] = row_at<SEG>(p, in0, ge)[c];
            if (go >= 0) O[c - xc0] = row_at<SEG>(p, in0, go)[c];
        }
        for (int c = f_hi16; c < f_hi; ++c) F[c - X0] = row_at<SEG>(p, in0, gf)[c];
        uint32_t bytes = fb;
        if (ge >= 0) bytes += rowb;
        if (go >= 0) bytes += rowb;
        mbar_expect_tx(&full[s], bytes);
        if (ge >= 0 && rowb) bulk_g2s(E + (c_lo - xc0), row_at<SEG>(p, in0, ge) + c_lo, rowb, &full[s], pol_keep);
        if (go >= 0 && rowb) bulk_g2s(O + (c_lo - xc0), row_at<SEG>(p, in0, go) + c_lo, rowb, &full[s], pol_drop);
        if (fb) bulk_g2s(F, row_at<SEG>(p, in0, gf) + X0, fb, &full[s], pol_keep);
    };
    const bool producer = (t == 0);
    if (producer)
        for (int k = 0; k < min(NS - 1, it.n); ++k) issue(k);

    uint32_t cS[V], cQ[V];
#pragma unroll
    for (int j = 0; j < V; ++j) { cS[j] = 0; cQ[j] = 0; }
    // per-quarter totals of cS / cQ (V/4 columns each), kept incrementally: the thread total
    // feeds the scan, and the quarter totals let the prefix run as 4 independent chains
    uint32_t qS[4] = {0, 0, 0, 0}, qQ[4] = {0, 0, 0, 0};

    const int xo = X0 + V * t;  // this thread's V output columns
    const bool has_out = (p.pad || V * t + V + 2 * p.rx + alpha <= p.NC) && (V * t < p.TW) &&
                         (xo < p.cols);
    const bool out_full = has_out && (xo + V <= p.cols) &&
                          ((reinterpret_cast<uintptr_t>(p.bin) | (uintptr_t)p.bin_pitch |
                            (uintptr_t)p.out_stride) & 15) == 0;
    const bool x_interior = (p.rx == p.r) && (xo - p.r >= 0) && (xo + V - 1 + p.r <= p.cols - 1);
    const int la0 = (alpha + V * t - MA) >> 2;
    const int lb0 = (alpha + 2 * p.rx + 1 + V * t - MB) >> 2;
    int aw[V / 4 + 1], bw[V / 4 + 1];
#pragma unroll
    for (int i = 0; i < V / 4 + 1; ++i) { aw[i] = pchunk_word(la0 + i); bw[i] = pchunk_word(lb0 + i); }
    // a warp with any x-border thread runs the (per-pixel count) border variant uniformly
    const bool x_border_warp = __any_sync(__activemask(), has_out && !x_interior);
    uint8_t* obase = p.bin + (int64_t)blockIdx.z * p.out_stride - (int64_t)p.out_begin * p.bin_pitch;
    // TMAP: RN(1/N) for the interior count, and 1/R when R is a power of two (exact scaling)
    double rnN = 0.0, rinv = 0.0;
    if constexpr (TMAP) {
        rnN = __drcp_rn((double)p.N);
        int e;
        if (frexp(p.rr, &e) == 0.5) rinv = ldexp(1.0, 1 - e);
    }

    auto release = [&](int k) {  // this warp is done with item k's stage
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[k % NS]);
    };

    // ---- warm-up: vertical window of the first output row
    for (int k = 0; k < it.nwarm; ++k) {
        const int s = k % NS;
        mbar_wait(&full[s], (k / NS) & 1);
        const int cnt = min(3, nwr - 3 * k);
        for (int i = 0; i < cnt; ++i) {
            const uint4* E = reinterpret_cast<const uint4*>(ring + (size_t)s * 3 * p.NC + i * p.NC + V * t);
            uint32_t w[V / 4];
#pragma unroll
            for (int q = 0; q < V / 16; ++q) {
                const uint4 a = E[q];
                w[4 * q] = a.x; w[4 * q + 1] = a.y; w[4 * q + 2] = a.z; w[4 * q + 3] = a.w;
            }
#pragma unroll
            for (int j = 0; j < V; ++j) {
                const uint32_t v = byte_at(w, j);
                cS[j] += v;
                cQ[j] += v * v;
            }
        }
        release(k);
        if (producer && k + NS - 1 < it.n) issue(k + NS - 1);
    }
#pragma unroll
    for (int j = 0; j < V; ++j) { qS[j / (V / 4)] += cS[j]; qQ[j / (V / 4)] += cQ[j]; }

    for (int k = it.nwarm; k < it.n; ++k) {
        const int y = it.ya + (k - it.nwarm);
        const int s = k % NS;
        mbar_wait(&full[s], (k / NS) & 1);
        const uint8_t* stage = ring + (size_t)s * 3 * p.NC;
        // Entering / leaving rows (all-zero on the band's first step and past the image), the
        // dp4a totals, the warp scan and the per-column vertical update form ONE basic block:
        // the scan's shuffle latency is hidden behind the independent column updates.
        const bool first = (k == it.nwarm);
        const bool ein = !first && y + p.r < p.H, oin = !first && y - p.r - 1 >= 0;
        uint32_t e[V / 4], o[V / 4];
        {
            const uint4* E = reinterpret_cast<const uint4*>(stage + V * t);
            const uint4* O = reinterpret_cast<const uint4*>(stage + p.NC + V * t);
#pragma unroll
            for (int q = 0; q < V / 16; ++q) {
                const uint4 a = ein ? E[q] : make_uint4(0, 0, 0, 0);
                const uint4 b = oin ? O[q] : make_uint4(0, 0, 0, 0);
                e[4 * q] = a.x; e[4 * q + 1] = a.y; e[4 * q + 2] = a.z; e[4 * q + 3] = a.w;
                o[4 * q] = b.x; o[4 * q + 1] = b.y; o[4 * q + 2] = b.z; o[4 * q + 3] = b.w;
            }
        }
#pragma unroll
        for (int q = 0; q < V / 4; ++q) {  // 4 columns per dp4a: sum of bytes / of squares
            qS[q / (V / 16)] += (uint32_t)__dp4a(e[q], 0x01010101u, 0u) -
                                (uint32_t)__dp4a(o[q], 0x01010101u, 0u);
            qQ[q / (V / 16)] += (uint32_t)__dp4a(e[q], e[q], 0u) - (uint32_t)__dp4a(o[q], o[q], 0u);
        }
        // ---- horizontal inclusive prefix, exact mod 2^32 (blockDim is a multiple of 32)
        const uint32_t TS = (qS[0] + qS[1]) + (qS[2] + qS[3]);
        const uint32_t TQ = (qQ[0] + qQ[1]) + (qQ[2] + qQ[3]);
        uint32_t iS = TS, iQ = TQ;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const uint32_t vs = __shfl_up_sync(0xffffffffu, iS, off);
            const uint32_t vq = __shfl_up_sync(0xffffffffu, iQ, off);
            if (lane >= off) { iS += vs; iQ += vq; }
        }
#pragma unroll
        for (int j = 0; j < V; ++j) {
            const uint32_t ev = byte_at(e, j), ov = byte_at(o, j);
            const uint32_t dv = ev - ov;
            cS[j] += dv;
            cQ[j] += dv * (ev + ov);
        }
        if (lane == 31) { sWS[warp] = iS; sWQ[warp] = iQ; }
        __syncthreads();
        if (producer && k + NS - 1 < it.n) issue(k + NS - 1);
        uint32_t bS = iS - TS, bQ = iQ - TQ;
        for (int w = 0; w < warp; ++w) { bS += sWS[w]; bQ += sWQ[w]; }
        // logical word Vt + m holds P[Vt + m - 1]: the first slot is this thread's base.
        // Four independent running chains, one per quarter of the thread's columns.
        uint32_t cbS[4], cbQ[4];
        cbS[0] = bS; cbQ[0] = bQ;
#pragma unroll
        for (int h = 1; h < 4; ++h) { cbS[h] = cbS[h - 1] + qS[h - 1]; cbQ[h] = cbQ[h - 1] + qQ[h - 1]; }
        bS = cbS[3] + qS[3];
        bQ = cbQ[3] + qQ[3];
#pragma unroll
        for (int j = 0; j < V / 4; j += 4) {
#pragma unroll
            for (int h = 0; h < 4; ++h) {
                const int c0 = h * (V / 4) + j;
                uint4 vs, vq;
                vs.x = cbS[h]; vq.x = cbQ[h];
                cbS[h] += cS[c0]; cbQ[h] += cQ[c0];
                vs.y = cbS[h]; vq.y = cbQ[h];
                cbS[h] += cS[c0 + 1]; cbQ[h] += cQ[c0 + 1];
                vs.z = cbS[h]; vq.z = cbQ[h];
                cbS[h] += cS[c0 + 2]; cbQ[h] += cQ[c0 + 2];
                vs.w = cbS[h]; vq.w = cbQ[h];
                cbS[h] += cS[c0 + 3]; cbQ[h] += cQ[c0 + 3];
                const int pw = pchunk_word(padc + (V / 4) * t + c0 / 4);
                DTB_CHECK(pw >= 0 && pw + 4 <= NCp);
                *reinterpret_cast<uint4*>(&sPS[pw]) = vs;
                *reinterpret_cast<uint4*>(&sPQ[pw]) = vq;
            }
        }
        if (p.pad) {
            // the row total, repeated over the padr words right of the strip (last warp)
            if (warp == nwarps - 1) {
                const uint32_t tS = __shfl_sync(0xffffffffu, bS, 31), tQ = __shfl_sync(0xffffffffu, bQ, 31);
                for (int L = lane; L < (p.padr >> 2); L += 32) {
                    const int pw = pchunk_word(padc + p.NC / 4 + L);
                    DTB_CHECK(pw >= 0 && pw + 4 <= NCp);
                    *reinterpret_cast<uint4*>(&sPS[pw]) = make_uint4(tS, tS, tS, tS);
                    *reinterpret_cast<uint4*>(&sPQ[pw]) = make_uint4(tQ, tQ, tQ, tQ);
                }
            }
        } else if (t == blockDim.x - 1) {  // logical word NC = P[NC - 1]
            const int pw = pchunk_word(p.NC / 4);
            sPS[pw] = bS;
            sPQ[pw] = bQ;
        }
        __syncthreads();

        // ---- outputs
        if (has_out) {
            const bool y_interior = (y - p.r >= 0) && (y + p.r <= p.H - 1);
            uint8_t* orow = obase + (int64_t)y * p.bin_pitch;
            const int ny = min(y + p.r, p.H - 1) - max(y - p.r, 0) + 1;
            const uint8_t* fsm = stage + 2 * p.NC + V * t;
            bool unc = false;
            uint32_t ow[V / 4];
            if constexpr (TMAP) {
                double* trow = reinterpret_cast<double*>(reinterpret_cast<uint8_t*>(p.tmap) +
                                                         (y - p.out_begin) * p.tmap_pitch) + xo;
                // (uniform) R a power of two: the interior variant is then free of branches
                if (y_interior && !x_border_warp) {
                    if (rinv != 0.0)
                        row_outputs_tmap<V, RXM4, METHOD, false, true>(sPS, sPQ, aw, bw, fsm, ow, trow, xo, p.cols, ny,
                                                               p.r, p, rnN, rinv);
                    else
                        row_outputs_tmap<V, RXM4, METHOD, false, false>(sPS, sPQ, aw, bw, fsm, ow, trow, xo, p.cols, ny,
                                                                p.r, p, rnN, rinv);
                } else {
                    row_outputs_tmap<V, RXM4, METHOD, true, false>(sPS, sPQ, aw, bw, fsm, ow, trow, xo, p.cols, ny,
                                                           p.r, p, rnN, rinv);
                }
            } else if (y_interior && !x_border_warp)
                unc = row_outputs<V, RXM4, METHOD, false>(sPS, sPQ, aw, bw, fsm, ow, xo, p.cols, ny,
                                                          p.r, p);
            else
                unc = row_outputs<V, RXM4, METHOD, true>(sPS, sPQ, aw, bw, fsm, ow, xo, p.cols, ny,
                                                         p.r, p);
            if (out_full) {
#pragma unroll
                for (int q = 0; q < V / 16; ++q)  // streaming store: the output is not re-read
                    __stcs(reinterpret_cast<uint4*>(orow + xo + 16 * q),
                           make_uint4(ow[4 * q], ow[4 * q + 1], ow[4 * q + 2], ow[4 * q + 3]));
            } else {
#pragma unroll
                for (int j = 0; j < V; ++j) {
                    const int x = xo + j;
                    if (x >= 0 && x < p.cols) orow[x] = (uint8_t)(ow[j >> 2] >> (8 * (j & 3)));
                }
            }
            if (__builtin_expect(unc, 0))
                fix_uncertain<METHOD>(sPS, sPQ, alpha + V * t, alpha + 2 * p.rx + 1 + V * t,
                                      row_at<SEG>(p, in0, y), orow, xo, V, p.cols, ny, p.r, p.N,
                                      p.cA, p.cC, p.a, p.c, p.tol, p.k, p.rr);
        }
        release(k);
    }
}


// =====================================================================================
// Warp-specialized variant (ws_kernel): column warps (vertical sums + horizontal prefix)
// and output warps (window sums -> certified decision -> bytes) run CONCURRENTLY on a
// double-buffered prefix.  Hand-off with named barriers: READY[b] (column -> output: P_k in
// buffer b = k&1 is complete) and FREE[b] (output -> column: row k-2 consumed, buffer b may
// be overwritten).  Column warps never wait for the latency-bound output phase of the same
// row, and output warps never sit behind the column warps' scan / barriers.
// =====================================================================================






#ifndef DTB_WS_MAXREG
#define DTB_WS_MAXREG 168
#endif
#ifndef DTB_WS_MAXREG16
#define DTB_WS_MAXREG16 80
#endif

// V: columns per column thread; VO: outputs per output thread.  V = VO = 32 (168 registers,
// 3 CTAs x 4 warps per SM) or V = VO = 16 (half the per-thread state, DTB_WS_MAXREG16
// registers, twice the warps per CTA).
template <int V, int VO, int RXM4, int MX>
__global__ void __maxnreg__(V == 16 ? DTB_WS_MAXREG16 : DTB_WS_MAXREG) ws_kernel(SlideParams p) {
    constexpr int METHOD = MX & 3;
    constexpr bool SEG = (MX & 4) != 0;
    constexpr int MA = (4 - RXM4) & 3;
    constexpr int MB = (RXM4 + 1) & 3;
    constexpr int NS = WS_STAGES;
    extern __shared__ __align__(128) uint32_t sm[];
    const int NCp = slide_padded_words(p.NC);
    uint32_t* sWS = sm + 4 * NCp;   // [2][8] per-column-warp totals, double buffered
    uint32_t* sWQ = sWS + 16;
    uint64_t* full = reinterpret_cast<uint64_t*>(sWS + 32);
    uint64_t* empty = full + NS;
    uint8_t* ring = reinterpret_cast<uint8_t*>(empty + NS);
    const int ncw = p.ncw, now = p.now, nthr = 32 * (ncw + now);

    // warps [0, ncw) are the column warps, [ncw, ncw + now) the output warps
    const int t = threadIdx.x;
    const int lane = t & 31, warp = t >> 5;
    const bool is_col = warp < ncw;
    const uint8_t* in = p.in + (int64_t)blockIdx.z * p.img_stride;
    const int X0 = (int)blockIdx.x * p.TW;
    const int alpha = (16 - (p.rx & 15)) & 15;
    const int xc0 = X0 - p.rx - alpha;
    const int ya = p.out_begin + (int)blockIdx.y * p.TH;
    const int yb = min(ya + p.TH, p.out_end);
    if (ya >= yb) return;
    const uint8_t* in0 = in - (int64_t)p.row0 * p.pitch;
    const int c_lo = max(xc0, 0);
    const int c_hi = min(xc0 + p.NC, p.cols);
    const int c_hi16 = c_lo + ((max(c_hi - c_lo, 0)) & ~15);
    const int f_hi = min(X0 + p.TW, p.cols);
    const int f_hi16 = X0 + ((max(f_hi - X0, 0)) & ~15);
    // warm-up items carry up to 3 warm-up rows each (E, O, F slots)
    Items it;
    it.g0 = max(ya - p.r, 0);
    const int nwr = min(ya + p.r, p.H - 1) - it.g0 + 1;  // warm-up rows
    it.nwarm = (nwr + 2) / 3;                             // warm-up items
    it.ya = ya;
    it.n = it.nwarm + (yb - ya);

    {
        uint4* r4 = reinterpret_cast<uint4*>(ring);
        const int n16 = NS * 3 * p.NC / 16;
        for (int i = t; i < n16; i += blockDim.x) r4[i] = make_uint4(0, 0, 0, 0);
    }
    if (t == 0) {
        for (int s = 0; s < NS; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], ncw + now);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    const uint64_t pol_keep = make_policy(p.l2hint ? 2 : 0), pol_drop = make_policy(p.l2hint ? 1 : 0);
    // ragged byte tails first, then the arrive that arms the stage publishes them (release)
    auto issue = [&](int k) {
        const int s = k % NS;
        if (k >= NS) mbar_wait(&empty[s], ((k / NS) - 1) & 1);
        uint8_t* E = ring + (size_t)s * 3 * p.NC;
        uint8_t* O = E + p.NC;
        uint8_t* F = O + p.NC;
        const uint32_t rowb = (uint32_t)(c_hi16 - c_lo);
        if (k < it.nwarm) {
            const int g = it.g0 + 3 * k, cnt = min(3, it.g0 + nwr - g);
            for (int i = 0; i < cnt; ++i)
                for (int c = c_hi16; c < c_hi; ++c) E[i * p.NC + c - xc0] = row_at<SEG>(p, in0, g + i)[c];
            mbar_expect_tx(&full[s], (uint32_t)cnt * rowb);
            for (int i = 0; i < cnt; ++i)
                if (rowb) bulk_g2s(E + i * p.NC + (c_lo - xc0), row_at<SEG>(p, in0, g + i) + c_lo, rowb, &full[s], pol_keep);
            return;
        }
        const int y = it.ya + (k - it.nwarm);
        const int gf = y;
        int ge = (k == it.nwarm) ? -1 : y + p.r;
        const int go = (k == it.nwarm) ? -1 : y - p.r - 1;
        if (ge >= p.H) ge = -1;
        const uint32_t fb = (uint32_t)(f_hi16 - X0);
        for (int c = c_hi16; c < c_hi; ++c) {
            if (ge >= 0) E[c - xc0] = row_at<SEG>(p, in0, ge)[c];
            if (go >= 0) O[c - xc0] = row_at<SEG>(p, in0, go)[c];
        }
        for (int c = f_hi16; c < f_hi; ++c) F[c - X0] = row_at<SEG>(p, in0, gf)[c];
        uint32_t bytes = fb;
        if (ge >= 0) bytes += rowb;
        if (go >= 0) bytes += rowb;
        mbar_expect_tx(&full[s], bytes);
        if (ge >= 0 && rowb) bulk_g2s(E + (c_lo - xc0), row_at<SEG>(p, in0, ge) + c_lo, rowb, &full[s], pol_keep);
        if (go >= 0 && rowb) bulk_g2s(O + (c_lo - xc0), row_at<SEG>(p, in0, go) + c_lo, rowb, &full[s], pol_drop);
        if (fb) bulk_g2s(F, row_at<SEG>(p, in0, gf) + X0, fb, &full[s], pol_keep);
    };

    if (is_col) {
        // ===================== column warps =====================
        int issued = 0;
        if (t == 0)
            while (issued < min(NS - 1, it.n)) issue(issued++);
        uint32_t cS[V], cQ[V];
#pragma unroll
        for (int j = 0; j < V; ++j) { cS[j] = 0; cQ[j] = 0; }
        uint32_t qS[4] = {0, 0, 0, 0}, qQ[4] = {0, 0, 0, 0};
        for (int k = 0; k < it.nwarm; ++k) {
            const int s = k % NS;
            mbar_wait(&full[s], (k / NS) & 1);
            const int cnt = min(3, nwr - 3 * k);
            for (int i = 0; i < cnt; ++i) {
                const uint4* E = reinterpret_cast<const uint4*>(ring + (size_t)s * 3 * p.NC + i * p.NC + V * t);
                uint32_t w[V / 4];
#pragma unroll
                for (int q = 0; q < V / 16; ++q) {
                    const uint4 a = E[q];
                    w[4 * q] = a.x; w[4 * q + 1] = a.y; w[4 * q + 2] = a.z; w[4 * q + 3] = a.w;
                }
#pragma unroll
                for (int j = 0; j < V; ++j) {
                    const uint32_t v = byte_at(w, j);
                    cS[j] += v;
                    cQ[j] += v * v;
                }
            }
            __syncwarp();
            // warm-up items are read by the column warps only: warp 0 arrives for the output warps
            if (lane == 0) mbar_arrive_cnt(&empty[s], warp == 0 ? 1 + now : 1);
            if (t == 0)
                while (issued < min(k + NS, it.n)) issue(issued++);
        }
#pragma unroll
        for (int j = 0; j < V; ++j) { qS[j / (V / 4)] += cS[j]; qQ[j / (V / 4)] += cQ[j]; }

        for (int k = it.nwarm; k < it.n; ++k) {
            const int y = it.ya + (k - it.nwarm);
            const int s = k % NS;
            const int b = (k - it.nwarm) & 1;
            mbar_wait(&full[s], (k / NS) & 1);
            const uint8_t* stage = ring + (size_t)s * 3 * p.NC;
            const bool first = (k == it.nwarm);
            const bool ein = !first && y + p.r < p.H, oin = !first && y - p.r - 1 >= 0;
            uint32_t e[V / 4], o[V / 4];
            {
                const uint4* E = reinterpret_cast<const uint4*>(stage + V * t);
                const uint4* O = reinterpret_cast<const uint4*>(stage + p.NC + V * t);
#pragma unroll
                for (int q = 0; q < V / 16; ++q) {
                    const uint4 a = ein ? E[q] : make_uint4(0, 0, 0, 0);
                    const uint4 bb = oin ? O[q] : make_uint4(0, 0, 0, 0);
                    e[4 * q] = a.x; e[4 * q + 1] = a.y; e[4 * q + 2] = a.z; e[4 * q + 3] = a.w;
                    o[4 * q] = bb.x; o[4 * q + 1] = bb.y; o[4 * q + 2] = bb.z; o[4 * q + 3] = bb.w;
                }
            }
#pragma unroll
            for (int q = 0; q < V / 4; ++q) {
                qS[q / (V / 16)] += (uint32_t)__dp4a(e[q], 0x01010101u, 0u) -
                                    (uint32_t)__dp4a(o[q], 0x01010101u, 0u);
                qQ[q / (V / 16)] += (uint32_t)__dp4a(e[q], e[q], 0u) - (uint32_t)__dp4a(o[q], o[q], 0u);
            }
            const uint32_t TS = (qS[0] + qS[1]) + (qS[2] + qS[3]);
            const uint32_t TQ = (qQ[0] + qQ[1]) + (qQ[2] + qQ[3]);
            uint32_t iS = TS, iQ = TQ;
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {
                const uint32_t vs = __shfl_up_sync(0xffffffffu, iS, off);
                const uint32_t vq = __shfl_up_sync(0xffffffffu, iQ, off);
                if (lane >= off) { iS += vs; iQ += vq; }
            }
#pragma unroll
            for (int j = 0; j < V; ++j) {
                const uint32_t ev = byte_at(e, j), ov = byte_at(o, j);
                const uint32_t dv = ev - ov;
                cS[j] += dv;
                cQ[j] += dv * (ev + ov);
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[s]);  // this warp is done with item k's rows
            if (lane == 31) { sWS[8 * b + warp] = iS; sWQ[8 * b + warp] = iQ; }
            nbar_sync(BAR_COLS, 32 * ncw);
            uint32_t bS = iS - TS, bQ = iQ - TQ;
            for (int w = 0; w < warp; ++w) { bS += sWS[8 * b + w]; bQ += sWQ[8 * b + w]; }
            // wait until the output warps have consumed row k-2 from this prefix buffer
            nbar_sync(BAR_FREE0 + b, nthr);
            uint32_t* sPS = sm + (2 * b) * NCp;
            uint32_t* sPQ = sm + (2 * b + 1) * NCp;
            uint32_t cbS[4], cbQ[4];
            cbS[0] = bS; cbQ[0] = bQ;
#pragma unroll
            for (int h = 1; h < 4; ++h) { cbS[h] = cbS[h - 1] + qS[h - 1]; cbQ[h] = cbQ[h - 1] + qQ[h - 1]; }
#pragma unroll
            for (int j = 0; j < V / 4; j += 4) {
#pragma unroll
                for (int h = 0; h < 4; ++h) {
                    const int c0 = h * (V / 4) + j;
                    uint4 vs, vq;
                    vs.x = cbS[h]; vq.x = cbQ[h];
                    cbS[h] += cS[c0]; cbQ[h] += cQ[c0];
                    vs.y = cbS[h]; vq.y = cbQ[h];
                    cbS[h] += cS[c0 + 1]; cbQ[h] += cQ[c0 + 1];
                    vs.z = cbS[h]; vq.z = cbQ[h];
                    cbS[h] += cS[c0 + 2]; cbQ[h] += cQ[c0 + 2];
                    vs.w = cbS[h]; vq.w = cbQ[h];
                    cbS[h] += cS[c0 + 3]; cbQ[h] += cQ[c0 + 3];
                    const int pw = pchunk_word((V / 4) * t + c0 / 4);
                DTB_CHECK(pw >= 0 && pw + 4 <= NCp);
                    *reinterpret_cast<uint4*>(&sPS[pw]) = vs;
                    *reinterpret_cast<uint4*>(&sPQ[pw]) = vq;
                }
            }
            if (t == 32 * ncw - 1) {  // logical word NC = P[NC - 1]
                const int pw = pchunk_word(p.NC / 4);
                sPS[pw] = cbS[3];
                sPQ[pw] = cbQ[3];
            }
            nbar_arrive(BAR_READY0 + b, nthr);
            if (t == 0)  // row staging after publishing row k: off READY's path
                while (issued < min(k + NS - 1, it.n)) issue(issued++);
        }
        // consume the output warps' last FREE arrivals so no named barrier is left pending
        const int rows = it.n - it.nwarm;
        if (rows >= 1) nbar_sync(BAR_FREE0 + (rows & 1), nthr);
        if (rows >= 2) nbar_sync(BAR_FREE0 + ((rows + 1) & 1), nthr);
    } else {
        // ===================== output warps =====================
        const int to = t - 32 * ncw;  // output thread index
        const int xo = X0 + VO * to;
        const bool has_out = (VO * to + VO + 2 * p.rx + alpha <= p.NC) && (VO * to < p.TW) &&
                             (xo < p.cols);
        const bool out_full = has_out && (xo + VO <= p.cols) &&
                              ((reinterpret_cast<uintptr_t>(p.bin) | (uintptr_t)p.bin_pitch |
                                (uintptr_t)p.out_stride) & 15) == 0;
        const bool x_interior = (p.rx == p.r) && (xo - p.r >= 0) && (xo + VO - 1 + p.r <= p.cols - 1);
        const int la0 = (alpha + VO * to - MA) >> 2;
        const int lb0 = (alpha + 2 * p.rx + 1 + VO * to - MB) >> 2;
        int aw[VO / 4 + 1], bw[VO / 4 + 1];
#pragma unroll
        for (int i = 0; i < VO / 4 + 1; ++i) { aw[i] = pchunk_word(la0 + i); bw[i] = pchunk_word(lb0 + i); }
        const bool x_border_warp = __any_sync(0xffffffffu, has_out && !x_interior);
        uint8_t* obase = p.bin + (int64_t)blockIdx.z * p.out_stride - (int64_t)p.out_begin * p.bin_pitch;
        nbar_arrive(BAR_FREE0, nthr);  // both prefix buffers start free
        nbar_arrive(BAR_FREE0 + 1, nthr);
        for (int k = it.nwarm; k < it.n; ++k) {
            const int y = it.ya + (k - it.nwarm);
            const int s = k % NS;
            const int b = (k - it.nwarm) & 1;
            nbar_sync(BAR_READY0 + b, nthr);
            mbar_wait(&full[s], (k / NS) & 1);  // (complete; makes the staged rows visible)
            const uint8_t* stage = ring + (size_t)s * 3 * p.NC;
            const uint32_t* sPS = sm + (2 * b) * NCp;
            const uint32_t* sPQ = sm + (2 * b + 1) * NCp;
            if (has_out) {
                const bool y_interior = (y - p.r >= 0) && (y + p.r <= p.H - 1);
                uint8_t* orow = obase + (int64_t)y * p.bin_pitch;
                const int ny = min(y + p.r, p.H - 1) - max(y - p.r, 0) + 1;
                const uint8_t* fsm = stage + 2 * p.NC + VO * to;
                uint32_t ow[VO / 4];
                bool unc;
                if (y_interior && !x_border_warp)
                    unc = row_outputs<VO, RXM4, METHOD, false>(sPS, sPQ, aw, bw, fsm, ow, xo, p.cols,
                                                              ny, p.r, p);
                else
                    unc = row_outputs<VO, RXM4, METHOD, true>(sPS, sPQ, aw, bw, fsm, ow, xo, p.cols,
                                                             ny, p.r, p);
                if (out_full) {
#pragma unroll
                    for (int q = 0; q < VO / 16; ++q)
                        __stcs(reinterpret_cast<uint4*>(orow + xo + 16 * q),
                               make_uint4(ow[4 * q], ow[4 * q + 1], ow[4 * q + 2], ow[4 * q + 3]));
                } else {
#pragma unroll
                    for (int j = 0; j < VO; ++j) {
                        const int x = xo + j;
                        if (x >= 0 && x < p.cols) orow[x] = (uint8_t)(ow[j >> 2] >> (8 * (j & 3)));
                    }
                }
                if (__builtin_expect(unc, 0))
                    fix_uncertain<METHOD>(sPS, sPQ, alpha + VO * to, alpha + 2 * p.rx + 1 + VO * to,
                                          row_at<SEG>(p, in0, y), orow, xo, VO, p.cols, ny, p.r,
                                          p.N, p.cA, p.cC, p.a, p.c, p.tol, p.k, p.rr);
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[s]);
            nbar_arrive(BAR_FREE0 + b, nthr);
        }
    }
}

// Certified tolerance (see header comment):  |t_fp32 - t_exact| <= E_fast and
// |t_reference - t_exact| <= E_ref, so |f - t_fp32| >= tol = 2 (E_fast + E_ref) fixes the sign of
// f - t_reference.  E_ref: the reference's var = Q/n - mean^2 carries <= 5u Q/n <= 3.6e-11
// absolute error (u = 2^-53, Q/n <= 255^2), hence std carries <= sqrt(3.6e-11) = 6.0e-6;
// Sauvola multiplies it by mean*k/R <= 255 k/R, Niblack by |k|.  E_fast: D is exact; the fp32
// rounding of D, sqrt.approx / rcp.approx (<= 2^-21 assumed each), the rounded constants and
// the fmas give a relative error <= 1.1e-6 on the threshold; we use 1.5e-6 times a bound on |t|.
void slide_constants(SlideParams& p) {
    static const int l2hint = [] { const char* e = getenv("DTB_L2HINT"); return e ? atoi(e) : 1; }();
    p.l2hint = l2hint;
    const double W = 2.0 * p.r + 1.0;
    const FastConsts fc = fast_constants(p.method, p.k, p.rr, W * W);
    p.N = fc.N;
    p.a = fc.a;
    p.c = fc.c;
    p.cA = fc.cA;
    p.cC = fc.cC;
    p.tol = fc.tol;
}

// Host-side launch state is cached per instantiation: the dynamic-smem opt-in is raised once to
// the largest size ever requested, and occupancy answers are memoised per (block, smem) -- the
// runtime queries cost tens of microseconds, which would dominate small images.
// Per-device launch state of one kernel: the dynamic-smem opt-in (cudaFuncSetAttribute applies
// to the current device only) and memoised occupancy answers (the runtime queries cost tens of
// microseconds, which would dominate small images).  Keyed by (device, kernel[, block, smem]),
// guarded by a mutex: the C ABI may be called from several host threads and devices.
static std::mutex g_launch_mu;
static std::map<std::pair<int, const void*>, size_t> g_granted;
static std::map<std::tuple<int, const void*, int, size_t>, int> g_occ;

static cudaError_t kernel_prepare(const void* fn, int nt, size_t smem, int* occ) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    std::lock_guard<std::mutex> lk(g_launch_mu);
    size_t& g = g_granted[{dev, fn}];
    if (smem > 48 * 1024 && smem > g) {
        e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        g = smem;
    }
    if (occ) {
        auto it = g_occ.find({dev, fn, nt, smem});
        if (it == g_occ.end()) {
            int blocks = 0;
            if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, fn, nt, smem) != cudaSuccess)
                blocks = 1;
            it = g_occ.emplace(std::make_tuple(dev, fn, nt, smem), std::max(blocks, 1)).first;
        }
        *occ = it->second;
    }
    return cudaSuccess;
}

template <int V, int RXM4, int METHOD>
static cudaError_t run_slide(dim3 grid, int nt, size_t smem, const SlideParams& p,
                             cudaStream_t st) {
    cudaError_t e = kernel_prepare((const void*)slide_kernel<V, RXM4, METHOD>, nt, smem, nullptr);
    if (e != cudaSuccess) return e;
    slide_kernel<V, RXM4, METHOD><<<grid, nt, smem, st>>>(p);
    return cudaGetLastError();
}

template <int V, int RXM4, int METHOD>
static int occupancy(int nt, size_t smem) {
    int blocks = 1;
    kernel_prepare((const void*)slide_kernel<V, RXM4, METHOD>, nt, smem, &blocks);
    return blocks;
}

// run (occ == nullptr) or query occupancy of the instantiation for (V, rx mod 4, method)
template <int V>
static cudaError_t dispatch_rx(int m, bool sv, dim3 grid, int nt, size_t smem,
                               const SlideParams& p, cudaStream_t st, int* occ) {
#define DTB_MX(M, X)                                                                         \
    if (occ) {                                                                               \
        *occ = occupancy<V, M, X>(nt, smem);                                                 \
        return cudaSuccess;                                                                  \
    }                                                                                        \
    return run_slide<V, M, X>(grid, nt, smem, p, st);
#define DTB_CASE(M)                                                                          \
    case M:                                                                                  \
        if constexpr (V == 32) {                                                             \
            if (p.nseg) {                                                                    \
                if (sv) { DTB_MX(M, DTB_METHOD_SAUVOLA | 4) } else { DTB_MX(M, DTB_METHOD_NIBLACK | 4) } \
            }                                                                                \
        }                                                                                    \
        if constexpr (V == 16) {                                                             \
            if (p.tmap) {                                                                    \
                if (sv) { DTB_MX(M, DTB_METHOD_SAUVOLA | 8) } else { DTB_MX(M, DTB_METHOD_NIBLACK | 8) } \
            }                                                                                \
        }                                                                                    \
        if (sv) { DTB_MX(M, DTB_METHOD_SAUVOLA) } else { DTB_MX(M, DTB_METHOD_NIBLACK) }
    switch (m) {
        DTB_CASE(0)
        DTB_CASE(1)
        DTB_CASE(2)
        DTB_CASE(3)
    }
#undef DTB_CASE
#undef DTB_MX
    return cudaErrorInvalidValue;
}

// ---- warp-specialized launcher
template <int V, int VO, int RXM4, int MX>
static cudaError_t ws_run(dim3 grid, int nt, size_t smem, const SlideParams& p, cudaStream_t st,
                          int* occ) {
    auto kern = ws_kernel<V, VO, RXM4, MX>;
    cudaError_t e = kernel_prepare((const void*)kern, nt, smem, occ);
    if (e != cudaSuccess || occ) return e;
    kern<<<grid, nt, smem, st>>>(p);
    return cudaGetLastError();
}

template <int V, int VO>
static cudaError_t ws_dispatch_vo(int m, bool sv, dim3 grid, int nt, size_t smem,
                                  const SlideParams& p, cudaStream_t st, int* occ) {
#define DTB_WS_M(M)                                                                          \
    if (p.nseg)                                                                              \
        return sv ? ws_run<V, VO, M, DTB_METHOD_SAUVOLA | 4>(grid, nt, smem, p, st, occ)      \
                  : ws_run<V, VO, M, DTB_METHOD_NIBLACK | 4>(grid, nt, smem, p, st, occ);     \
    return sv ? ws_run<V, VO, M, DTB_METHOD_SAUVOLA>(grid, nt, smem, p, st, occ)              \
              : ws_run<V, VO, M, DTB_METHOD_NIBLACK>(grid, nt, smem, p, st, occ);
    switch (m) {
        case 0: { DTB_WS_M(0) }
        case 1: { DTB_WS_M(1) }
        case 2: { DTB_WS_M(2) }
        default: { DTB_WS_M(3) }
    }
#undef DTB_WS_M
}

static cudaError_t ws_dispatch(int m, bool sv, dim3 grid, int nt, size_t smem, const SlideParams& p,
                               cudaStream_t st, int* occ) {
    return ws_dispatch_vo<32, 32>(m, sv, grid, nt, smem, p, st, occ);
}

static int use_ws() {  // DTB_WS=0/1 forces the classic / warp-specialised kernel (read once)
    static const int v = [] { const char* e = getenv("DTB_WS"); return e ? atoi(e) : DTB_WS_DEFAULT; }();
    return v;
}

// Debug: DTB_PRINT_PLAN=1 prints each launch's strip/band plan (read once)
static bool print_plan() {
    static const bool v = [] { const char* e = getenv("DTB_PRINT_PLAN"); return e && e[0] == '1'; }();
    return v;
}

static thread_local const char* g_last_kernel = "";
const char* last_kernel() { return g_last_kernel; }
void set_last_kernel(const char* name) { g_last_kernel = name; }

cudaError_t set_fp32_audit(unsigned long long* counters) {
    const cudaError_t e = cudaMemcpyToSymbol(g_fp32_audit, &counters, sizeof(counters));
    return e != cudaSuccess ? e : set_fp32_audit_block(counters);
}

// DTB_BB: 0 never, 1 whenever eligible, 2 (default): eligible and either r >= DTB_BB_MIN_R, or
// r >= DTB_BB_MIN_R_LARGE on pages of >= 2^26 output pixels.  Measured on the 4096^2 page
// (scripts/c5_probe.py, round 2c): W59 (r=29) 0.098 ms on either kernel, W63 0.068 vs 0.108 ms,
// W67 0.078 vs 0.104; at W <= 51 the 13 columns of block slack are too large a share of the window
// (most groups stay open: W43 0.30 ms, W19 0.40 ms vs 0.09 on the per-pixel kernel).
#ifndef DTB_BB_MIN_R
#define DTB_BB_MIN_R 31
#endif
#ifndef DTB_BB_MIN_R_LARGE
#define DTB_BB_MIN_R_LARGE 24
#endif
// DTB_PAD: 0 never, 1 whenever the image fits one strip, 2 (default) when it also saves >= 10%
// of the column work (read per launch: tests switch it)
static int pad_mode() {
    const char* e = getenv("DTB_PAD");
    return e ? atoi(e) : 2;
}
static int bb_mode() {  // read per launch (tests switch it)
    const char* e = getenv("DTB_BB");
    return e ? atoi(e) : 2;
}

// Band count minimising waves * (TH + wf (2r+1)) + tf * TH in main-row units per CTA slot
// (bb_kernel's planner uses the same model).
static int plan_bands(int rows_out, int units, int slots, int r, double wf, double tf) {
    int nbands = 1;
    double best_cost = 1e300;
    const int nb_max = std::max(1, std::min((rows_out + 7) / 8, 4 * slots / std::max(1, units) + 1));
    for (int nb = 1; nb <= nb_max; ++nb) {
        const int th = (rows_out + nb - 1) / nb;
        const int waves = (units * nb + slots - 1) / slots;
        const double cost = waves * (th + wf * (2 * r + 1)) + tf * th;
        if (cost < best_cost) { best_cost = cost; nbands = nb; }
    }
    return std::max(1, std::min(nbands, (rows_out + 7) / 8));
}

cudaError_t launch_slide(SlideParams p, int n_images, int num_sms, cudaStream_t st) {
    slide_constants(p);
    // segmented variants: V = 32 only; the tmap variant runs V = 16 (half the registers per
    // thread: twice the resident warps for its fp64 epilogue)
    int V = p.tmap ? 16 : 32;
    const int rows_out = p.out_end - p.out_begin;
    const int alpha = (16 - (p.rx & 15)) & 15;
    // strip plan: w warps -> NC = 32 V w columns; pick the w (1..8) with the least total column
    // work (strips x NC) for this image width, balancing the strips' output widths.
    struct Plan { int w, strips, tw; long work; };
    auto plan_for = [&](int Vx) {
        Plan b{0, 0, 0, 0};
        for (int w = 1; w <= 8; ++w) {
            const int nc = 32 * Vx * w;
            const int twmax = 32 * ((nc - 2 * p.rx - alpha) / 32);
            if (twmax < 32) continue;
            const int ns = (p.cols + twmax - 1) / twmax;
            const int tw = 32 * ((p.cols + 32 * ns - 1) / (32 * ns));
            const long work = (long)ns * nc;
            if (b.w == 0 || work < b.work) b = Plan{w, ns, tw, work};
        }
        return b;
    };
    {
        const int bbm = bb_mode();
        const long long px = (long long)p.cols * (p.out_end - p.out_begin) * n_images;
        if (bbm && !p.tmap && bb_eligible(p) && bb_tma_ok(p, n_images) &&
            (bbm == 1 || p.r >= DTB_BB_MIN_R || (p.r >= DTB_BB_MIN_R_LARGE && px >= (1ll << 26))))
            return launch_block(p, n_images, num_sms, st, print_plan());
    }
    Plan pl = plan_for(V);
    int best_w = pl.w, best_strips = pl.strips, best_tw = pl.tw;
    p.pad = p.padr = 0;
    // Edge-padded single strip (slide_kernel): an image no wider than one strip needs no halo
    // columns at all -- its left and right halos lie outside the image.  Taken when that cuts the
    // column work by >= 10% (C3, 2048 wide, W31: 5 strips x 512 columns -> one of 2048).
    if (!p.nseg && pad_mode()) {
        // V = 16 only: 32 columns per thread measured slower on every page that fits (C3 0.712 vs
        // 0.672 ms, C2 W15 0.136 vs 0.048 ms; scripts/pad_probe.py)
        const int Vp = 16;
        const int wp = (p.cols + 32 * Vp - 1) / (32 * Vp);
        const long workp = 32L * Vp * wp;
        // the halo plan it competes with: the V = 16 one where the rule below would take it
        // (C2's 2480-wide page is one 2560-column strip either way and stays on the halo layout,
        // measured 1-4% faster there)
        long halo_work = pl.work;
        if (!p.tmap && V == 32) {
            const Plan h16 = plan_for(16);
            if (h16.w > 0 && (pl.w == 0 || h16.work * 10 <= pl.work * 9)) halo_work = h16.work;
        }
        if (wp <= 8 && (pad_mode() == 1 || best_w == 0 || workp * 10 <= halo_work * 9)) {
            V = Vp;
            p.pad = 32 * ((p.rx + 31) / 32);
            p.padr = 4 * ((p.rx + 4) / 4 + 1);
            best_w = wp; best_strips = 1; best_tw = 32 * ((p.cols + 31) / 32);
        }
    }
    if (best_w == 0) return cudaErrorInvalidValue;  // window too wide for 8 warps (caller checks)
    // Auto V: 16 columns per thread give strips in 512-column steps (and 128-register warps);
    // take them when that cuts the staged column work by >= 10% (C2 pages 2480 wide: one strip
    // of 2560 instead of three of 1024 -- W15 0.119 -> 0.058 ms; C5 W3: 0.093 -> 0.078 ms;
    // C5 W67 / W131 within 2%).
    if (!p.nseg && !p.tmap && V == 32 && !p.pad) {
        const Plan p16 = plan_for(16);
        if (p16.w > 0 && p16.work * 10 <= pl.work * 9) {
            V = 16;
            best_w = p16.w; best_strips = p16.strips; best_tw = p16.tw;
        }
    }
    // warp-specialized kernel when the strip has >= 2 column warps (measured: C4 0.624 vs 0.656
    // ms; single-column-warp strips such as C3's are faster on the classic kernel)
    const int ws_mode = use_ws();
    if (V == 32 && !p.pad && (ws_mode == 1 || (ws_mode == 2 && best_w >= 2))) {
        p.ncw = best_w;
        p.now = (best_tw + 32 * 32 - 1) / (32 * 32);
        p.NC = 1024 * best_w;
        p.PL = p.NC;
        p.TW = best_tw;
        const int nt = 32 * (p.ncw + p.now);
        const size_t smem = ws_smem_bytes(p.NC);
        const int m = p.rx & 3;
        const bool sv = p.method == DTB_METHOD_SAUVOLA;
        int occ = 1;
        ws_dispatch(m, sv, dim3(), nt, smem, p, st, &occ);
        const int slots = num_sms * occ;
        int nbands = std::max(1, slots / std::max(1, best_strips * n_images));
        nbands = std::max(1, std::min(nbands, (rows_out + 7) / 8));  // one wave (the model measured
                                                                     // 1-4% slower here, C5 W195+)
        p.TH = (rows_out + nbands - 1) / nbands;
        dim3 grid(best_strips, (rows_out + p.TH - 1) / p.TH, n_images);
        if (print_plan())
            fprintf(stderr, "[dtb plan] ws_kernel cols=%d rows=%d r=%d w=%d strips=%d TW=%d occ=%d bands=%d TH=%d\n",
                    p.cols, rows_out, p.r, best_w, best_strips, best_tw, occ, (int)grid.y, p.TH);
        g_last_kernel = "ws_kernel";
        return ws_dispatch(m, sv, grid, nt, smem, p, st, nullptr);
    }
    const int nt = 32 * best_w;
    p.NC = V * nt;
    p.TW = best_tw;
    p.PL = p.pad ? p.pad + p.NC + p.padr + 16 : p.NC;
    const int nstrips = best_strips;
    const size_t smem = slide_smem_bytes(p.NC, p.PL);
    const int m = p.rx & 3;
    const bool sv = p.method == DTB_METHOD_SAUVOLA;
    int occ = 1;
    if (V == 16) dispatch_rx<16>(m, sv, dim3(), nt, smem, p, st, &occ);
    else dispatch_rx<32>(m, sv, dim3(), nt, smem, p, st, &occ);
    // cost-model band count (C3 0.949 -> 0.885 ms, C5 W19..W179 2-4% faster than one wave; a
    // band's warm-up costs 2r+1 rows of vertical work)
    const int slots = num_sms * occ;
    const int nbands = plan_bands(rows_out, nstrips * n_images, slots, p.r, 0.25, 0.1);
    p.TH = (rows_out + nbands - 1) / nbands;
    dim3 grid(nstrips, (rows_out + p.TH - 1) / p.TH, n_images);
    if (print_plan())
        fprintf(stderr, "[dtb plan] slide_kernel V=%d cols=%d rows=%d r=%d w=%d strips=%d TW=%d occ=%d bands=%d TH=%d pad=%d\n",
                V, p.cols, rows_out, p.r, best_w, nstrips, best_tw, occ, (int)grid.y, p.TH, p.pad);
    g_last_kernel = "slide_kernel";
    return V == 16 ? dispatch_rx<16>(m, sv, grid, nt, smem, p, st, nullptr)
                   : dispatch_rx<32>(m, sv, grid, nt, smem, p, st, nullptr);
}

}  // namespace dtb
