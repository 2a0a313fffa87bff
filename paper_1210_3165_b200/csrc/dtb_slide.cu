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
#include <cstdlib>
#include <cstdio>

#include "docthresh_b200.h"
#include "dtb_common.cuh"
#include "dtb_slide.cuh"
#include "dtb_async.cuh"

// Tuning switches (measured on B200, C4: quarters 0.662 vs 0.684 ms; a 3-lane producer 0.73 ms)
#ifndef DTB_PREFIX_QUARTERS
#define DTB_PREFIX_QUARTERS 1
#endif
#ifndef DTB_WS_DEFAULT
#define DTB_WS_DEFAULT 2  // 0 classic, 1 always warp-specialized, 2 auto
#endif
#ifndef DTB_ALU_BALANCE
#define DTB_ALU_BALANCE 0
#endif
// diagnostics only (wrong results): 1 = skip the output phase, 2 = skip prefix stores
#ifndef DTB_DIAG_SKIP
#define DTB_DIAG_SKIP 0
#endif
#ifndef DTB_D_SPLIT
#define DTB_D_SPLIT 0
#endif
#ifndef DTB_PAR_PRODUCER
#define DTB_PAR_PRODUCER 0
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
                    DTB_CHECK(aw[2 * g + q] >= 0 && aw[2 * g + q] + 4 <= slide_padded_words(p.NC));
                    const uint4 v = *reinterpret_cast<const uint4*>(sp + aw[2 * g + q]);
                    A[4 * q] = v.x; A[4 * q + 1] = v.y; A[4 * q + 2] = v.z; A[4 * q + 3] = v.w;
                }
                if (q < 2 || MB) {
                    DTB_CHECK(bw[2 * g + q] >= 0 && bw[2 * g + q] + 4 <= slide_padded_words(p.NC));
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
template <int V, int RXM4, bool BORDER>
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
            const double t = t_exact_fast(S8[j], Q8[j], n, rn, p.method, p.k, p.rr, rinv);
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
#ifndef DTB_SLIDE_MINB
#define DTB_SLIDE_MINB(V) ((V) == 16 ? 2 : 1)
#endif

// MX = method code | 4 for the segmented-input variant (dtb_binarize_segments)
template <int V, int RXM4, int MX>
__global__ void __launch_bounds__(256, DTB_SLIDE_MINB(V)) slide_kernel(SlideParams p) {
    constexpr int METHOD = MX & 3;
    constexpr bool SEG = (MX & 4) != 0;
    constexpr bool TMAP = (MX & 8) != 0;  // also write the fp64 threshold map (exact per pixel)
    constexpr int MA = (4 - RXM4) & 3;
    constexpr int MB = (RXM4 + 1) & 3;
    constexpr int NS = SLIDE_STAGES;
    extern __shared__ __align__(128) uint32_t sm[];
    const int NCp = slide_padded_words(p.NC);
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
    const int alpha = (16 - (p.rx & 15)) & 15;
    const int xc0 = X0 - p.rx - alpha;
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

    // warm-up items carry up to 3 warm-up rows each (E, O, F slots), as in gb_kernel
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
    // Lanes 0..2 of warp 0 issue the entering / leaving / centre copies in parallel; lane 0 also
    // arms the full barrier with the byte count (tx-count may transiently go negative).
    auto issue = [&](int k, int which) {
        const int s = k % NS;
        if (k >= NS) mbar_wait(&empty[s], ((k / NS) - 1) & 1);
        uint8_t* E = ring + (size_t)s * 3 * p.NC;
        uint8_t* O = E + p.NC;
        uint8_t* F = O + p.NC;
        int ge, go = -1, gf = -1;
        if (k < it.nwarm) {
            // warm-up rows g0+3k .. g0+3k+2 into the E, O, F slots (full strip width each)
            if ((!DTB_PAR_PRODUCER || which == 0)) {
                const uint32_t rowb = (uint32_t)(c_hi16 - c_lo);
                const int g = it.g0 + 3 * k, cnt = min(3, it.g0 + nwr - g);
                mbar_expect_tx(&full[s], (uint32_t)cnt * rowb);
                for (int i = 0; i < cnt; ++i) {
                    uint8_t* D = E + i * p.NC;
                    if (rowb) bulk_g2s(D + (c_lo - xc0), row_at<SEG>(p, in0, g + i) + c_lo, rowb, &full[s], pol_keep);
                    for (int c = c_hi16; c < c_hi; ++c) D[c - xc0] = row_at<SEG>(p, in0, g + i)[c];
                }
            }
            return;
        } else {
            const int y = it.ya + (k - it.nwarm);
            gf = y;
            ge = (k == it.nwarm) ? -1 : y + p.r;
            go = (k == it.nwarm) ? -1 : y - p.r - 1;
            if (ge >= p.H) ge = -1;
        }
        const uint32_t rowb = (uint32_t)(c_hi16 - c_lo), fb = (uint32_t)(f_hi16 - X0);
        if (!DTB_PAR_PRODUCER) {
            uint32_t bytes = 0;
            if (ge >= 0) bytes += rowb;
            if (go >= 0) bytes += rowb;
            if (gf >= 0) bytes += fb;
            mbar_expect_tx(&full[s], bytes);
            if (ge >= 0 && rowb)
                bulk_g2s(E + (c_lo - xc0), row_at<SEG>(p, in0, ge) + c_lo, rowb, &full[s], pol_keep);
            if (go >= 0 && rowb)
                bulk_g2s(O + (c_lo - xc0), row_at<SEG>(p, in0, go) + c_lo, rowb, &full[s], pol_drop);
            if (gf >= 0 && fb) bulk_g2s(F, row_at<SEG>(p, in0, gf) + X0, fb, &full[s], pol_keep);
            for (int c = c_hi16; c < c_hi; ++c) {
                if (ge >= 0) E[c - xc0] = row_at<SEG>(p, in0, ge)[c];
                if (go >= 0) O[c - xc0] = row_at<SEG>(p, in0, go)[c];
            }
            for (int c = f_hi16; c < f_hi; ++c)
                if (gf >= 0) F[c - X0] = row_at<SEG>(p, in0, gf)[c];
        } else if (which == 0) {
            uint32_t bytes = 0;
            if (ge >= 0) bytes += rowb;
            if (go >= 0) bytes += rowb;
            if (gf >= 0) bytes += fb;
            mbar_expect_tx(&full[s], bytes);
            if (ge >= 0 && rowb)
                bulk_g2s(E + (c_lo - xc0), row_at<SEG>(p, in0, ge) + c_lo, rowb, &full[s], pol_keep);
            for (int c = c_hi16; c < c_hi; ++c) {
                if (ge >= 0) E[c - xc0] = row_at<SEG>(p, in0, ge)[c];
                if (go >= 0) O[c - xc0] = row_at<SEG>(p, in0, go)[c];
            }
            for (int c = f_hi16; c < f_hi; ++c)
                if (gf >= 0) F[c - X0] = row_at<SEG>(p, in0, gf)[c];
        } else if (which == 1) {
            if (go >= 0 && rowb)
                bulk_g2s(O + (c_lo - xc0), row_at<SEG>(p, in0, go) + c_lo, rowb, &full[s], pol_drop);
        } else {
            if (gf >= 0 && fb) bulk_g2s(F, row_at<SEG>(p, in0, gf) + X0, fb, &full[s], pol_keep);
        }
    };
    const bool producer = DTB_PAR_PRODUCER ? (warp == 0 && lane < 3) : (t == 0);
    if (producer)
        for (int k = 0; k < min(NS - 1, it.n); ++k) issue(k, lane);

    uint32_t cS[V], cQ[V];
#pragma unroll
    for (int j = 0; j < V; ++j) { cS[j] = 0; cQ[j] = 0; }
    // per-quarter totals of cS / cQ (V/4 columns each), kept incrementally: the thread total
    // feeds the scan, and the quarter totals let the prefix run as 4 independent chains
    uint32_t qS[4] = {0, 0, 0, 0}, qQ[4] = {0, 0, 0, 0};

    const int xo = X0 + V * t;  // this thread's V output columns
    const bool has_out = (V * t + V + 2 * p.rx + alpha <= p.NC) && (V * t < p.TW) &&
                         (xo < p.cols);
    const bool out_full = has_out && (xo + 32 <= p.cols) &&
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
        if (producer && k + NS - 1 < it.n) issue(k + NS - 1, lane);
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
#if DTB_ALU_BALANCE
            cS[j] = cS[j] + ev - ov;                 // IADD3 (ALU pipe)
            const uint32_t nov = 0u - ov;            // IADD3
            cQ[j] = ev * ev + cQ[j];                 // IMAD
            cQ[j] = nov * ov + cQ[j];                // IMAD
#else
            const uint32_t dv = ev - ov;
            cS[j] += dv;
            cQ[j] += dv * (ev + ov);
#endif
        }
        if (lane == 31) { sWS[warp] = iS; sWQ[warp] = iQ; }
        __syncthreads();
        if (producer && k + NS - 1 < it.n) issue(k + NS - 1, lane);
        uint32_t bS = iS - TS, bQ = iQ - TQ;
        for (int w = 0; w < warp; ++w) { bS += sWS[w]; bQ += sWQ[w]; }
#if DTB_PREFIX_QUARTERS
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
#if DTB_ALU_BALANCE
                // P[j+1] = P[j-1] + c[j] + c[j+1]: 3-input adds (IADD3) halve the chain depth
                vs.x = cbS[h]; vq.x = cbQ[h];
                vs.y = cbS[h] + cS[c0]; vq.y = cbQ[h] + cQ[c0];
                vs.z = cbS[h] + cS[c0] + cS[c0 + 1]; vq.z = cbQ[h] + cQ[c0] + cQ[c0 + 1];
                vs.w = vs.y + cS[c0 + 1] + cS[c0 + 2]; vq.w = vq.y + cQ[c0 + 1] + cQ[c0 + 2];
                cbS[h] = vs.z + cS[c0 + 2] + cS[c0 + 3]; cbQ[h] = vq.z + cQ[c0 + 2] + cQ[c0 + 3];
#else
                vs.x = cbS[h]; vq.x = cbQ[h];
                cbS[h] += cS[c0]; cbQ[h] += cQ[c0];
                vs.y = cbS[h]; vq.y = cbQ[h];
                cbS[h] += cS[c0 + 1]; cbQ[h] += cQ[c0 + 1];
                vs.z = cbS[h]; vq.z = cbQ[h];
                cbS[h] += cS[c0 + 2]; cbQ[h] += cQ[c0 + 2];
                vs.w = cbS[h]; vq.w = cbQ[h];
                cbS[h] += cS[c0 + 3]; cbQ[h] += cQ[c0 + 3];
#endif
                const int pw = pchunk_word((V / 4) * t + c0 / 4);
                DTB_CHECK(pw >= 0 && pw + 4 <= NCp);
                if (!(DTB_DIAG_SKIP & 2)) {
                    *reinterpret_cast<uint4*>(&sPS[pw]) = vs;
                    *reinterpret_cast<uint4*>(&sPQ[pw]) = vq;
                }
            }
        }
#else
        // logical word Vt + m holds P[Vt + m - 1]: the first slot is this thread's base
#pragma unroll
        for (int j = 0; j < V; j += 4) {
            uint4 vs, vq;
            vs.x = bS; vq.x = bQ;
            bS += cS[j]; bQ += cQ[j];
            vs.y = bS; vq.y = bQ;
            bS += cS[j + 1]; bQ += cQ[j + 1];
            vs.z = bS; vq.z = bQ;
            bS += cS[j + 2]; bQ += cQ[j + 2];
            vs.w = bS; vq.w = bQ;
            bS += cS[j + 3]; bQ += cQ[j + 3];
            const int pw = pchunk_word((V / 4) * t + j / 4);
            *reinterpret_cast<uint4*>(&sPS[pw]) = vs;
            *reinterpret_cast<uint4*>(&sPQ[pw]) = vq;
        }
#endif
        if (t == blockDim.x - 1) {  // logical word NC = P[NC - 1]
            const int pw = pchunk_word(p.NC / 4);
            sPS[pw] = bS;
            sPQ[pw] = bQ;
        }
        __syncthreads();

        // ---- outputs
        if (has_out && !(DTB_DIAG_SKIP & 1)) {
            const bool y_interior = (y - p.r >= 0) && (y + p.r <= p.H - 1);
            uint8_t* orow = obase + (int64_t)y * p.bin_pitch;
            const int ny = min(y + p.r, p.H - 1) - max(y - p.r, 0) + 1;
            const uint8_t* fsm = stage + 2 * p.NC + V * t;
            bool unc = false;
            uint32_t ow[V / 4];
            if constexpr (TMAP) {
                double* trow = reinterpret_cast<double*>(reinterpret_cast<uint8_t*>(p.tmap) +
                                                         (y - p.out_begin) * p.tmap_pitch) + xo;
                if (y_interior && !x_border_warp)
                    row_outputs_tmap<V, RXM4, false>(sPS, sPQ, aw, bw, fsm, ow, trow, xo, p.cols, ny,
                                                     p.r, p, rnN, rinv);
                else
                    row_outputs_tmap<V, RXM4, true>(sPS, sPQ, aw, bw, fsm, ow, trow, xo, p.cols, ny,
                                                    p.r, p, rnN, rinv);
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


#ifndef DTB_WS_V16_DEFAULT
#define DTB_WS_V16_DEFAULT 0  // C4: 0.759 ms with V = VO = 16 (24 warps/SM) vs 0.609 with 32 (12)
#endif

#ifndef DTB_WS_UNIFORM_OFFS
#define DTB_WS_UNIFORM_OFFS 0  // C4: 0.6165 (1) vs 0.6086 (0) ms -- the compiler keeps them per-thread anyway
#endif

#ifndef DTB_WS_ISSUE_POS
#define DTB_WS_ISSUE_POS 2  // C4: 0.6122 (2) vs 0.6153 (0) vs 0.674 (1) ms at 4 stages
#endif

#ifndef DTB_WS_SWAP_BUILD
#define DTB_WS_SWAP_BUILD 0
#endif

// Warm-up split: the 2r+1 rows that prime a band's column sums are consumed alternately by
// the column warps (even items) and the otherwise idle output warps (odd items, partial sums
// for the same columns), which hand their partials over through the not-yet-used prefix area.
#ifndef DTB_WS_SPLIT_WARM
#define DTB_WS_SPLIT_WARM 0  // measured no gain on C4 (0.6157 vs 0.6149 ms); kept for A/B
#endif

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

    // Logical thread index.  Warp w of a CTA issues from SM sub-partition w % 4, so with
    // fixed role slots every sub-partition would host one role only (column warps idle at
    // barriers on two of them while output warps saturate the other two).  Alternate groups
    // of CTAs (role_div = SMs, i.e. one group per residency wave) put the output role first.
    const int tp = threadIdx.x;
#if DTB_WS_SWAP_BUILD
    const int bid = (int)(blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z));
    const bool swap = p.role_div > 0 && ((bid / p.role_div) & 1);
    const int t = swap ? (tp < 32 * now ? tp + 32 * ncw : tp - 32 * now) : tp;
#else
    const int t = tp;  // role slots fixed (the swap measured slower; build with -DDTB_WS_SWAP_BUILD=1)
#endif
    const int lane = tp & 31, warp = t >> 5;
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
    // warm-up items carry up to 3 warm-up rows each (E, O, F slots), as in gb_kernel
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
    auto issue = [&](int k) {
        const int s = k % NS;
        if (k >= NS) mbar_wait(&empty[s], ((k / NS) - 1) & 1);
        uint8_t* E = ring + (size_t)s * 3 * p.NC;
        uint8_t* O = E + p.NC;
        uint8_t* F = O + p.NC;
        int ge, go = -1, gf = -1;
        if (k < it.nwarm) {
            // warm-up rows g0+3k .. g0+3k+2 into the E, O, F slots (full strip width each)
            if (true) {
                const uint32_t rowb = (uint32_t)(c_hi16 - c_lo);
                const int g = it.g0 + 3 * k, cnt = min(3, it.g0 + nwr - g);
                mbar_expect_tx(&full[s], (uint32_t)cnt * rowb);
                for (int i = 0; i < cnt; ++i) {
                    uint8_t* D = E + i * p.NC;
                    if (rowb) bulk_g2s(D + (c_lo - xc0), row_at<SEG>(p, in0, g + i) + c_lo, rowb, &full[s], pol_keep);
                    for (int c = c_hi16; c < c_hi; ++c) D[c - xc0] = row_at<SEG>(p, in0, g + i)[c];
                }
            }
            return;
        } else {
            const int y = it.ya + (k - it.nwarm);
            gf = y;
            ge = (k == it.nwarm) ? -1 : y + p.r;
            go = (k == it.nwarm) ? -1 : y - p.r - 1;
            if (ge >= p.H) ge = -1;
        }
        const uint32_t rowb = (uint32_t)(c_hi16 - c_lo), fb = (uint32_t)(f_hi16 - X0);
        uint32_t bytes = 0;
        if (ge >= 0) bytes += rowb;
        if (go >= 0) bytes += rowb;
        if (gf >= 0) bytes += fb;
        mbar_expect_tx(&full[s], bytes);
        if (ge >= 0 && rowb)
            bulk_g2s(E + (c_lo - xc0), row_at<SEG>(p, in0, ge) + c_lo, rowb, &full[s], pol_keep);
        if (go >= 0 && rowb)
            bulk_g2s(O + (c_lo - xc0), row_at<SEG>(p, in0, go) + c_lo, rowb, &full[s], pol_drop);
        if (gf >= 0 && fb) bulk_g2s(F, row_at<SEG>(p, in0, gf) + X0, fb, &full[s], pol_keep);
        for (int c = c_hi16; c < c_hi; ++c) {
            if (ge >= 0) E[c - xc0] = row_at<SEG>(p, in0, ge)[c];
            if (go >= 0) O[c - xc0] = row_at<SEG>(p, in0, go)[c];
        }
        for (int c = f_hi16; c < f_hi; ++c)
            if (gf >= 0) F[c - X0] = row_at<SEG>(p, in0, gf)[c];
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
        // warm-up split: column warp c has a helper (output warp c) when c < now; helped warps
        // take the even items only, unhelped ones every item.  Arrivals per item stay ncw + now.
        const bool split = DTB_WS_SPLIT_WARM && it.nwarm > 1;
        const int nh = min(ncw, now);  // helped column warps
        const bool helped = split && warp < nh;
        for (int k = 0; k < it.nwarm; k += helped ? 2 : 1) {
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
            // even items: warp 0 also arrives for the output warps; odd items (unhelped warps
            // only): the output warps arrive for the helped column warps
            if (lane == 0)
                mbar_arrive_cnt(&empty[s], (warp == 0 && (!split || (k & 1) == 0)) ? 1 + now : 1);
            if (t == 0)
                while (issued < min(k + NS, it.n)) issue(issued++);
        }
#if DTB_WS_SPLIT_WARM
        if (split) {
            nbar_sync(BAR_WARM, nthr);  // the helpers' partial sums (odd items) are in smem
            if (helped) {
                const uint4* hp = reinterpret_cast<const uint4*>(sm + 2 * V * t);
#pragma unroll
                for (int q = 0; q < V / 4; ++q) {
                    const uint4 a = hp[q], b = hp[V / 4 + q];
                    cS[4 * q] += a.x; cS[4 * q + 1] += a.y; cS[4 * q + 2] += a.z; cS[4 * q + 3] += a.w;
                    cQ[4 * q] += b.x; cQ[4 * q + 1] += b.y; cQ[4 * q + 2] += b.z; cQ[4 * q + 3] += b.w;
                }
            }
        }
#endif
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
            // Row staging for a later row.  Issuing item j needs item j-NS released by every
            // warp; FREE(k-2) guarantees that for j <= k+NS-2, so ISSUE_POS 1 never stalls the
            // producer here, while ISSUE_POS 0 (lookahead NS-1) can hold column warp 0 -- and
            // with it READY(k) -- until the output warps finish row k-1.
            if (DTB_WS_ISSUE_POS == 0 && t == 0)
                while (issued < min(k + NS - 1, it.n)) issue(issued++);
            if (DTB_WS_ISSUE_POS == 1 && t == 0)
                while (issued < min(k + NS - 2, it.n)) issue(issued++);
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
            if (DTB_WS_ISSUE_POS == 2 && t == 0)  // after publishing row k: off READY's path
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
#if DTB_WS_UNIFORM_OFFS
        // Run chunk addresses = per-thread base + launch-uniform offsets: thread `to`'s A run
        // starts at chunk 8*to + dA (dA = (alpha - MA)/4 in 0..3, the same for every thread),
        // and pchunk_word(8*to + d) = 36*to + 4*(d + d/8) for d >= 0, so the compiler can keep
        // the 2 x 9 offsets in uniform registers instead of per-thread ones.
        static_assert(VO == 32, "uniform run offsets assume 8 chunks per output thread");
        const int dA = (alpha - MA) >> 2, dB = (alpha + 2 * p.rx + 1 - MB) >> 2;
        const int tb = 36 * to;
        int aw[VO / 4 + 1], bw[VO / 4 + 1];
#pragma unroll
        for (int i = 0; i < VO / 4 + 1; ++i) {
            aw[i] = tb + 4 * (dA + i + ((dA + i) >> 3));
            bw[i] = tb + 4 * (dB + i + ((dB + i) >> 3));
            DTB_CHECK(aw[i] == pchunk_word(((alpha + VO * to - MA) >> 2) + i));
            DTB_CHECK(bw[i] == pchunk_word(((alpha + 2 * p.rx + 1 + VO * to - MB) >> 2) + i));
        }
#else
        const int la0 = (alpha + VO * to - MA) >> 2;
        const int lb0 = (alpha + 2 * p.rx + 1 + VO * to - MB) >> 2;
        int aw[VO / 4 + 1], bw[VO / 4 + 1];
#pragma unroll
        for (int i = 0; i < VO / 4 + 1; ++i) { aw[i] = pchunk_word(la0 + i); bw[i] = pchunk_word(lb0 + i); }
#endif
        const bool x_border_warp = __any_sync(0xffffffffu, has_out && !x_interior);
        uint8_t* obase = p.bin + (int64_t)blockIdx.z * p.out_stride - (int64_t)p.out_begin * p.bin_pitch;
#if DTB_WS_SPLIT_WARM
        if (it.nwarm > 1) {
            // odd warm-up items: partial column sums for column thread `to`'s columns
            const int nh = min(ncw, now);
            const bool helper = to < 32 * nh;
            uint32_t hS[V], hQ[V];
#pragma unroll
            for (int j = 0; j < V; ++j) { hS[j] = 0; hQ[j] = 0; }
            for (int k = 1; k < it.nwarm; k += 2) {
                const int s = k % NS;
                mbar_wait(&full[s], (k / NS) & 1);
                if (helper) {
                    for (int i = 0; i < min(3, nwr - 3 * k); ++i) {
                        const uint4* E = reinterpret_cast<const uint4*>(ring + (size_t)s * 3 * p.NC + i * p.NC + V * to);
                        uint32_t w[V / 4];
#pragma unroll
                        for (int q = 0; q < V / 16; ++q) {
                            const uint4 a = E[q];
                            w[4 * q] = a.x; w[4 * q + 1] = a.y; w[4 * q + 2] = a.z; w[4 * q + 3] = a.w;
                        }
#pragma unroll
                        for (int j = 0; j < V; ++j) {
                            const uint32_t v = byte_at(w, j);
                            hS[j] += v;
                            hQ[j] += v * v;
                        }
                    }
                }
                __syncwarp();
                // output warp 0 arrives for the helped column warps, which skip odd items
                if (lane == 0) mbar_arrive_cnt(&empty[s], (to >> 5) == 0 ? 1 + nh : 1);
            }
            if (helper) {
                uint4* hp = reinterpret_cast<uint4*>(sm + 2 * V * to);
#pragma unroll
                for (int q = 0; q < V / 4; ++q) {
                    hp[q] = make_uint4(hS[4 * q], hS[4 * q + 1], hS[4 * q + 2], hS[4 * q + 3]);
                    hp[V / 4 + q] = make_uint4(hQ[4 * q], hQ[4 * q + 1], hQ[4 * q + 2], hQ[4 * q + 3]);
                }
            }
            nbar_arrive(BAR_WARM, nthr);
        }
#endif
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

// =====================================================================================
// Group-bound kernel (gb_kernel, Sauvola with 0 < k <= 1).  Warp-specialised like ws_kernel
// (same ring, same READY/FREE hand-off), with a leaner column phase and a different output
// phase:
//
// * Residue-decimated prefix layout.  Word k of a prefix array (k in [0, NC]; word k = sum of
//   strip columns [0, k)) lives in plane rho = k & 3 at dec index m = k >> 2.  Dec index m
//   belongs to column lane t = m >> 3, half hh = (m >> 2) & 1, element m & 3, stored at
//   plane + 4*(hh*(T+1) + t) + (m & 3) (T column lanes).  A column lane writes its 32 words
//   as 8 STS.128 (two per plane) and an output lane reads every 4th word of a run -- the only
//   words the group bounds need -- as 2-3 LDS.128 per stream.  Both are bank-conflict free.
//
// * Group bounds.  For 4 adjacent outputs x0..x0+3 the window sums satisfy, because the
//   column sums are >= 0 (prefix words are nondecreasing),
//       S_I <= S(x) <= S_U,   Q(x) <= Q_U
//   with I = [x0+3-r, x0+r] (intersection of the 4 windows) and U = [x0-r, x0+3+r] (union):
//       S_U = P[b+3] - P[a],  S_I = P[b] - P[a+3],  Q_U = PQ[b+3] - PQ[a]   (a, b: run starts).
//   Sauvola's t = m (1-k) + (k/R) m s is nondecreasing in s and, for 0 <= 1-k, in m, so
//       t_lo = m_lo (1-k) <= t <= t_hi = m_hi ((1-k) + (k/R) sqrt(Q_U/n_lo - m_lo^2))
//   (m_lo = S_I/n_hi, m_hi = S_U/n_lo; n_lo..n_hi the pixels' counts).  Evaluated in fp32
//   with directed slack (relative 2^-17 on every factor, 1e-4 absolute) the bounds also
//   enclose the reference's fp64 threshold.  A pixel with f < ceil(t_lo) is black, one with
//   f >= ceil(t_hi) is white (f is an integer); the compare runs on 16-bit SWAR lanes, four
//   pixels per handful of instructions.  Pixels in [ceil(t_lo), ceil(t_hi)) are uncertain:
//   their group is re-decided per pixel (exact S, Q from the prefix -> certified fp32 ->
//   fp64 replay), out of line.  On document pages this is ~1e-5 of the groups at W=127.
// =====================================================================================
#ifndef GB_STAGES
#define GB_STAGES 3  // with 128 registers: 4 CTAs per SM (C4: 0.498 vs 0.584 ms at 5 stages, 168 regs, 3 CTAs)
#endif
#ifndef DTB_GB_MAXREG
#define DTB_GB_MAXREG 128
#endif


#ifndef GB_NCW
#define GB_NCW 2  // column warps (= output warps) per CTA; NC = 1024 * GB_NCW strip columns
#endif
#define GB_NC (1024 * GB_NCW)
// words of one residue plane: 2 rows of (T+1) chunks
__host__ __device__ constexpr int gb_plane_words(int NC) { return 8 * (NC / 32 + 1); }

__host__ __device__ inline size_t gb_smem_bytes(int NC) {
    // 2 buffers x (S, Q) x 4 planes, warp totals, 2*NS mbarriers, NS stages x 3 row segments
    return sizeof(uint32_t) * (16 * (size_t)gb_plane_words(NC) + 32) + 2 * GB_STAGES * sizeof(uint64_t) +
           (size_t)GB_STAGES * 3 * NC;
}

// word k of a residue-decimated prefix array (rare paths only)
__device__ __forceinline__ uint32_t gb_word(const uint32_t* arr, int PW, int T1, int k) {
    const int m = k >> 2;
    return arr[(k & 3) * PW + 4 * (((m >> 2) & 1) * T1 + (m >> 3)) + (m & 3)];
}

// 8 consecutive dec words m0..m0+7 of one plane, m0 = 8*t0 + D (D compile-time, 0..7)
template <int D>
__device__ __forceinline__ void gb_stream(const uint32_t* plane, int t0, int T1, uint32_t (&w)[8]) {
    constexpr int MU = D & 3;
    const uint32_t* c0 = plane + 4 * ((D < 4 ? 0 : T1) + t0);
    const uint32_t* c1 = plane + 4 * ((D < 4 ? T1 : 0) + t0 + (D < 4 ? 0 : 1));
    const uint32_t* c2 = plane + 4 * ((D < 4 ? 0 : T1) + t0 + 1);
    uint32_t v[12];
    {
        const uint4 x = *reinterpret_cast<const uint4*>(c0);
        v[0] = x.x; v[1] = x.y; v[2] = x.z; v[3] = x.w;
        const uint4 y = *reinterpret_cast<const uint4*>(c1);
        v[4] = y.x; v[5] = y.y; v[6] = y.z; v[7] = y.w;
        if (MU) {
            const uint4 z = *reinterpret_cast<const uint4*>(c2);
            v[8] = z.x; v[9] = z.y; v[10] = z.z; v[11] = z.w;
        } else {
            v[8] = v[9] = v[10] = v[11] = 0;
        }
    }
#pragma unroll
    for (int g = 0; g < 8; ++g) w[g] = v[MU + g];
}

// ceil(x) for x in (-0.5, 2^22) as a pair of 16-bit lanes (x, x): FADD.RP onto 2^23 leaves
// 2^23 + ceil(x), whose bit pattern minus 0x4B000000 is ceil(x); the IMAD replicates it.
__device__ __forceinline__ uint32_t gb_ceil2(float x) {
    const uint32_t bits = __float_as_uint(__fadd_ru(x, 8388608.0f));
    return bits * 0x10001u - 0x4B000000u * 0x10001u;
}

// Uncertain group of 4 pixels x0..x0+3 (gb_kernel), out of line.  First a tighter lower
// bound: the window contains the group's intersection window I, and a subset's squared
// deviations about its own mean bound the window's from below, so var >= (n_I/n) var_I
// (var_I = Q_I/n_I - m_I^2, evaluated lowered) and t >= m_lo ((1-k) + (k/R) s_lo).  Pixels the
// refined bounds still leave open get exact S, Q from the residue-decimated prefix, the
// certified fp32 decision and, within tol, the reference fp64 replay.  All four bytes are
// rewritten after the caller's vector stores (program order).
__device__ __noinline__ void gb_fix_group(const uint32_t* sPS, const uint32_t* sPQ, int PW, int T1,
                                          int a_word, int b_word, const uint8_t* f4, uint8_t* orow,
                                          int x0, int cols, int ny, int r, float cA, float cC,
                                          float ca, float cc, float tol, double kk, double rr) {
    const float kUp = 1.0f + 7.62939453125e-6f, kDn = 1.0f - 7.62939453125e-6f;  // 1 +- 2^-17
    int nmin = 1 << 30, nmax = 0;
    for (int i = 0; i < 4; ++i) {
        const int x = x0 + i;
        const int nx = min(x + r, cols - 1) - max(x - r, 0) + 1;
        nmin = min(nmin, nx); nmax = max(nmax, nx);
    }
    nmin = max(nmin, 1);
    const float rlo = rcp_ftz((float)(ny * nmin)) * kUp, rhi = rcp_ftz((float)(ny * nmax)) * kDn;
    const uint32_t pa0 = gb_word(sPS, PW, T1, a_word), pa3 = gb_word(sPS, PW, T1, a_word + 3);
    const uint32_t pb0 = gb_word(sPS, PW, T1, b_word), pb3 = gb_word(sPS, PW, T1, b_word + 3);
    const uint32_t qa0 = gb_word(sPQ, PW, T1, a_word), qa3 = gb_word(sPQ, PW, T1, a_word + 3);
    const uint32_t qb0 = gb_word(sPQ, PW, T1, b_word), qb3 = gb_word(sPQ, PW, T1, b_word + 3);
    const float fSI = (float)(pb0 - pa3);
    const float mhi = (float)(pb3 - pa0) * rlo, mlo = fSI * rhi;
    const float v = __fmaf_rn((float)(qb3 - qa0), rlo, -(mlo * mlo));
    const float thi = fminf(__fmaf_rn(mhi, __fmaf_rn(sqrt_ftz(fmaxf(v, 0.f)), cc, ca), tol), 4096.f);
    const int nxI = min(x0 + r, cols - 1) - max(x0 + 3 - r, 0) + 1;
    float sl = 0.f;
    if (nxI >= 1) {
        const float nI = (float)(ny * nxI), rnI = rcp_ftz(nI);
        const float mI = fSI * (rnI * kUp);
        const float vI = __fmaf_rn((float)(qb0 - qa3), rnI * kDn, -(mI * mI));
        sl = sqrt_ftz(fmaxf(vI, 0.f) * (nI * rhi));
    }
    const float tlo = __fmaf_rn(mlo, __fmaf_rn(sl, cc * kDn, ca), -tol);
    for (int i = 0; i < 4; ++i) {
        const int x = x0 + i;
        if (x >= cols) break;
        const uint32_t f = f4[i];
        uint32_t white;
        if ((float)f < tlo) {
            white = 0u;
        } else if ((float)f >= thi) {
            white = 0xFFu;
        } else {
            const uint32_t S = gb_word(sPS, PW, T1, b_word + i) - gb_word(sPS, PW, T1, a_word + i);
            const uint32_t Q = gb_word(sPQ, PW, T1, b_word + i) - gb_word(sPQ, PW, T1, a_word + i);
            const int nx = min(x + r, cols - 1) - max(x - r, 0) + 1;
            const uint32_t n = (uint32_t)(ny * nx);
            const float d = fast_diff<DTB_METHOD_SAUVOLA, true>(S, Q, f, n, cA, cC, ca, cc);
            if (fabsf(d) >= tol) {
                white = d < 0.f ? 0u : 0xFFu;
            } else {
                white = exact_white(S, Q, (double)n, f, DTB_METHOD_SAUVOLA, kk, rr);
                if (unsigned long long* audit = g_fp32_audit) {
                    atomicAdd(&audit[0], 1ull);
                    if (white != (d < 0.f ? 0u : 0xFFu)) atomicAdd(&audit[1], 1ull);
                }
            }
        }
        orow[x] = (uint8_t)white;
    }
}

// DTB_GB_TIMES=1 (debug): per-CTA start/end %globaltimer, printed by the launcher.
__device__ unsigned long long g_gb_times[2 * 8192];
__device__ int g_gb_times_on = 0;
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

// R16 = r & 15 (fixes every stream's alignment); interior rows/lanes use n = (2r+1)^2.
// SEG: segmented input (dtb_binarize_segments, e.g. halo rows read in place from a
// neighbour GPU's band over NVLink); a compile-time variant like ws_kernel's.
template <int R16, bool SEG>
__global__ void __maxnreg__(DTB_GB_MAXREG) gb_kernel(SlideParams p) {
    constexpr int NS = GB_STAGES;
    constexpr int ALPHA = (16 - R16) & 15;
    constexpr int EB = (ALPHA + 2 * R16 + 1) & 31;  // (alpha + 2r + 1) mod 32
    // compile-time dec offsets (mod 8) of the six streams
    constexpr int D_A0 = (ALPHA >> 2) & 7, D_A3 = ((ALPHA + 3) >> 2) & 7;
    constexpr int D_B0 = (EB >> 2) & 7, D_B3 = ((EB + 3) >> 2) & 7;
    constexpr int R_A0 = ALPHA & 3, R_A3 = (ALPHA + 3) & 3, R_B0 = EB & 3, R_B3 = (EB + 3) & 3;
    extern __shared__ __align__(128) uint32_t sm[];
    constexpr int NC = GB_NC;  // GB_NCW column warps (the host launches with ncw = now = GB_NCW)
    constexpr int PW = gb_plane_words(NC);
    constexpr int T = NC / 32, T1 = T + 1;
    uint32_t* sWS = sm + 16 * PW;  // [2][8] per-column-warp totals, double buffered
    uint32_t* sWQ = sWS + 16;
    uint64_t* full = reinterpret_cast<uint64_t*>(sWS + 32);
    uint64_t* empty = full + NS;
    uint8_t* ring = reinterpret_cast<uint8_t*>(empty + NS);
    const int ncw = p.ncw, now = p.now, nthr = 32 * (ncw + now);
    const int bid = (int)(blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z));
    // Warp w issues from SM sub-partition w % 4, so fixed role slots put each role on two
    // sub-partitions only; with role_div > 0, alternate groups of role_div CTAs swap the slots
    // (column warps on sub-partitions 2, 3) so co-resident CTAs spread both roles.
    const bool swap = p.role_div > 0 && ((bid / p.role_div) & 1);
    const int t = swap ? (int)(threadIdx.x ^ (32u * GB_NCW)) : (int)threadIdx.x;  // ncw = now
    const int lane = t & 31, warp = t >> 5;
    const bool is_col = warp < ncw;
    if (g_gb_times_on && t == 0 && bid < 8192) g_gb_times[2 * bid] = gtimer();
    const uint8_t* in = p.in + (int64_t)blockIdx.z * p.img_stride;
    const int X0 = (int)blockIdx.x * p.TW;
    const int xc0 = X0 - p.r - ALPHA;
    const int ya = p.out_begin + (int)blockIdx.y * p.TH;
    const int yb = min(ya + p.TH, p.out_end);
    if (ya >= yb) return;
    const uint8_t* in0 = in - (int64_t)p.row0 * p.pitch;
    const int c_lo = max(xc0, 0);
    const int c_hi = min(xc0 + NC, p.cols);
    const int c_hi16 = c_lo + ((max(c_hi - c_lo, 0)) & ~15);
    const int f_hi = min(X0 + p.TW, p.cols);
    const int f_hi16 = X0 + ((max(f_hi - X0, 0)) & ~15);
    // Items: warm-up items first, each carrying up to three warm-up rows (in the entering,
    // leaving and centre slots -- a warm-up row needs only its bytes), then one item per output
    // row.  Packing triples the warm-up rows in flight on the 3-stage ring.
    Items it;
    it.g0 = max(ya - p.r, 0);
    const int nwr = min(ya + p.r, p.H - 1) - it.g0 + 1;  // warm-up rows
    it.nwarm = (nwr + 2) / 3;                             // warm-up items
    it.ya = ya;
    it.n = it.nwarm + (yb - ya);

    {
        uint4* r4 = reinterpret_cast<uint4*>(ring);
        const int n16 = NS * 3 * NC / 16;
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
    auto issue = [&](int k) {
        const int s = k % NS;
        if (k >= NS) mbar_wait(&empty[s], ((k / NS) - 1) & 1);
        uint8_t* E = ring + (size_t)s * 3 * NC;
        uint8_t* O = E + NC;
        uint8_t* F = O + NC;
        int ge, go = -1, gf = -1;
        if (k < it.nwarm) {
            // warm-up rows g0+3k .. g0+3k+2 into the E, O, F slots (full strip width each)
            const uint32_t rowb = (uint32_t)(c_hi16 - c_lo);
            const int g = it.g0 + 3 * k, cnt = min(3, it.g0 + nwr - g);
            mbar_expect_tx(&full[s], (uint32_t)cnt * rowb);
            for (int i = 0; i < cnt; ++i) {
                uint8_t* D = E + i * NC;
                if (rowb) bulk_g2s(D + (c_lo - xc0), row_at<SEG>(p, in0, g + i) + c_lo, rowb, &full[s], pol_keep);
                for (int c = c_hi16; c < c_hi; ++c) D[c - xc0] = row_at<SEG>(p, in0, g + i)[c];
            }
            return;
        } else {
            const int y = it.ya + (k - it.nwarm);
            gf = y;
            ge = (k == it.nwarm) ? -1 : y + p.r;
            go = (k == it.nwarm) ? -1 : y - p.r - 1;
            if (ge >= p.H) ge = -1;
        }
        const uint32_t rowb = (uint32_t)(c_hi16 - c_lo), fb = (uint32_t)(f_hi16 - X0);
        uint32_t bytes = 0;
        if (ge >= 0) bytes += rowb;
        if (go >= 0) bytes += rowb;
        if (gf >= 0) bytes += fb;
        mbar_expect_tx(&full[s], bytes);
        if (ge >= 0 && rowb) bulk_g2s(E + (c_lo - xc0), row_at<SEG>(p, in0, ge) + c_lo, rowb, &full[s], pol_keep);
        if (go >= 0 && rowb) bulk_g2s(O + (c_lo - xc0), row_at<SEG>(p, in0, go) + c_lo, rowb, &full[s], pol_drop);
        if (gf >= 0 && fb) bulk_g2s(F, row_at<SEG>(p, in0, gf) + X0, fb, &full[s], pol_keep);
        for (int c = c_hi16; c < c_hi; ++c) {
            if (ge >= 0) E[c - xc0] = row_at<SEG>(p, in0, ge)[c];
            if (go >= 0) O[c - xc0] = row_at<SEG>(p, in0, go)[c];
        }
        for (int c = f_hi16; c < f_hi; ++c)
            if (gf >= 0) F[c - X0] = row_at<SEG>(p, in0, gf)[c];
    };

    // The producer is lane 0 of the first OUTPUT warp: it refills a ring slot once all four
    // warps released it, so a column warp never blocks on the output warps' progress (a
    // column-warp producer stalled READY(k) behind output row k-1).
    const bool producer = (t == 32 * ncw);
    if (is_col) {
        // ===================== column warps =====================
        uint32_t cS[32], cQ[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) { cS[j] = 0; cQ[j] = 0; }
        for (int k = 0; k < it.nwarm; ++k) {
            const int s = k % NS;
            mbar_wait(&full[s], (k / NS) & 1);
            const int cnt = min(3, nwr - 3 * k);
            for (int i = 0; i < cnt; ++i) {
                const uint4* E = reinterpret_cast<const uint4*>(ring + (size_t)s * 3 * NC + i * NC + 32 * t);
                uint32_t w[8];
#pragma unroll
                for (int q = 0; q < 2; ++q) {
                    const uint4 a = E[q];
                    w[4 * q] = a.x; w[4 * q + 1] = a.y; w[4 * q + 2] = a.z; w[4 * q + 3] = a.w;
                }
#pragma unroll
                for (int j = 0; j < 32; ++j) {
                    const uint32_t v = byte_at(w, j);
                    cS[j] += v;
                    cQ[j] += v * v;
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive_cnt(&empty[s], warp == 0 ? 1 + now : 1);
        }

        // quarter sums of the column sums (columns 8h..8h+7), then kept incrementally with dp4a
        uint32_t qS[4], qQ[4];
#pragma unroll
        for (int h = 0; h < 4; ++h) {
            const int c = 8 * h;
            qS[h] = ((cS[c] + cS[c + 1]) + (cS[c + 2] + cS[c + 3])) + ((cS[c + 4] + cS[c + 5]) + (cS[c + 6] + cS[c + 7]));
            qQ[h] = ((cQ[c] + cQ[c + 1]) + (cQ[c + 2] + cQ[c + 3])) + ((cQ[c + 4] + cQ[c + 5]) + (cQ[c + 6] + cQ[c + 7]));
        }
        for (int k = it.nwarm; k < it.n; ++k) {
            const int y = it.ya + (k - it.nwarm);
            const int s = k % NS;
            const int b = (k - it.nwarm) & 1;
            mbar_wait(&full[s], (k / NS) & 1);
            const uint8_t* stage = ring + (size_t)s * 3 * NC;
            const bool first = (k == it.nwarm);
            const bool ein = !first && y + p.r < p.H, oin = !first && y - p.r - 1 >= 0;
            // entering / leaving row bytes of this lane's 32 columns (zero when outside the image)
            uint32_t e[8], o[8];
            {
                const uint4* E = reinterpret_cast<const uint4*>(stage + 32 * t);
                const uint4* O = reinterpret_cast<const uint4*>(stage + NC + 32 * t);
                if (ein && oin) {
#pragma unroll
                    for (int q = 0; q < 2; ++q) {
                        const uint4 a = E[q], bb = O[q];
                        e[4 * q] = a.x; e[4 * q + 1] = a.y; e[4 * q + 2] = a.z; e[4 * q + 3] = a.w;
                        o[4 * q] = bb.x; o[4 * q + 1] = bb.y; o[4 * q + 2] = bb.z; o[4 * q + 3] = bb.w;
                    }
                } else {
#pragma unroll
                    for (int q = 0; q < 2; ++q) {
                        const uint4 a = ein ? E[q] : make_uint4(0, 0, 0, 0);
                        const uint4 bb = oin ? O[q] : make_uint4(0, 0, 0, 0);
                        e[4 * q] = a.x; e[4 * q + 1] = a.y; e[4 * q + 2] = a.z; e[4 * q + 3] = a.w;
                        o[4 * q] = bb.x; o[4 * q + 1] = bb.y; o[4 * q + 2] = bb.z; o[4 * q + 3] = bb.w;
                    }
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[s]);  // this warp is done with item k's rows
            // quarter totals (dp4a) -> lane total -> warp scan; the scan's shuffle latency and
            // the column-warp hand-off overlap the vertical update below
#pragma unroll
            for (int h = 0; h < 4; ++h) {
                qS[h] = dp4a_sub(o[2 * h + 1], dp4a_sub(o[2 * h], __dp4a(e[2 * h + 1], 0x01010101u,
                                                      __dp4a(e[2 * h], 0x01010101u, qS[h]))));
                qQ[h] += __dp4a(e[2 * h + 1], e[2 * h + 1], __dp4a(e[2 * h], e[2 * h], 0u)) -
                         __dp4a(o[2 * h + 1], o[2 * h + 1], __dp4a(o[2 * h], o[2 * h], 0u));
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
            // column warp 0 hands its total to warp 1 (ncw = 2): arrive now, warp 1 syncs later;
            // with more column warps every warp publishes and all sync after the update
            if (GB_NCW == 2 && warp == 0) {
                if (lane == 31) { sWS[8 * b] = iS; sWQ[8 * b] = iQ; }
                nbar_arrive(BAR_COLS, 32 * ncw);
            }
            if (GB_NCW > 2 && lane == 31) { sWS[8 * b + warp] = iS; sWQ[8 * b + warp] = iQ; }
#pragma unroll
            for (int j = 0; j < 32; ++j) {
                const uint32_t ev = byte_at(e, j), ov = byte_at(o, j);
                cS[j] = cS[j] + ev - ov;
                cQ[j] = cQ[j] + ev * ev - ov * ov;
            }
            uint32_t bS = iS - TS, bQ = iQ - TQ;
            if (GB_NCW > 2) {
                nbar_sync(BAR_COLS, 32 * ncw);
#pragma unroll
                for (int w = 0; w < GB_NCW - 1; ++w)
                    if (w < warp) { bS += sWS[8 * b + w]; bQ += sWQ[8 * b + w]; }
            } else if (warp == 1) {
                nbar_sync(BAR_COLS, 32 * ncw);
                bS += sWS[8 * b]; bQ += sWQ[8 * b];
            }
            // wait until the output warps have consumed row k-2 from this prefix buffer
            nbar_sync(BAR_FREE0 + b, nthr);
            uint32_t* sPS = sm + (2 * b) * 4 * PW + 4 * t;
            uint32_t* sPQ = sPS + 4 * PW;
            // exclusive running prefix, stored residue-decimated: half hh of the lane's columns
            // (two quarter chains) -> plane rho chunk (hh, t) = {pre[16hh+rho+4i], i = 0..3}
            {
                uint32_t cb0S = bS, cb0Q = bQ;
#pragma unroll
                for (int hh = 0; hh < 2; ++hh) {
                    uint32_t c1S = cb0S + qS[2 * hh], c1Q = cb0Q + qQ[2 * hh];
                    uint32_t vS[4][4], vQ[4][4];  // [rho][i]
                    uint32_t r0S = cb0S, r0Q = cb0Q, r1S = c1S, r1Q = c1Q;
#pragma unroll
                    for (int i = 0; i < 8; ++i) {
                        const int j0 = 16 * hh + i, j1 = j0 + 8;
                        vS[i & 3][i >> 2] = r0S; vQ[i & 3][i >> 2] = r0Q;
                        vS[i & 3][2 + (i >> 2)] = r1S; vQ[i & 3][2 + (i >> 2)] = r1Q;
                        r0S += cS[j0]; r0Q += cQ[j0];
                        r1S += cS[j1]; r1Q += cQ[j1];
                    }
#pragma unroll
                    for (int rho = 0; rho < 4; ++rho) {
                        const int pos = rho * PW + 4 * hh * T1;
                        *reinterpret_cast<uint4*>(&sPS[pos]) = make_uint4(vS[rho][0], vS[rho][1], vS[rho][2], vS[rho][3]);
                        *reinterpret_cast<uint4*>(&sPQ[pos]) = make_uint4(vQ[rho][0], vQ[rho][1], vQ[rho][2], vQ[rho][3]);
                    }
                    cb0S = c1S + qS[2 * hh + 1]; cb0Q = c1Q + qQ[2 * hh + 1];
                }
                if (t == 32 * ncw - 1) {  // word NC: plane 0, dec index 8T -> chunk (0, T)
                    sPS[4] = cb0S;
                    sPQ[4] = cb0Q;
                }
            }
            nbar_arrive(BAR_READY0 + b, nthr);
        }
        const int rows = it.n - it.nwarm;
        if (rows >= 1) nbar_sync(BAR_FREE0 + (rows & 1), nthr);
        if (rows >= 2) nbar_sync(BAR_FREE0 + ((rows + 1) & 1), nthr);
    } else {
        // ===================== output warps =====================
        const int to = t - 32 * ncw;
        const int xo = X0 + 32 * to;
        const bool has_out = (32 * to + 32 + 2 * p.r + ALPHA <= NC) && (32 * to < p.TW) && (xo < p.cols);
        const bool out_full = has_out && (xo + 32 <= p.cols) &&
                              ((reinterpret_cast<uintptr_t>(p.bin) | (uintptr_t)p.bin_pitch |
                                (uintptr_t)p.out_stride) & 15) == 0;
        const bool x_interior = (xo - p.r >= 0) && (xo + 31 + p.r <= p.cols - 1);
        const bool border_warp = __any_sync(0xffffffffu, has_out && !x_interior);
        const int qB = (ALPHA + 2 * p.r + 1) >> 5;  // lane offset of the B streams
        const int qB3 = (ALPHA + 2 * p.r + 4) >> 5;
        const float W = (float)(2 * p.r + 1);
        const float a1 = p.a, cK = p.c;  // 1-k, k/R
        const float kUp = 1.0f + 7.62939453125e-6f, kDn = 1.0f - 7.62939453125e-6f;  // 1 +- 2^-17
        const float dAbs = p.tol;  // >= the reference's own fp64 error on t (slide_constants)
        uint8_t* obase = p.bin + (int64_t)blockIdx.z * p.out_stride - (int64_t)p.out_begin * p.bin_pitch;
        nbar_arrive(BAR_FREE0, nthr);  // both prefix buffers start free
        nbar_arrive(BAR_FREE0 + 1, nthr);
        int issued = 0;
        if (producer) {  // the ring's first NS items, then every warm-up slot as it frees up
            while (issued < min(NS, it.n)) issue(issued++);
            while (issued < min(it.nwarm + NS - 1, it.n)) issue(issued++);
        }
        for (int k = it.nwarm; k < it.n; ++k) {
            const int y = it.ya + (k - it.nwarm);
            const int s = k % NS;
            const int b = (k - it.nwarm) & 1;
            nbar_sync(BAR_READY0 + b, nthr);
            // every warp released item k-1 by now (output warps: program order before READY(k);
            // column warps: before READY(k-1)), so refilling its slot never blocks
            if (producer)
                while (issued < min(k + NS, it.n)) issue(issued++);
            mbar_wait(&full[s], (k / NS) & 1);  // (complete; makes the staged rows visible)
            const uint8_t* stage = ring + (size_t)s * 3 * NC;
            const uint32_t* sPS = sm + (2 * b) * 4 * PW;
            const uint32_t* sPQ = sPS + 4 * PW;
            if (has_out) {
                uint8_t* orow = obase + (int64_t)y * p.bin_pitch;
                const int ny = min(y + p.r, p.H - 1) - max(y - p.r, 0) + 1;
                const uint8_t* fsm = stage + 2 * NC + 32 * to;
                uint32_t fw[8];
#pragma unroll
                for (int q = 0; q < 2; ++q) {
                    const uint4 v = *reinterpret_cast<const uint4*>(fsm + 16 * q);
                    fw[4 * q] = v.x; fw[4 * q + 1] = v.y; fw[4 * q + 2] = v.z; fw[4 * q + 3] = v.w;
                }
                uint32_t SA0[8], SA3[8], SB0[8], SB3[8], QA0[8], QB3[8];
                gb_stream<D_A0>(sPS + R_A0 * PW, to, T1, SA0);
                gb_stream<D_A3>(sPS + R_A3 * PW, to, T1, SA3);
                gb_stream<D_B0>(sPS + R_B0 * PW, to + qB, T1, SB0);
                gb_stream<D_B3>(sPS + R_B3 * PW, to + qB3, T1, SB3);
                gb_stream<D_A0>(sPQ + R_A0 * PW, to, T1, QA0);
                gb_stream<D_B3>(sPQ + R_B3 * PW, to + qB3, T1, QB3);
                // 1/n for the row (interior lanes: n = ny * W for every pixel), with the slack;
                // the intersection window I has n_I = ny (2r-2) pixels
                const float rnr = rcp_ftz((float)ny * W);  // rel. error << the 2^-17 slack
                const float rloR = rnr * kUp, rhiR = rnr * kDn;
                uint32_t ow[8];
                uint32_t um = 0;  // groups with an uncertain pixel
                // rlo / rhi: 1/n_lo, 1/n_hi with the slack
                auto group = [&](int g, float rlo, float rhi) {
                    const uint32_t SU = SB3[g] - SA0[g];
                    const uint32_t SI = SB0[g] - SA3[g];
                    const uint32_t QU = QB3[g] - QA0[g];
                    const float fSI = (float)SI;
                    const float mhi = (float)SU * rlo;
                    const float mlo = fSI * rhi;
                    // upper: var <= Q_U/n_lo - m_lo^2 (raised)
                    const float v = __fmaf_rn((float)QU, rlo, -(mlo * mlo));
                    const float sd = sqrt_ftz(fmaxf(v, 0.f));
                    const float thi = fminf(__fmaf_rn(mhi, __fmaf_rn(sd, cK, a1), dAbs), 4096.f);
                    const float tlo = __fmaf_rn(mlo, a1, -dAbs);
                    const uint32_t H2 = gb_ceil2(thi), L2 = gb_ceil2(tlo);
                    // SWAR: 16-bit lanes (f | 0x8000) - T: bit 15 set iff f >= T
                    const uint32_t f4 = fw[g];
                    const uint32_t fA = prmt(f4, 0x80808080u, 0x4240);  // pixels 0, 2
                    const uint32_t fB = prmt(f4, 0x80808080u, 0x4341);  // pixels 1, 3
                    const uint32_t wA = fA - H2, wB = fB - H2;
                    ow[g] = prmt(wA, wB, 0xFBD9);  // bytes 0xFF where f >= ceil(t_hi)
                    const uint32_t u = ((fA - L2) & ~wA) | ((fB - L2) & ~wB);
                    if (u & 0x80008000u) um |= 1u << g;
                };
                if (!border_warp) {
#pragma unroll
                    for (int g = 0; g < 8; ++g) group(g, rloR, rhiR);
                } else {
                    // a warp with image-edge lanes: every lane takes per-group counts (warp-uniform)
#pragma unroll
                    for (int g = 0; g < 8; ++g) {
                        int nmin = 1 << 30, nmax = 0;
#pragma unroll
                        for (int i = 0; i < 4; ++i) {
                            const int x = xo + 4 * g + i;
                            const int nx = min(x + p.r, p.cols - 1) - max(x - p.r, 0) + 1;
                            nmin = min(nmin, nx); nmax = max(nmax, nx);
                        }
                        nmin = max(nmin, 1);
                        group(g, rcp_ftz((float)(ny * nmin)) * kUp, rcp_ftz((float)(ny * nmax)) * kDn);
                    }
                }
                if (out_full) {
#pragma unroll
                    for (int q = 0; q < 2; ++q)
                        __stcs(reinterpret_cast<uint4*>(orow + xo + 16 * q),
                               make_uint4(ow[4 * q], ow[4 * q + 1], ow[4 * q + 2], ow[4 * q + 3]));
                } else {
#pragma unroll
                    for (int j = 0; j < 32; ++j) {
                        const int x = xo + j;
                        if (x < p.cols) orow[x] = (uint8_t)(ow[j >> 2] >> (8 * (j & 3)));
                    }
                }
                // Uncertain groups, out of line and after the vector stores (program order): each
                // round, every lane with a flagged group re-decides one of them per pixel.
                const unsigned am = __activemask();  // the lanes with outputs
                while (__builtin_expect(__any_sync(am, um != 0u), 0)) {
                    if (um) {
                        const int g = __ffs(um) - 1;
                        um &= um - 1;
                        gb_fix_group(sPS, sPQ, PW, T1, ALPHA + 32 * to + 4 * g,
                                     ALPHA + 2 * p.r + 1 + 32 * to + 4 * g, fsm + 4 * g, orow,
                                     xo + 4 * g, p.cols, ny, p.r, p.cA, p.cC, p.a, p.c, p.tol, p.k, p.rr);
                    }
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[s]);
            nbar_arrive(BAR_FREE0 + b, nthr);
        }
    }
    if (g_gb_times_on && bid < 8192) {
        __syncthreads();
        if (t == 0) g_gb_times[2 * bid + 1] = gtimer();
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
    const char* env = getenv("DTB_L2HINT");
    p.l2hint = env ? atoi(env) : 1;
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
template <int V, int RXM4, int METHOD>
static cudaError_t ensure_smem(size_t smem) {
    static size_t granted = 48 * 1024;
    if (smem <= granted) return cudaSuccess;
    const cudaError_t e = cudaFuncSetAttribute(slide_kernel<V, RXM4, METHOD>,
                                               cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e == cudaSuccess) granted = smem;
    return e;
}

template <int V, int RXM4, int METHOD>
static cudaError_t run_slide(dim3 grid, int nt, size_t smem, const SlideParams& p,
                             cudaStream_t st) {
    cudaError_t e = ensure_smem<V, RXM4, METHOD>(smem);
    if (e != cudaSuccess) return e;
    slide_kernel<V, RXM4, METHOD><<<grid, nt, smem, st>>>(p);
    return cudaGetLastError();
}

template <int V, int RXM4, int METHOD>
static int occupancy(int nt, size_t smem) {
    static int cache_nt[16], cache_occ[16];
    static size_t cache_smem[16];
    static int n_cached = 0;
    for (int i = 0; i < n_cached; ++i)
        if (cache_nt[i] == nt && cache_smem[i] == smem) return cache_occ[i];
    int blocks = 0;
    ensure_smem<V, RXM4, METHOD>(smem);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, slide_kernel<V, RXM4, METHOD>, nt,
                                                      smem) != cudaSuccess)
        blocks = 1;
    blocks = std::max(blocks, 1);
    if (n_cached < 16) {
        cache_nt[n_cached] = nt; cache_smem[n_cached] = smem; cache_occ[n_cached] = blocks;
        ++n_cached;
    }
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

// DTB_PLAN_TIE=1: on equal staged work prefer more column warps per strip (fewer strips);
// measured neutral (C3 -1%, C5 W163/W179 +4%), so the default keeps the narrowest plan
static bool plan_tie_wide() {
    static int v = -1;
    if (v < 0) { const char* e = getenv("DTB_PLAN_TIE"); v = e ? atoi(e) : 0; }
    return v == 1;
}

// DTB_SLIDE_V=16 / 32 forces the columns per thread of the sliding kernels; unset = auto
static int slide_v() {
    static int v = -1;
    if (v < 0) {
        const char* env = getenv("DTB_SLIDE_V");
        v = env ? (atoi(env) == 16 ? 16 : 32) : 0;
    }
    return v;
}


// ---- warp-specialized launcher
template <int V, int VO, int RXM4, int MX>
static cudaError_t ws_run(dim3 grid, int nt, size_t smem, const SlideParams& p, cudaStream_t st,
                          int* occ) {
    static size_t granted = 48 * 1024;
    auto kern = ws_kernel<V, VO, RXM4, MX>;
    if (smem > granted) {
        const cudaError_t e =
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        granted = smem;
    }
    if (occ) {
        static int c_nt[16], c_occ[16];
        static size_t c_smem[16];
        static int nc = 0;
        for (int i = 0; i < nc; ++i)
            if (c_nt[i] == nt && c_smem[i] == smem) { *occ = c_occ[i]; return cudaSuccess; }
        int blocks = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, kern, nt, smem) != cudaSuccess)
            blocks = 1;
        *occ = std::max(blocks, 1);
        if (nc < 16) { c_nt[nc] = nt; c_smem[nc] = smem; c_occ[nc] = *occ; ++nc; }
        return cudaSuccess;
    }
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

// V = VO = 16 variant (DTB_WS_V16=1): half the per-thread state, twice the warps
static int ws_v16() {
    static int v = -1;
    if (v < 0) { const char* e = getenv("DTB_WS_V16"); v = e ? atoi(e) : DTB_WS_V16_DEFAULT; }
    return v;
}

static cudaError_t ws_dispatch(int m, bool sv, dim3 grid, int nt, size_t smem, const SlideParams& p,
                               cudaStream_t st, int* occ, bool v16) {
    if (v16) return ws_dispatch_vo<16, 16>(m, sv, grid, nt, smem, p, st, occ);
    return ws_dispatch_vo<32, 32>(m, sv, grid, nt, smem, p, st, occ);
}

static int use_ws() {
    static int v = -1;
    if (v < 0) {
        const char* env = getenv("DTB_WS");
        v = env ? atoi(env) : DTB_WS_DEFAULT;
    }
    return v;
}

// Debug / tuning knobs read once: DTB_PRINT_PLAN=1 prints each launch's strip/band plan;
// DTB_BAND_SCALE scales the band count (1 = one full wave of resident CTAs).
static bool print_plan() {
    static int v = -1;
    if (v < 0) { const char* e = getenv("DTB_PRINT_PLAN"); v = (e && e[0] == '1') ? 1 : 0; }
    return v == 1;
}
static double band_scale() {
    static double v = -1.0;
    if (v < 0) { const char* e = getenv("DTB_BAND_SCALE"); v = e ? atof(e) : 1.0; if (!(v > 0)) v = 1.0; }
    return v;
}

// ---- group-bound launcher (gb_kernel)
template <int R16, bool SEG>
static cudaError_t gb_run(dim3 grid, int nt, size_t smem, const SlideParams& p, cudaStream_t st,
                          int* occ) {
    static size_t granted = 48 * 1024;
    auto kern = gb_kernel<R16, SEG>;
    if (smem > granted) {
        const cudaError_t e =
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        granted = smem;
    }
    if (occ) {
        static int c_nt[16], c_occ[16];
        static size_t c_smem[16];
        static int nc = 0;
        for (int i = 0; i < nc; ++i)
            if (c_nt[i] == nt && c_smem[i] == smem) { *occ = c_occ[i]; return cudaSuccess; }
        int blocks = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, kern, nt, smem) != cudaSuccess)
            blocks = 1;
        *occ = std::max(blocks, 1);
        if (nc < 16) { c_nt[nc] = nt; c_smem[nc] = smem; c_occ[nc] = *occ; ++nc; }
        return cudaSuccess;
    }
    kern<<<grid, nt, smem, st>>>(p);
    return cudaGetLastError();
}

static cudaError_t gb_dispatch(int r16, dim3 grid, int nt, size_t smem, const SlideParams& p,
                               cudaStream_t st, int* occ) {
    switch (r16) {
#define DTB_GB_CASE(R) case R: return p.nseg ? gb_run<R, true>(grid, nt, smem, p, st, occ) \
                                              : gb_run<R, false>(grid, nt, smem, p, st, occ);
        DTB_GB_CASE(0) DTB_GB_CASE(1) DTB_GB_CASE(2) DTB_GB_CASE(3)
        DTB_GB_CASE(4) DTB_GB_CASE(5) DTB_GB_CASE(6) DTB_GB_CASE(7)
        DTB_GB_CASE(8) DTB_GB_CASE(9) DTB_GB_CASE(10) DTB_GB_CASE(11)
        DTB_GB_CASE(12) DTB_GB_CASE(13) DTB_GB_CASE(14) DTB_GB_CASE(15)
#undef DTB_GB_CASE
    }
    return cudaErrorInvalidValue;
}

// DTB_GB: 0 never, 1 whenever eligible, 2 (default) eligible and r >= DTB_GB_MIN_R.
#ifndef DTB_GB_MIN_R
#define DTB_GB_MIN_R 31
#endif
#ifndef DTB_GB_MIN_COLS
#define DTB_GB_MIN_COLS 1536
#endif
// Auto mode also wants a large page: on 4096^2 pages with sigma-12 noise (C5) many groups need
// the out-of-line re-decision and the one-wave plan has ~20-row bands under 2r+1 warm-up rows,
// which measured 1.1-1.3x slower than ws_kernel at W 67..179 (profiles/r01d_config_table.json).
#ifndef DTB_GB_MIN_PIXELS
#define DTB_GB_MIN_PIXELS (1ll << 26)
#endif
static int gb_mode() {  // read per launch (tests switch it)
    const char* e = getenv("DTB_GB");
    return e ? atoi(e) : 2;
}

static thread_local const char* g_last_kernel = "";
const char* last_kernel() { return g_last_kernel; }
void set_last_kernel(const char* name) { g_last_kernel = name; }

cudaError_t set_fp32_audit(unsigned long long* counters) {
    const cudaError_t e = cudaMemcpyToSymbol(g_fp32_audit, &counters, sizeof(counters));
    return e != cudaSuccess ? e : set_fp32_audit_block(counters);
}

// DTB_BB: 0 never, 1 whenever eligible, 2 (default): eligible and either r >= DTB_BB_MIN_R, or
// r >= DTB_BB_MIN_R_LARGE on pages of >= 2^26 output pixels.  Measured (profiles/r02_config_table
// files): C4 (16384^2, r=63) 0.40 vs 0.50 ms; 4096^2 pages at r=9..49 are 1.2-6x slower on
// bb_kernel than on the per-pixel kernels (each pipeline's 2r-row warm-up dominates a short
// band), break even near r=50 and win from r~57 (W115: 0.113 vs 0.117 ms, W243: 0.140 vs 0.154).
#ifndef DTB_BB_MIN_R
#define DTB_BB_MIN_R 56
#endif
#ifndef DTB_BB_MIN_R_LARGE
#define DTB_BB_MIN_R_LARGE 24
#endif
static int bb_mode() {  // read per launch (tests switch it)
    const char* e = getenv("DTB_BB");
    return e ? atoi(e) : 2;
}

// Band count minimising waves * (TH + wf (2r+1)) + tf * TH in main-row units per CTA slot
// (see the gb_kernel launcher); DTB_BAND_SCALE overrides with scale x one wave.
static int plan_bands(int rows_out, int units, int slots, int r, double wf, double tf) {
    int nbands = 1;
    if (getenv("DTB_BAND_SCALE")) {
        nbands = std::max(1, (int)(band_scale() * slots / std::max(1, units)));
    } else {
        double best_cost = 1e300;
        const int nb_max = std::max(1, std::min((rows_out + 7) / 8, 4 * slots / std::max(1, units) + 1));
        for (int nb = 1; nb <= nb_max; ++nb) {
            const int th = (rows_out + nb - 1) / nb;
            const int waves = (units * nb + slots - 1) / slots;
            const double cost = waves * (th + wf * (2 * r + 1)) + tf * th;
            if (cost < best_cost) { best_cost = cost; nbands = nb; }
        }
    }
    return std::max(1, std::min(nbands, (rows_out + 7) / 8));
}

static int slide_band_model() {  // DTB_BAND_MODEL=0: one full wave (the previous rule)
    static int v = -1;
    if (v < 0) { const char* e = getenv("DTB_BAND_MODEL"); v = e ? atoi(e) : 1; }
    return v;
}

cudaError_t launch_slide(SlideParams p, int n_images, int num_sms, cudaStream_t st) {
    slide_constants(p);
    const int vset = slide_v();
    // segmented variants: V = 32 only; the tmap variant runs V = 16 (half the registers per
    // thread: twice the resident warps for its fp64 epilogue)
    int V = p.tmap ? 16 : (p.nseg ? 32 : (vset ? vset : 32));
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
            if (b.w == 0 || work < b.work || (plan_tie_wide() && work == b.work)) b = Plan{w, ns, tw, work};
        }
        return b;
    };
    {
        const int bbm = bb_mode();
        const long long px = (long long)p.cols * (p.out_end - p.out_begin) * n_images;
        if (bbm && !p.tmap && bb_eligible(p) &&
            (bbm == 1 || p.r >= DTB_BB_MIN_R || (p.r >= DTB_BB_MIN_R_LARGE && px >= (1ll << 26))))
            return launch_block(p, n_images, num_sms, st, print_plan());
    }
    Plan pl = plan_for(V);
    int best_w = pl.w, best_strips = pl.strips, best_tw = pl.tw;
    if (best_w == 0) return cudaErrorInvalidValue;  // window too wide for 8 warps (caller checks)
    // group-bound kernel: Sauvola with 0 < k <= 1, strips of 2 column warps (see gb_kernel)
    const int gbm = gb_mode();
    const int gb_tw = 32 * ((GB_NC - 2 * p.rx - alpha) / 32);
    // r <= 127: the union window's Q_U (2r+4 columns) stays below 2^32 (65025 * 258 * 255);
    // slide_ok alone admits W = 257, whose union sums could wrap
    if (V == 32 && p.method == DTB_METHOD_SAUVOLA && p.k > 0.0 && p.k <= 1.0 &&
        p.rx == p.r && p.r <= 127 && gb_tw >= 32 &&
        (gbm == 1 || (gbm == 2 && p.r >= DTB_GB_MIN_R && p.cols >= DTB_GB_MIN_COLS &&
                      (long long)p.cols * (p.out_end - p.out_begin) * n_images >= DTB_GB_MIN_PIXELS))) {
        const int ns = (p.cols + gb_tw - 1) / gb_tw;
        best_strips = ns;
        best_tw = 32 * ((p.cols + 32 * ns - 1) / (32 * ns));
        best_w = GB_NCW;
        p.ncw = best_w;
        p.now = GB_NCW;  // (the role swap below pairs the two equal halves of the CTA)
        {
            const char* se = getenv("DTB_GB_SWAP");
            p.role_div = (se && atoi(se) > 0) ? atoi(se) : 0;
        }
        p.NC = GB_NC;
        p.TW = best_tw;
        const int nt = 32 * (p.ncw + p.now);
        const size_t smem = gb_smem_bytes(p.NC);
        int occ = 1;
        const cudaError_t qe = gb_dispatch(p.r & 15, dim3(), nt, smem, p, st, &occ);
        if (qe != cudaSuccess) return qe;
        const int slots = num_sms * occ;
        // Band count from a cost model, in main-row units per CTA slot:
        //   waves * (TH + 0.25 (2r+1))  +  0.3 TH
        // (a warm-up row -- column sums only -- costs ~1/4 of a main row; the last term stands
        // for the content-dependent spread of band cost: uncertain groups cluster in dark page
        // regions, and a one-wave launch waits on its slowest bands).  C4: 2 waves of 125-row
        // bands (0.498 ms vs 0.518 at one wave); 4096^2 pages: one wave (bands of 2r+1 rows of
        // warm-up over ~20 output rows otherwise dominate).
        int nbands = 1;
        {
            const char* bse = getenv("DTB_BAND_SCALE");
            const int units = std::max(1, best_strips * n_images);
            if (bse) {
                nbands = std::max(1, (int)(band_scale() * slots / units));
            } else {
                double best_cost = 1e300;
                const int nb_max = std::max(1, std::min((rows_out + 7) / 8, 4 * slots / units + 1));
                for (int nb = 1; nb <= nb_max; ++nb) {
                    const int th = (rows_out + nb - 1) / nb;
                    const int waves = (units * nb + slots - 1) / slots;
                    const double cost = waves * (th + 0.25 * (2 * p.r + 1)) + 0.3 * th;
                    if (cost < best_cost) { best_cost = cost; nbands = nb; }
                }
            }
            nbands = std::max(1, std::min(nbands, (rows_out + 7) / 8));
        }
        p.TH = (rows_out + nbands - 1) / nbands;
        dim3 grid(best_strips, (rows_out + p.TH - 1) / p.TH, n_images);
        if (print_plan())
            fprintf(stderr, "[dtb plan] gb_kernel cols=%d rows=%d r=%d w=%d strips=%d TW=%d occ=%d bands=%d TH=%d smem=%zu\n",
                    p.cols, rows_out, p.r, best_w, best_strips, best_tw, occ, (int)grid.y, p.TH, smem);
        g_last_kernel = "gb_kernel";
        const char* tenv = getenv("DTB_GB_TIMES");
        if (tenv && tenv[0] == '1') {
            const int on = 1;
            cudaMemcpyToSymbol(g_gb_times_on, &on, sizeof(on));
            const cudaError_t e = gb_dispatch(p.r & 15, grid, nt, smem, p, st, nullptr);
            cudaDeviceSynchronize();
            static unsigned long long h[2 * 8192];
            cudaMemcpyFromSymbol(h, g_gb_times, sizeof(h));
            const int nb = std::min(8192, (int)(grid.x * grid.y * grid.z));
            unsigned long long t0 = ~0ull, t1 = 0;
            for (int i = 0; i < nb; ++i) { t0 = std::min(t0, h[2 * i]); t1 = std::max(t1, h[2 * i + 1]); }
            fprintf(stderr, "[gb times] ctas=%d span=%.1f us\n", nb, (t1 - t0) * 1e-3);
            for (int i = 0; i < nb; ++i)
                fprintf(stderr, "[gb cta] %d strip=%d band=%d start=%.1f end=%.1f\n", i, i % (int)grid.x,
                        (i / (int)grid.x) % (int)grid.y, (h[2 * i] - t0) * 1e-3, (h[2 * i + 1] - t0) * 1e-3);
            return e;
        }
        return gb_dispatch(p.r & 15, grid, nt, smem, p, st, nullptr);
    }
    // Auto V: 16 columns per thread give strips in 512-column steps (and 128-register warps);
    // take them when that cuts the staged column work by >= 10% (C2 pages 2480 wide: one strip
    // of 2560 instead of three of 1024 -- W15 0.119 -> 0.058 ms; C5 W3: 0.093 -> 0.078 ms;
    // C5 W67 / W131 within 2%).
    if (!vset && !p.nseg && !p.tmap && V == 32) {
        const Plan p16 = plan_for(16);
        if (p16.w > 0 && p16.work * 10 <= pl.work * 9) {
            V = 16;
            best_w = p16.w; best_strips = p16.strips; best_tw = p16.tw;
        }
    }
    // warp-specialized kernel when the strip has >= 2 column warps (measured: C4 0.624 vs 0.656
    // ms; single-column-warp strips such as C3's are faster on the classic kernel)
    const int ws_mode = use_ws();
    if (V == 32 && (ws_mode == 1 || (ws_mode == 2 && best_w >= 2))) {
        const bool v16 = ws_v16() && best_w <= 4;  // column-warp totals table holds 8 warps
        const int vo = v16 ? 16 : 32;
        p.ncw = v16 ? 2 * best_w : best_w;
        p.now = (best_tw + 32 * vo - 1) / (32 * vo);
        {
            static int swap_mode = -1;
            if (swap_mode < 0) {
                const char* env = getenv("DTB_WS_SWAP");
                swap_mode = env ? atoi(env) : 0;  // measured: 0.656 vs 0.621 ms (C4) with it on
            }
            p.role_div = swap_mode ? num_sms : 0;
        }
        p.NC = 1024 * best_w;
        p.TW = best_tw;
        const int nt = 32 * (p.ncw + p.now);
        const size_t smem = ws_smem_bytes(p.NC);
        const int m = p.rx & 3;
        const bool sv = p.method == DTB_METHOD_SAUVOLA;
        int occ = 1;
        ws_dispatch(m, sv, dim3(), nt, smem, p, st, &occ, v16);
        const int slots = num_sms * occ;
        int nbands = std::max(1, (int)(band_scale() * slots / std::max(1, best_strips * n_images)));
        nbands = std::max(1, std::min(nbands, (rows_out + 7) / 8));  // one wave (the model measured
                                                                     // 1-4% slower here, C5 W195+)
        p.TH = (rows_out + nbands - 1) / nbands;
        dim3 grid(best_strips, (rows_out + p.TH - 1) / p.TH, n_images);
        if (print_plan())
            fprintf(stderr, "[dtb plan] ws_kernel cols=%d rows=%d r=%d w=%d strips=%d TW=%d occ=%d bands=%d TH=%d\n",
                    p.cols, rows_out, p.r, best_w, best_strips, best_tw, occ, (int)grid.y, p.TH);
        g_last_kernel = "ws_kernel";
        return ws_dispatch(m, sv, grid, nt, smem, p, st, nullptr, v16);
    }
    const int nt = 32 * best_w;
    p.NC = V * nt;
    p.TW = best_tw;
    const int nstrips = best_strips;
    const size_t smem = slide_smem_bytes(p.NC);
    const int m = p.rx & 3;
    const bool sv = p.method == DTB_METHOD_SAUVOLA;
    int occ = 1;
    if (V == 16) dispatch_rx<16>(m, sv, dim3(), nt, smem, p, st, &occ);
    else dispatch_rx<32>(m, sv, dim3(), nt, smem, p, st, &occ);
    // bands: one full wave of resident CTAs (bands as tall as possible: the warm-up of each
    // band costs 2r+1 rows of vertical work)
    const int slots = num_sms * occ;
    int nbands = std::max(1, (int)(band_scale() * slots / std::max(1, nstrips * n_images)));
    nbands = std::max(1, std::min(nbands, (rows_out + 7) / 8));
    // cost-model band count (C3 0.949 -> 0.885 ms, C5 W19..W179 2-4% faster than one wave)
    if (slide_band_model()) nbands = plan_bands(rows_out, nstrips * n_images, slots, p.r, 0.25, 0.1);
    p.TH = (rows_out + nbands - 1) / nbands;
    dim3 grid(nstrips, (rows_out + p.TH - 1) / p.TH, n_images);
    if (print_plan())
        fprintf(stderr, "[dtb plan] slide_kernel V=%d cols=%d rows=%d r=%d w=%d strips=%d TW=%d occ=%d bands=%d TH=%d\n",
                V, p.cols, rows_out, p.r, best_w, nstrips, best_tw, occ, (int)grid.y, p.TH);
    g_last_kernel = "slide_kernel";
    return V == 16 ? dispatch_rx<16>(m, sv, grid, nt, smem, p, st, nullptr)
                   : dispatch_rx<32>(m, sv, grid, nt, smem, p, st, nullptr);
}

}  // namespace dtb
