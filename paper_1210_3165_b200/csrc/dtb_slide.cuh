// dtb_slide.cuh -- parameters and launcher of the fast sliding-sum binarization kernel.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace dtb {

struct SlideParams {
    const uint8_t* in;
    int64_t pitch;
    int64_t img_stride;
    int cols, row0, H, out_begin, out_end;
    int in_rows;       // rows the input buffer (or the segments together) holds from row0
    int r, rx;
    int NC;     // columns per strip (= 32 * blockDim.x), set by launch_slide
    int TW;     // outputs per strip (multiple of 32), set by launch_slide
    int TH;     // output rows per band, set by launch_slide
    uint8_t* bin;
    int64_t bin_pitch;
    int64_t out_stride;
    int method;
    double k, rr;
    uint32_t N;        // (2r+1)^2: count of an unclipped window
    float cA, cC, tol; // fp32 fast-path constants (for n = N) and certified tolerance
    float a, c;        // Sauvola: 1-k, k/R; Niblack: 1, k (border constants are rebuilt per n)
    int l2hint;        // 1: evict_last / evict_first L2 policies on the staged row copies
    int ncw, now;      // warp-specialized kernel: column warps, output warps
    // slide_kernel, edge-padded single strip (pad > 0): the strip's NC columns are the image
    // columns [0, NC) themselves -- no halo columns are staged or summed.  The prefix array is
    // shifted right by `pad` words (= rx + alpha, a multiple of 32); the pad on the left stays
    // zero (P of a negative column) and `padr` words on the right repeat the row total (P of a
    // column past the image), so the output side reads both runs exactly as in the halo layout.
    int pad, padr;
    int PL;            // logical words of one prefix array (NC, or NC + pad + padr), set by launch_slide
    // Optional segmented input (dtb_binarize_segments): global rows [seg_lo[i], seg_lo[i+1]) live
    // at seg_ptr[i] with pitch seg_pitch[i] -- e.g. a neighbour GPU's halo rows read in place
    // over NVLink (peer / IPC pointers).  nseg == 0: the single buffer in/pitch/row0.
    int nseg;
    const uint8_t* seg_ptr[3];
    int64_t seg_pitch[3];
    int seg_lo[3];

    // optional fp64 threshold map (slide_kernel TMAP variant): tmap + y * tmap_pitch (bytes)
    double* tmap;
    int64_t tmap_pitch;
};

#ifndef WS_STAGES
#define WS_STAGES 6  // ws_kernel ring depth (C4: 0.6094 ms at 6 vs 0.6122 at 4, issue after READY)
#endif
static_assert(WS_STAGES >= 3, "the ring protocol needs at least 3 stages");
#ifndef SLIDE_STAGES
#define SLIDE_STAGES 4
#endif
static_assert(SLIDE_STAGES >= 3, "the ring protocol needs at least 3 stages");

// Words of one padded prefix array (logical 16-byte chunk L stored at chunk L + L/8).
__host__ __device__ inline int slide_padded_words(int NC) {
    const int chunks = NC / 4 + 4;
    return 4 * (chunks + chunks / 8 + 1);
}

// Dynamic shared memory of the fast kernel: 2 padded prefix arrays, warp totals, 2*NS
// mbarriers, and NS ring stages of (entering, leaving, centre) row segments of NC bytes.
__host__ __device__ inline size_t slide_smem_bytes(int NC, int PL) {
    return sizeof(uint32_t) * (2 * (size_t)slide_padded_words(PL) + 16) +
           2 * SLIDE_STAGES * sizeof(uint64_t) + (size_t)SLIDE_STAGES * 3 * NC;
}

// Warp-specialized kernel: two prefix buffers instead of one.
__host__ __device__ inline size_t ws_smem_bytes(int NC) {  // uses WS_STAGES
    return sizeof(uint32_t) * (4 * (size_t)slide_padded_words(NC) + 32) +
           2 * WS_STAGES * sizeof(uint64_t) + (size_t)WS_STAGES * 3 * NC;
}

// Fills N / cA / cC / tol from (r, method, k, rr) -- see the error analysis in dtb_slide.cu.
void slide_constants(SlideParams& p);

cudaError_t launch_slide(SlideParams p, int n_images, int num_sms, cudaStream_t st);

// Block-sum group-bound Sauvola kernel (dtb_block.cu): eligibility and launcher.
bool bb_eligible(const SlideParams& p);
bool bb_tma_ok(const SlideParams& p, int n_images);  // tensor-map staging prerequisites
cudaError_t launch_block(SlideParams p, int n_images, int num_sms, cudaStream_t st, bool print);
cudaError_t set_fp32_audit_block(unsigned long long* counters);
cudaError_t bb_exact_count(unsigned long long* out, bool reset);
cudaError_t bb_set_times(unsigned long long* buf, int cap);


}  // namespace dtb
