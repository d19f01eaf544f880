// selective_common.cuh -- device helpers shared by the two selective-unit kernels
// (selective_tc.cu: patch preparation + CNN2 on tcgen05; selective.cu: CNN3 + decision).
// Not ABI.
//
// Patch preparation, §3.3: "the analyzed region is read from the original
// grayscale image together with certain neighborhood and scaled to the size of 51x55 pixels.
// Then, the equalization of its histogram and mirror reflection ... are carried out"; readings
// O5 (window centre, 51/35 x 55/39 expansion), O2 (fixed-point bilinear sampling, clamp to
// edge) and O6 (round-half-up equalisation), DESIGN.md.  All geometry is IEEE double with
// explicit _rn intrinsics (never contracted), bit-identical to the oracle.
#pragma once
#include "ccnn_internal.h"

namespace ccnn {
namespace sel {

// O2 sample coordinate: clamp to [0, n-1], i0 = floor(s), a = floor((s - i0)*2048 + 0.5)
__device__ __forceinline__ uint32_t bilin_coord(double s, int n)
{
    if (s < 0.0) s = 0.0;
    const double hi = (double)(n - 1);
    if (s > hi) s = hi;
    const double f = floor(s);
    const int a = (int)floor(__dadd_rn(__dmul_rn(__dsub_rn(s, f), 2048.0), 0.5));
    return (uint32_t)(int)f | ((uint32_t)a << 16);
}

// O5: the patch region of the survivor (ix, iy) of a level with scale sigma: left edge rx and
// width rw (columns), top edge ry and height rh (rows), in original-image pixels
struct PatchRegion { double rx, rw, ry, rh; };
__device__ __forceinline__ PatchRegion patch_region(int ix, int iy, double sigma)
{
    PatchRegion g;
    const double cx = __ddiv_rn(__dadd_rn((double)(4 * ix), 13.5), sigma);
    const double cy = __ddiv_rn(__dadd_rn((double)(4 * iy), 15.5), sigma);
    g.rw = __ddiv_rn(__ddiv_rn(1377.0, 35.0), sigma);            // 27*51/35
    g.rh = __ddiv_rn(__ddiv_rn(1705.0, 39.0), sigma);            // 31*55/39
    g.rx = __dsub_rn(cx, __ddiv_rn(g.rw, 2.0));
    g.ry = __dsub_rn(cy, __ddiv_rn(g.rh, 2.0));
    return g;
}
// sampling coordinate of patch column u (0..50) / row v (0..54) as an O2 table entry
__device__ __forceinline__ uint32_t region_col(const PatchRegion& g, int u, int W)
{
    const double t = __ddiv_rn(__dmul_rn(__dadd_rn((double)u, 0.5), g.rw), 51.0);
    return bilin_coord(__dsub_rn(__dadd_rn(g.rx, t), 0.5), W);
}
__device__ __forceinline__ uint32_t region_row(const PatchRegion& g, int v, int H)
{
    const double t = __ddiv_rn(__dmul_rn(__dadd_rn((double)v, 0.5), g.rh), 55.0);
    return bilin_coord(__dsub_rn(__dadd_rn(g.ry, t), 0.5), H);
}
__device__ __forceinline__ uint32_t patch_col(int ix, double sigma, int u, int W)
{
    return region_col(patch_region(ix, 0, sigma), u, W);
}
__device__ __forceinline__ uint32_t patch_row(int iy, double sigma, int v, int H)
{
    return region_row(patch_region(0, iy, sigma), v, H);
}

// O2 blend of the 2x2 footprint at table entries xt (column) / yt (row) of a frame
__device__ __forceinline__ uint32_t sample(const uint8_t* __restrict__ frame, int64_t pitch, int W, int H,
                                           uint32_t xt, uint32_t yt)
{
    const uint32_t x0 = xt & 0xFFFFu, y0 = yt & 0xFFFFu;
    const uint32_t x1 = min(x0 + 1u, (uint32_t)(W - 1)), y1 = min(y0 + 1u, (uint32_t)(H - 1));
    const uint8_t* r0 = frame + (int64_t)y0 * pitch;
    const uint8_t* r1 = frame + (int64_t)y1 * pitch;
    const uint32_t ax = xt >> 16, ay = yt >> 16;
    const uint32_t top = __ldg(r0 + x0) * (2048u - ax) + __ldg(r0 + x1) * ax;
    const uint32_t bot = __ldg(r1 + x0) * (2048u - ax) + __ldg(r1 + x1) * ax;
    return (top * (2048u - ay) + bot * ay + (1u << 21)) >> 22;
}

// O6 equalisation LUT from a 256-bin histogram of the N = 2805 patch pixels, by one warp:
// out(v) = (2*255*(cdf(v) - c_min) + (N - c_min)) div (2 (N - c_min)), c_min = the count of the
// smallest occupied value; a single-valued patch is unchanged
__device__ __forceinline__ void warp_lut(const int* __restrict__ hist, uint8_t* __restrict__ lut)
{
    const int lane = (int)(threadIdx.x & 31);
    int h[8], run = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) { run += hist[lane * 8 + k]; h[k] = run; }
    int incl = run;                                   // inclusive scan of lane totals
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const int t = __shfl_up_sync(0xFFFFFFFFu, incl, d);
        if (lane >= d) incl += t;
    }
    const int excl = incl - run;
    int first = 256;
#pragma unroll
    for (int k = 7; k >= 0; --k) if (hist[lane * 8 + k] > 0) first = lane * 8 + k;
#pragma unroll
    for (int d = 16; d >= 1; d >>= 1) first = min(first, __shfl_xor_sync(0xFFFFFFFFu, first, d));
    const int cmin = hist[first];
    const int N = kPatchN;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        const int v = lane * 8 + k;
        const int cdf = excl + h[k];
        lut[v] = (N == cmin) ? (uint8_t)v
                             : (uint8_t)((2 * 255 * (cdf - cmin) + (N - cmin)) / (2 * (N - cmin)));
    }
}

// O8 raw box: the stage-1 window mapped back to original pixels, round half up
__device__ __forceinline__ void raw_box(const S1Cand& cd, double sigma, SelOut& so)
{
    so.bx = (int)floor(__dadd_rn(__ddiv_rn((double)(4 * cd.ix), sigma), 0.5));
    so.by = (int)floor(__dadd_rn(__ddiv_rn((double)(4 * cd.iy), sigma), 0.5));
    so.bw = (int)floor(__dadd_rn(__ddiv_rn(27.0, sigma), 0.5));
    so.bh = (int)floor(__dadd_rn(__ddiv_rn(31.0, sigma), 0.5));
}

}  // namespace sel
}  // namespace ccnn
