// pyramid.cu -- image pyramid construction on sm_100a (DESIGN.md kernel K1).
//
// PAPER.md P:87 ("The first CNN densely scans in series each image of the pyramid"),
// P:121 (GPU pyramid), P:156 (minSize / scaleFactor); reading O2: every level is a
// bilinear resample of the ORIGINAL frame with half-pixel centres, clamp-to-edge and
// 11-bit fixed-point weights, so CPU and GPU levels are bit-identical.  The sampling
// coordinates (x0, ax) / (y0, ay) are IEEE-double geometry evaluated on the host
// (runtime.cu, -ffp-contract=off) and uploaded as packed tables; this kernel is pure
// integer arithmetic.
//
// Roofline: HBM-bound in principle (the frame read once + 1 B written per level pixel;
// DESIGN.md "Roofline"), in practice issue-bound on the byte gathers.  grid.y = frame,
// grid.x = tiles of the frame with the most (surplus CTAs of smaller frames exit); a CTA
// owns a tile of 128 consecutive output columns x 8 rows of one level: each thread loads
// its column's x-table entry once and walks the rows; the row setup is CTA-uniform;
// adjacent lanes gather adjacent output pixels (their frame reads stay within 32/sigma
// bytes) and store one 128-byte line per warp-row; all 8 rows' gathers are issued before
// any blend.
// Measured alternatives: 4 adjacent pixels per lane, whole source
// rows staged in shared memory, one pixel per thread on a flat grid, CTA per output row.
#include "ccnn_internal.h"

namespace ccnn {
namespace {

template <bool SAFE>
__global__ void __launch_bounds__(kPyrCols) pyramid_kernel(
    const FrameInfo* __restrict__ frames, uint8_t* __restrict__ levels,
    const LevelInfo* __restrict__ lv, const uint32_t* __restrict__ tabs)
{
    const FrameInfo F = frames[blockIdx.y];
    if ((int)blockIdx.x >= F.tiles) return;
    // level of this tile: linear scan from the frame's largest level (most tiles lie in
    // the first levels; cta0 is relative to the frame's first level)
    int l = F.level0;
    const int l_end = F.level0 + F.nlevels;
    while (l + 1 < l_end && lv[l + 1].cta0 <= (int)blockIdx.x) ++l;
    const LevelInfo& L = lv[l];
    const int tiles_x = (L.pitch + kPyrCols - 1) / kPyrCols;
    const int t = blockIdx.x - L.cta0;
    const int ty = t / tiles_x, tx = t - ty * tiles_x;
    const int xo = tx * kPyrCols + threadIdx.x;                // output column (pitch-padded)
    if (xo >= L.pitch) return;
    // SAFE (every frame W, H >= 2): the tables encode the edge so that i1 = i0 + 1 always
    // (runtime.cu sample_entry); otherwise the clamped form
    const uint32_t e = __ldg(tabs + L.tab_off + min(xo, L.lw - 1));   // padding = edge pixel
    const uint32_t x0 = e & 0xFFFFu;
    const uint32_t x1 = SAFE ? x0 + 1u : min(x0 + 1u, (uint32_t)(F.w - 1));
    const int ax = (int)(e >> 16);
    uint8_t* dst = levels + L.offset + xo;
    const uint32_t* yt = tabs + L.tab_off + L.lw;
    const int y_beg = ty * kPyrRows;
    const int nr = min(kPyrRows, L.lh - y_beg);                 // CTA-uniform
    // all rows' table entries and frame bytes are loaded before any blend: 8 rows of
    // independent gathers in flight per thread
    int p[kPyrRows][4], ay[kPyrRows];
#pragma unroll
    for (int r = 0; r < kPyrRows; ++r) {
        const uint32_t ye = __ldg(yt + y_beg + min(r, nr - 1));
        const uint32_t y0 = ye & 0xFFFFu;
        const uint32_t y1 = SAFE ? y0 + 1u : min(y0 + 1u, (uint32_t)(F.h - 1));
        ay[r] = (int)(ye >> 16);
        const uint8_t* r0 = F.data + (int64_t)y0 * F.pitch;
        const uint8_t* r1 = F.data + (int64_t)y1 * F.pitch;
        p[r][0] = __ldg(r0 + x0);
        p[r][1] = __ldg(r0 + x1);
        p[r][2] = __ldg(r1 + x0);
        p[r][3] = __ldg(r1 + x1);
    }
#pragma unroll
    for (int r = 0; r < kPyrRows; ++r) {
        // p0*(2048-a) + p1*a == (p0 << 11) + (p1 - p0)*a, exactly (O2)
        const int top = (p[r][0] << 11) + (p[r][1] - p[r][0]) * ax;
        const int bot = (p[r][2] << 11) + (p[r][3] - p[r][2]) * ax;
        if (r < nr) dst[(int64_t)(y_beg + r) * L.pitch] = (uint8_t)(((top << 11) + (bot - top) * ay[r] + (1 << 21)) >> 22);
    }
}

}  // namespace

void launch_pyramid(const FrameInfo* d_frames, int n_frames, int max_tiles, bool safe,
                    uint8_t* levels, const LevelInfo* d_levels, const uint32_t* d_tabs,
                    cudaStream_t s)
{
    if (n_frames <= 0 || max_tiles <= 0) return;
    const dim3 grid(max_tiles, n_frames);      // frames of other sizes: surplus CTAs exit
    if (safe)
        pyramid_kernel<true><<<grid, kPyrCols, 0, s>>>(d_frames, levels, d_levels, d_tabs);
    else
        pyramid_kernel<false><<<grid, kPyrCols, 0, s>>>(d_frames, levels, d_levels, d_tabs);
}

}  // namespace ccnn
