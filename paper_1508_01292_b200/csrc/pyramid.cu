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
// DESIGN.md "Roofline"), in practice issue/ALU-bound on the byte gathers.  One CTA per
// (level row, frame) does the row setup once; its lanes stride over CONSECUTIVE output
// pixels, so each warp's byte gathers from the frame stay within 32/sigma bytes and its
// byte stores form one 32-byte sector; 4 pixels per lane are in flight at once.
// Measured alternatives: 4 adjacent pixels per lane spread every
// load instruction 4x wider; staging whole source rows in shared memory moved 5x the
// frame through L2; one pixel per thread with a flat grid paid the row setup per pixel.
#include "ccnn_internal.h"

namespace ccnn {
namespace {

constexpr int kPyrThreads = 128;

template <bool SAFE>
__global__ void __launch_bounds__(kPyrThreads) pyramid_kernel(
    const uint8_t* __restrict__ frames, int64_t frame_stride, int64_t pitch, int W, int H,
    uint8_t* __restrict__ levels, int64_t level_frame_stride,
    const LevelInfo* __restrict__ lv, int n_levels, const uint32_t* __restrict__ tabs)
{
    const int row = blockIdx.x;                        // row of the concatenated levels
    const int f = blockIdx.y;
    int l = 0;
    while (l + 1 < n_levels && lv[l + 1].row0 <= row) ++l;
    const LevelInfo& L = lv[l];
    const int y = row - L.row0;
    const uint32_t yt = __ldg(tabs + L.tab_off + L.lw + y);
    // SAFE (W, H >= 2): the tables encode the edge so that i1 = i0 + 1 always (runtime.cu
    // sample_entry); otherwise the clamped form
    const uint32_t y0 = yt & 0xFFFFu, ay = yt >> 16;
    const uint32_t y1 = SAFE ? y0 + 1u : min(y0 + 1u, (uint32_t)(H - 1));
    const uint8_t* src = frames + (int64_t)f * frame_stride;
    const uint8_t* __restrict__ r0 = src + (int64_t)y0 * pitch;
    const uint8_t* __restrict__ r1 = src + (int64_t)y1 * pitch;
    const uint32_t* __restrict__ xt = tabs + L.tab_off;
    uint8_t* dst = levels + (int64_t)f * level_frame_stride + L.offset + (int64_t)y * L.pitch;
    const int lwm = L.lw - 1;
    for (int xb = threadIdx.x; xb < L.pitch; xb += 4 * kPyrThreads) {
        uint32_t e[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) e[u] = __ldg(xt + min(xb + u * kPyrThreads, lwm));
        int p[4][4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const uint32_t x0 = e[u] & 0xFFFFu;
            p[u][0] = __ldg(r0 + x0);
            p[u][1] = SAFE ? __ldg(r0 + x0 + 1) : __ldg(r0 + min(x0 + 1u, (uint32_t)(W - 1)));
            p[u][2] = __ldg(r1 + x0);
            p[u][3] = SAFE ? __ldg(r1 + x0 + 1) : __ldg(r1 + min(x0 + 1u, (uint32_t)(W - 1)));
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int xo = xb + u * kPyrThreads;
            const int ax = (int)(e[u] >> 16);
            // p0*(2048-a) + p1*a == (p0 << 11) + (p1 - p0)*a, exactly (O2)
            const int top = (p[u][0] << 11) + (p[u][1] - p[u][0]) * ax;
            const int bot = (p[u][2] << 11) + (p[u][3] - p[u][2]) * ax;
            const int v = ((top << 11) + (bot - top) * (int)ay + (1 << 21)) >> 22;
            if (xo < L.pitch) dst[xo] = (uint8_t)v;      // pitch padding replicates the edge
        }
    }
}

}  // namespace

void launch_pyramid(const uint8_t* frames, int64_t frame_stride, int64_t pitch, int W, int H,
                    uint8_t* levels, int64_t level_frame_stride, const LevelInfo* d_levels,
                    const LevelInfo* h_levels, int n_levels, const uint32_t* d_tabs, int n,
                    cudaStream_t s)
{
    if (n_levels <= 0) return;
    const LevelInfo& last = h_levels[n_levels - 1];
    dim3 grid(last.row0 + last.lh, n);
    if (W >= 2 && H >= 2)
        pyramid_kernel<true><<<grid, kPyrThreads, 0, s>>>(frames, frame_stride, pitch, W, H, levels,
                                                          level_frame_stride, d_levels, n_levels, d_tabs);
    else
        pyramid_kernel<false><<<grid, kPyrThreads, 0, s>>>(frames, frame_stride, pitch, W, H, levels,
                                                           level_frame_stride, d_levels, n_levels, d_tabs);
}

}  // namespace ccnn
