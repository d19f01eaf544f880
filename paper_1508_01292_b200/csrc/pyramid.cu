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
// Roofline: HBM/L2-bound.  Algorithmic bytes per level pixel: 1 B written + the
// frame read once per frame.  One CTA per (level row, frame);
// each thread produces 4 consecutive pixels and stores them as one 32-bit word.
#include "ccnn_internal.h"

namespace ccnn {
namespace {

__device__ __forceinline__ uint32_t blend(const uint8_t* r0, const uint8_t* r1, uint32_t xt,
                                          uint32_t ay, int W)
{
    uint32_t x0 = xt & 0xFFFFu;
    uint32_t ax = xt >> 16;
    uint32_t x1 = min(x0 + 1u, (uint32_t)(W - 1));
    uint32_t top = (uint32_t)__ldg(r0 + x0) * (2048u - ax) + (uint32_t)__ldg(r0 + x1) * ax;
    uint32_t bot = (uint32_t)__ldg(r1 + x0) * (2048u - ax) + (uint32_t)__ldg(r1 + x1) * ax;
    return (top * (2048u - ay) + bot * ay + (1u << 21)) >> 22;
}

__global__ void __launch_bounds__(128) pyramid_kernel(
    const uint8_t* __restrict__ frames, int64_t frame_stride, int64_t pitch, int W, int H,
    uint8_t* __restrict__ levels, int64_t level_frame_stride,
    const LevelInfo* __restrict__ lv, int n_levels, const uint32_t* __restrict__ tabs)
{
    const int row = blockIdx.x;              // row in the concatenation of all levels
    const int f = blockIdx.y;
    int l = 0;
    while (l + 1 < n_levels && lv[l + 1].row0 <= row) ++l;
    const LevelInfo L = lv[l];
    const int y = row - L.row0;
    const uint32_t yt = tabs[L.tab_off + L.lw + y];
    const uint32_t y0 = yt & 0xFFFFu, ay = yt >> 16;
    const uint32_t y1 = min(y0 + 1u, (uint32_t)(H - 1));
    const uint8_t* src = frames + (int64_t)f * frame_stride;
    const uint8_t* r0 = src + (int64_t)y0 * pitch;
    const uint8_t* r1 = src + (int64_t)y1 * pitch;
    uint32_t* dst = reinterpret_cast<uint32_t*>(levels + (int64_t)f * level_frame_stride +
                                                L.offset + (int64_t)y * L.pitch);
    const uint32_t* xt = tabs + L.tab_off;
    const int nwords = L.pitch >> 2;
    for (int k = threadIdx.x; k < nwords; k += blockDim.x) {
        uint32_t word = 0;
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            int x = min(4 * k + b, L.lw - 1);    // pitch padding replicates the last pixel
            word |= blend(r0, r1, __ldg(xt + x), ay, W) << (8 * b);
        }
        dst[k] = word;
    }
}

}  // namespace

void launch_pyramid(const uint8_t* frames, int64_t frame_stride, int64_t pitch, int W, int H,
                    uint8_t* levels, int64_t level_frame_stride, const LevelInfo* d_levels,
                    const LevelInfo* h_levels, int n_levels, const uint32_t* d_tabs, int n,
                    cudaStream_t s)
{
    if (n_levels <= 0) return;
    const int rows = h_levels[n_levels - 1].row0 + h_levels[n_levels - 1].lh;
    dim3 grid(rows, n);
    pyramid_kernel<<<grid, 128, 0, s>>>(frames, frame_stride, pitch, W, H, levels,
                                        level_frame_stride, d_levels, n_levels, d_tabs);
}

}  // namespace ccnn
