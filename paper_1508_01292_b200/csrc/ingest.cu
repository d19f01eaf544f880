// ingest.cu -- frame ingest for interleaved R,G,B rasters (SURVEY §8(f) NEXT #2 optional
// RGB->gray; reading I1: the paper assumes grayscale input).
//
// Rec.601 luma in exact integers, (299 R + 587 G + 114 B + 500) / 1000, bit-identical to
// the oracle's or_to_gray.  HBM-bound: 3 B read + 1 B written per pixel.  grid.y = job
// (one RGB frame of the batch), grid.x strides over its rows; a thread converts 4 adjacent
// pixels (12 source bytes) and writes one 32-bit word when the destination row allows.
#include "ccnn_internal.h"

namespace ccnn {
namespace {

constexpr int kGrayThreads = 256;

__device__ __forceinline__ uint32_t luma(uint32_t r, uint32_t g, uint32_t b)
{
    return (299u * r + 587u * g + 114u * b + 500u) / 1000u;
}

__global__ void __launch_bounds__(kGrayThreads) to_gray_kernel(const GrayJob* __restrict__ jobs)
{
    const GrayJob J = jobs[blockIdx.y];
    const int quads = (J.w + 3) >> 2;
    const int64_t total = (int64_t)quads * J.h;
    for (int64_t q = (int64_t)blockIdx.x * kGrayThreads + threadIdx.x; q < total;
         q += (int64_t)gridDim.x * kGrayThreads) {
        const int y = (int)(q / quads);
        const int x = (int)(q - (int64_t)y * quads) * 4;
        const uint8_t* s = J.src + (int64_t)y * J.src_pitch + 3 * x;
        uint8_t* d = J.dst + (int64_t)y * J.dst_pitch + x;
        if (x + 4 <= J.w) {
            uint32_t v = 0;
#pragma unroll
            for (int k = 0; k < 4; ++k)
                v |= luma(__ldg(s + 3 * k), __ldg(s + 3 * k + 1), __ldg(s + 3 * k + 2)) << (8 * k);
            *reinterpret_cast<uint32_t*>(d) = v;      // dst rows are 16-B aligned, x % 4 == 0
        } else {
            for (int k = 0; x + k < J.w; ++k)
                d[k] = (uint8_t)luma(__ldg(s + 3 * k), __ldg(s + 3 * k + 1), __ldg(s + 3 * k + 2));
        }
    }
}

}  // namespace

void launch_to_gray(const GrayJob* d_jobs, int n_jobs, int sm_count, cudaStream_t s)
{
    if (n_jobs <= 0) return;
    // ~4 CTAs of 256 threads per SM in all, spread over the jobs
    const int gx = std::max(1, (4 * sm_count + n_jobs - 1) / n_jobs);
    to_gray_kernel<<<dim3(gx, n_jobs), kGrayThreads, 0, s>>>(d_jobs);
}

}  // namespace ccnn
