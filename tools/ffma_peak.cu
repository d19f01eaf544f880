// ffma_peak.cu -- FP32 FFMA throughput microbenchmark on the B200.
// Measures warp-FFMA issue for the operand forms the stage-1 kernel uses:
//   (a) FFMA R, R, UR, R   weights in uniform registers (kernel-parameter constants)
//   (b) FFMA R, R, R, R    weights in registers
// 16 independent accumulators per thread, 148 x k CTAs, CUDA-event timed.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ffma_peak tools/ffma_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

struct Wts { float w[64]; };

template <int MODE>
__global__ void __launch_bounds__(256) ffma_kernel(const __grid_constant__ Wts W, float* out, int iters)
{
    float acc[16];
    float x0 = threadIdx.x * 1e-7f, x1 = x0 + 1e-7f;
#pragma unroll
    for (int k = 0; k < 16; ++k) acc[k] = k * 1e-3f;
    float wr[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) wr[k] = out[k + 1024] + W.w[k];   // runtime registers
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int j = 0; j < 8; ++j)
#pragma unroll
            for (int k = 0; k < 16; ++k) {
                const float w = MODE == 0 ? W.w[(j * 16 + k) & 63] : wr[(j + k) & 7];
                acc[k] = fmaf((k & 1) ? x1 : x0, w, acc[k]);
            }
    }
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < 16; ++k) s += acc[k];
    if (s == 1234.5f) out[threadIdx.x] = s;
}

int main()
{
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    float* out;
    cudaMalloc(&out, 1 << 20);
    cudaMemset(out, 0, 1 << 20);
    Wts w;
    for (int k = 0; k < 64; ++k) w.w[k] = 1e-3f * k;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int iters = 20000;
    for (int mode = 0; mode < 2; ++mode)
        for (int bps = 1; bps <= 8; bps *= 2) {
            dim3 grid(sms * bps);
            for (int rep = 0; rep < 2; ++rep) {
                cudaEventRecord(a);
                if (mode == 0) ffma_kernel<0><<<grid, 256>>>(w, out, iters);
                else ffma_kernel<1><<<grid, 256>>>(w, out, iters);
                cudaEventRecord(b);
                cudaEventSynchronize(b);
            }
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            double flops = 2.0 * 128 * iters * (double)grid.x * 256;
            printf("{\"mode\": \"%s\", \"ctas_per_sm\": %d, \"warps_per_smsp\": %d, \"tflops\": %.2f}\n",
                   mode == 0 ? "FFMA R,R,UR,R" : "FFMA R,R,R,R", bps, bps * 2, flops / ms / 1e9);
        }
    return 0;
}
