// hmma_peak.cu -- legacy tensor-core (mma.sync m16n8k16, f16 x f16 -> f32) throughput on the
// B200, alone and interleaved with FFMA work, to size a stage-1 layer-1 HMMA design
// (DESIGN.md "Stage 1").  Each warp issues independent MMAs on 8 accumulator tiles.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o hmma_peak tools/hmma_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void mma16816(float (&d)[4], const unsigned (&a)[4], const unsigned (&b)[2])
{
    asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                 : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
                 : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}

// FF = FFMAs per thread interleaved per MMA
template <int FF>
__global__ void __launch_bounds__(128) hmma_kernel(float* out, int iters)
{
    unsigned a[4], b[2];
#pragma unroll
    for (int k = 0; k < 4; ++k) a[k] = 0x3c003c00u ^ (threadIdx.x * 7 + k);
    b[0] = 0x3c003c00u ^ threadIdx.x;
    b[1] = 0x38003800u;
    float d[8][4];
#pragma unroll
    for (int t = 0; t < 8; ++t)
#pragma unroll
        for (int k = 0; k < 4; ++k) d[t][k] = 0.f;
    float f[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) f[k] = threadIdx.x * 1e-3f + k;
    const float w = out[4096] + 1.0001f;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int t = 0; t < 8; ++t) {
            mma16816(d[t], a, b);
#pragma unroll
            for (int k = 0; k < FF; ++k) f[k & 7] = fmaf(f[k & 7], w, 1e-7f);
        }
    }
    float s = 0.f;
#pragma unroll
    for (int t = 0; t < 8; ++t) s += d[t][0] + d[t][1] + d[t][2] + d[t][3];
#pragma unroll
    for (int k = 0; k < 8; ++k) s += f[k];
    if (s == 1234.5f) out[threadIdx.x] = s;
}

template <int FF>
void run(int sms, float* out, cudaEvent_t a, cudaEvent_t b)
{
    const int iters = 4000;
    for (int bps = 1; bps <= 8; bps *= 2) {
        dim3 grid(sms * bps);
        float ms = 0.f;
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(a);
            hmma_kernel<FF><<<grid, 128>>>(out, iters);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            cudaEventElapsedTime(&ms, a, b);
        }
        const double mmas = 8.0 * iters * grid.x * 4;            // warp MMAs
        const double tf = mmas * 4096.0 / ms / 1e9;
        const double ffma_tf = 2.0 * FF * 8.0 * iters * grid.x * 128 / ms / 1e9;
        printf("{\"ffma_per_mma\": %d, \"ctas_per_sm\": %d, \"hmma_tflops\": %.1f, \"ffma_tflops\": %.1f, "
               "\"warp_mma_per_clk_per_sm\": %.3f}\n",
               FF, bps, tf, ffma_tf, mmas / sms / (ms * 1e-3 * 1.965e9));
    }
}

int main()
{
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    float* out;
    cudaMalloc(&out, 1 << 20);
    cudaMemset(out, 0, 1 << 20);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    run<0>(sms, out, a, b);
    run<8>(sms, out, a, b);
    run<16>(sms, out, a, b);
    run<32>(sms, out, a, b);
    return 0;
}
