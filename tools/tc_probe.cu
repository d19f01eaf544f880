// tc_probe.cu -- validates the tcgen05 building blocks the stage-1 kernel relies on, and
// measures their throughput on the B200 (K2, "tcgen05 stage 1"):
//   T1  an M=128 kind::f16 MMA whose A operand is the stage-1 "entry" layout (row m = entry m
//       of 16 B; the two K chunks are two image rows LBO bytes apart), checked on the host;
//   T1b the same with LBO = 16 B (the two K chunks are entries m and m+1 of one row: overlapping
//       core matrices);  T1c  N = 24 (not a multiple of 16);
//   T2  MMA issue throughput (cycles per M=128 x N x K=16 MMA, one issuing thread per CTA);
//   T3  tcgen05.ld throughput (32x32b.x16 + wait, 4 or 8 warps).
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_1508_01292_b200/csrc -o tc_probe tools/tc_probe.cu
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include "tc05.cuh"

using namespace ccnn;

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("CUDA %s at %d: %s\n", #x, __LINE__, cudaGetErrorString(e_)); exit(1); } } while (0)

constexpr int NE = 136;            // entries per row
constexpr int RP = NE * 16;        // row pitch (bytes)

__global__ void __launch_bounds__(128) t1_kernel(const __half* R, const __half* B, float* out, int lbo, int n)
{
    extern __shared__ __align__(1024) uint8_t sm[];
    __half* sR = reinterpret_cast<__half*>(sm);                 // 2 rows
    __half* sB = reinterpret_cast<__half*>(sm + 2 * RP);        // [2 chunks][32 n][8]
    __shared__ uint32_t s_tmem;
    __shared__ __align__(8) uint64_t bar;
    for (int i = threadIdx.x; i < 2 * RP / 2; i += 128) sR[i] = R[i];
    for (int i = threadIdx.x; i < 2 * 32 * 8; i += 128) sB[i] = B[i];
    if (threadIdx.x < 32) tc05::tmem_alloc(&s_tmem, 32);
    if (threadIdx.x == 0) { tc05::mbar_init(&bar, 1); tc05::mbar_fence_init(); }
    tc05::fence_async_smem();
    tc05::fence_before();
    __syncthreads();
    tc05::fence_after();
    const uint32_t tm = s_tmem;
    if (threadIdx.x == 0) {
        const uint64_t ad = tc05::sdesc(tc05::smem_u32(sR), (uint32_t)lbo, 128);
        const uint64_t bd = tc05::sdesc(tc05::smem_u32(sB), 512, 128);
        tc05::mma_f16(tm, ad, bd, tc05::idesc_f16(128, n), 0);
        tc05::commit(&bar);
    }
    tc05::mbar_wait(&bar, 0);
    tc05::fence_after();
    const int w = threadIdx.x >> 5;
    float v[16];
    for (int h = 0; h < 2; ++h) {
        tc05::ld16(tm + ((uint32_t)(32 * w) << 16) + 16 * h, v);
        for (int i = 0; i < 16; ++i) out[threadIdx.x * 32 + 16 * h + i] = v[i];
    }
    tc05::fence_before();
    __syncthreads();
    if (threadIdx.x < 32) tc05::tmem_dealloc(tm, 32);
}

// T2: one thread issues `iters` MMAs (M=128, N, K=16) into TMEM, all into one accumulator
template <int N>
__global__ void __launch_bounds__(128) t2_kernel(long long* cyc, int iters)
{
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint32_t s_tmem;
    __shared__ __align__(8) uint64_t bar;
    for (int i = threadIdx.x; i < 16384 / 4; i += 128) reinterpret_cast<uint32_t*>(sm)[i] = 0x3c003c00u;
    if (threadIdx.x < 32) tc05::tmem_alloc(&s_tmem, 256);
    if (threadIdx.x == 0) { tc05::mbar_init(&bar, 1); tc05::mbar_fence_init(); }
    tc05::fence_async_smem();
    tc05::fence_before();
    __syncthreads();
    tc05::fence_after();
    const uint32_t tm = s_tmem;
    if (threadIdx.x == 0) {
        const uint64_t ad = tc05::sdesc(tc05::smem_u32(sm), 2176, 128);
        const uint64_t bd = tc05::sdesc(tc05::smem_u32(sm + 8192), 2048, 128);
        const long long t0 = clock64();
        for (int i = 0; i < iters; ++i) tc05::mma_f16(tm + (i & 1) * 128, ad, bd, tc05::idesc_f16(128, N), i > 1);
        tc05::commit(&bar);
        tc05::mbar_wait(&bar, 0);
        cyc[blockIdx.x] = clock64() - t0;
    }
    tc05::fence_before();
    __syncthreads();
    tc05::fence_after();
    if (threadIdx.x < 32) tc05::tmem_dealloc(tm, 256);
}

// T3: every warp loads 16 columns x its 32 lanes `iters` times
__global__ void t3_kernel(long long* cyc, float* sink, int iters)
{
    __shared__ uint32_t s_tmem;
    if (threadIdx.x < 32) tc05::tmem_alloc(&s_tmem, 256);
    tc05::fence_before();
    __syncthreads();
    tc05::fence_after();
    const uint32_t tm = s_tmem;
    const int w = threadIdx.x >> 5;
    const uint32_t base = tm + ((uint32_t)(32 * (w & 3)) << 16) + 16 * (w >> 2);
    float acc = 0.f, v[16];
    __syncthreads();
    const long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        tc05::ld16(base + 32 * (i & 3), v);
#pragma unroll
        for (int k = 0; k < 16; ++k) acc += v[k];
    }
    __syncthreads();
    if (threadIdx.x == 0) cyc[blockIdx.x] = clock64() - t0;
    sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    tc05::fence_before();
    __syncthreads();
    tc05::fence_after();
    if (threadIdx.x < 32) tc05::tmem_dealloc(tm, 256);
}


// T4: A (128 x 16 fp16) written to TMEM with tcgen05.st from registers, B from smem
__global__ void __launch_bounds__(128) t4_kernel(const __half* A, const __half* B, float* out, int n)
{
    extern __shared__ __align__(1024) uint8_t sm[];
    __half* sB = reinterpret_cast<__half*>(sm);                 // [2 chunks][32 n][8]
    __shared__ uint32_t s_tmem;
    __shared__ __align__(8) uint64_t bar;
    for (int i = threadIdx.x; i < 2 * 32 * 8; i += 128) sB[i] = B[i];
    if (threadIdx.x < 32) tc05::tmem_alloc(&s_tmem, 64);
    if (threadIdx.x == 0) { tc05::mbar_init(&bar, 1); tc05::mbar_fence_init(); }
    tc05::fence_async_smem();
    tc05::fence_before();
    __syncthreads();
    tc05::fence_after();
    const uint32_t tm = s_tmem;
    const int w = threadIdx.x >> 5;
    const uint32_t lane_base = (uint32_t)(32 * w) << 16;
    // row m = threadIdx.x: 16 fp16 -> 8 words at columns 32..39
    const uint32_t* a32 = reinterpret_cast<const uint32_t*>(A) + threadIdx.x * 8;
    tc05::st4(tm + lane_base + 32, a32[0], a32[1], a32[2], a32[3]);
    tc05::st4(tm + lane_base + 36, a32[4], a32[5], a32[6], a32[7]);
    tc05::st_wait();
    tc05::fence_before();
    __syncthreads();
    tc05::fence_after();
    if (threadIdx.x == 0) {
        const uint64_t bd = tc05::sdesc(tc05::smem_u32(sB), 512, 128);
        tc05::mma_f16_ts(tm, tm + 32, bd, tc05::idesc_f16(128, n), 0);
        tc05::commit(&bar);
    }
    tc05::mbar_wait(&bar, 0);
    tc05::fence_after();
    float v[16];
    for (int h = 0; h < 2; ++h) {
        tc05::ld16(tm + lane_base + 16 * h, v);
        for (int i = 0; i < 16; ++i) out[threadIdx.x * 32 + 16 * h + i] = v[i];
    }
    tc05::fence_before();
    __syncthreads();
    if (threadIdx.x < 32) tc05::tmem_dealloc(tm, 64);
}

// T5: MMA throughput with A in TMEM (TS) or A in smem at a different address every MMA (SS)
template <int N, bool TS, int CH>
__global__ void __launch_bounds__(128) t5_kernel(long long* cyc, int iters)
{
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint32_t s_tmem;
    __shared__ __align__(8) uint64_t bar;
    for (int i = threadIdx.x; i < 65536 / 4; i += 128) reinterpret_cast<uint32_t*>(sm)[i] = 0x3c003c00u;
    if (threadIdx.x < 32) tc05::tmem_alloc(&s_tmem, 256);
    if (threadIdx.x == 0) { tc05::mbar_init(&bar, 1); tc05::mbar_fence_init(); }
    tc05::fence_async_smem();
    tc05::fence_before();
    __syncthreads();
    tc05::fence_after();
    const uint32_t tm = s_tmem;
    if (threadIdx.x == 0) {
        const uint64_t bd = tc05::sdesc(tc05::smem_u32(sm + 49152), 4096, 128);
        const long long t0 = clock64();
        for (int i = 0; i < iters; ++i) {
            const uint32_t d = tm + (i % CH) * (128 / CH);
            if (TS) tc05::mma_f16_ts(d, tm + 128 + 8 * (i & 7), bd, tc05::idesc_f16(128, N), i >= CH);
            else tc05::mma_f16(d, tc05::sdesc(tc05::smem_u32(sm + 2048 * (i & 15)), 4096, 128), bd,
                               tc05::idesc_f16(128, N), i >= CH);
        }
        tc05::commit(&bar);
        tc05::mbar_wait(&bar, 0);
        cyc[blockIdx.x] = clock64() - t0;
    }
    tc05::fence_before();
    __syncthreads();
    tc05::fence_after();
    if (threadIdx.x < 32) tc05::tmem_dealloc(tm, 256);
}

static float h2f(__half h) { return __half2float(h); }

static int run_t1(int lbo, int n, const char* name)
{
    std::vector<__half> R(2 * RP / 2), B(2 * 32 * 8);
    for (int r = 0; r < 2; ++r)
        for (int e = 0; e < NE; ++e)
            for (int c = 0; c < 8; ++c) R[(r * NE + e) * 8 + c] = __float2half((float)(((r * 7 + e * 3 + c * 5) % 17) - 8));
    for (int ch = 0; ch < 2; ++ch)
        for (int nn = 0; nn < 32; ++nn)
            for (int c = 0; c < 8; ++c) B[(ch * 32 + nn) * 8 + c] = __float2half((float)(((ch * 11 + nn * 5 + c * 3) % 13) - 6) * 0.25f);
    __half *dR, *dB;
    float* dO;
    CK(cudaMalloc(&dR, R.size() * 2)); CK(cudaMalloc(&dB, B.size() * 2)); CK(cudaMalloc(&dO, 128 * 32 * 4));
    CK(cudaMemcpy(dR, R.data(), R.size() * 2, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dB, B.data(), B.size() * 2, cudaMemcpyHostToDevice));
    CK(cudaMemset(dO, 0, 128 * 32 * 4));
    const int smem = 2 * RP + 2 * 32 * 16;
    CK(cudaFuncSetAttribute(t1_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    t1_kernel<<<1, 128, smem>>>(dR, dB, dO, lbo, n);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("{\"test\": \"%s\", \"error\": \"%s\"}\n", name, cudaGetErrorString(e)); return 1; }
    std::vector<float> O(128 * 32);
    CK(cudaMemcpy(O.data(), dO, O.size() * 4, cudaMemcpyDeviceToHost));
    int bad = 0;
    double maxerr = 0;
    for (int m = 0; m < 128; ++m)
        for (int nn = 0; nn < n; ++nn) {
            double ref = 0;
            for (int k = 0; k < 16; ++k) {
                const int ch = k >> 3, c = k & 7;
                // chunk 1 sits LBO bytes after chunk 0: entry index offset lbo/16 in the flat array
                const int flat = m + ch * (lbo / 16);
                const float a = h2f(R[flat * 8 + c]);
                ref += (double)a * h2f(B[(ch * 32 + nn) * 8 + c]);
            }
            const double d = fabs(ref - O[m * 32 + nn]);
            if (d > maxerr) maxerr = d;
            if (d > 1e-3) ++bad;
        }
    printf("{\"test\": \"%s\", \"lbo\": %d, \"n\": %d, \"bad\": %d, \"max_err\": %g, \"d00\": %g}\n", name, lbo, n, bad, maxerr, O[0]);
    cudaFree(dR); cudaFree(dB); cudaFree(dO);
    return bad != 0;
}

template <int N>
static void run_t2(int sms)
{
    long long* d;
    CK(cudaMalloc(&d, sizeof(long long) * sms * 4));
    CK(cudaFuncSetAttribute(t2_kernel<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384));
    for (int per = 1; per <= 2; ++per) {
        const int iters = 4096;
        t2_kernel<N><<<sms * per, 128, 16384>>>(d, iters);
        CK(cudaDeviceSynchronize());
        std::vector<long long> h(sms * per);
        CK(cudaMemcpy(h.data(), d, h.size() * 8, cudaMemcpyDeviceToHost));
        double s = 0;
        for (long long x : h) s += x;
        printf("{\"test\": \"T2 mma\", \"M\": 128, \"N\": %d, \"ctas_per_sm\": %d, \"cycles_per_mma\": %.2f}\n", N, per,
               s / h.size() / iters);
    }
    cudaFree(d);
}

static void run_t3(int sms)
{
    long long* d;
    float* sink;
    CK(cudaMalloc(&d, sizeof(long long) * sms * 2));
    CK(cudaMalloc(&sink, sizeof(float) * sms * 2 * 256));
    for (int warps = 4; warps <= 8; warps += 4)
        for (int per = 1; per <= 2; ++per) {
            const int iters = 2048;
            t3_kernel<<<sms * per, 32 * warps>>>(d, sink, iters);
            CK(cudaDeviceSynchronize());
            std::vector<long long> h(sms * per);
            CK(cudaMemcpy(h.data(), d, h.size() * 8, cudaMemcpyDeviceToHost));
            double s = 0;
            for (long long x : h) s += x;
            const double cyc = s / h.size();
            const double bytes = (double)iters * warps * 32 * 16 * 4 * per;   // per SM
            printf("{\"test\": \"T3 tmem ld x16\", \"warps\": %d, \"ctas_per_sm\": %d, \"cycles_per_ld\": %.2f, \"bytes_per_cycle_per_sm\": %.1f}\n",
                   warps, per, cyc / iters, bytes / cyc);
        }
    cudaFree(d); cudaFree(sink);
}


static int run_t4(int n)
{
    std::vector<__half> A(128 * 16), B(2 * 32 * 8);
    for (int m = 0; m < 128; ++m)
        for (int k = 0; k < 16; ++k) A[m * 16 + k] = __float2half((float)(((m * 5 + k * 7) % 19) - 9));
    for (int ch = 0; ch < 2; ++ch)
        for (int nn = 0; nn < 32; ++nn)
            for (int c = 0; c < 8; ++c) B[(ch * 32 + nn) * 8 + c] = __float2half((float)(((ch * 11 + nn * 5 + c * 3) % 13) - 6) * 0.25f);
    __half *dA, *dB;
    float* dO;
    CK(cudaMalloc(&dA, A.size() * 2)); CK(cudaMalloc(&dB, B.size() * 2)); CK(cudaMalloc(&dO, 128 * 32 * 4));
    CK(cudaMemcpy(dA, A.data(), A.size() * 2, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dB, B.data(), B.size() * 2, cudaMemcpyHostToDevice));
    t4_kernel<<<1, 128, 2 * 32 * 16>>>(dA, dB, dO, n);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("{\"test\": \"T4\", \"error\": \"%s\"}\n", cudaGetErrorString(e)); return 1; }
    std::vector<float> O(128 * 32);
    CK(cudaMemcpy(O.data(), dO, O.size() * 4, cudaMemcpyDeviceToHost));
    int bad = 0;
    for (int m = 0; m < 128; ++m)
        for (int nn = 0; nn < n; ++nn) {
            double ref = 0;
            for (int k = 0; k < 16; ++k) ref += (double)h2f(A[m * 16 + k]) * h2f(B[((k >> 3) * 32 + nn) * 8 + (k & 7)]);
            if (fabs(ref - O[m * 32 + nn]) > 1e-3) ++bad;
        }
    printf("{\"test\": \"T4 A in TMEM\", \"n\": %d, \"bad\": %d}\n", n, bad);
    return bad != 0;
}

template <int N, bool TS, int CH>
static void run_t5(int sms)
{
    long long* d;
    CK(cudaMalloc(&d, sizeof(long long) * sms * 4));
    CK(cudaFuncSetAttribute(t5_kernel<N, TS, CH>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536));
    for (int per = 1; per <= 2; ++per) {
        const int iters = 4096;
        t5_kernel<N, TS, CH><<<sms * per, 128, 65536>>>(d, iters);
        CK(cudaDeviceSynchronize());
        std::vector<long long> h(sms * per);
        CK(cudaMemcpy(h.data(), d, h.size() * 8, cudaMemcpyDeviceToHost));
        double s = 0;
        for (long long x : h) s += x;
        printf("{\"test\": \"T5 mma %s\", \"N\": %d, \"chains\": %d, \"ctas_per_sm\": %d, \"cycles_per_mma_per_sm\": %.2f}\n",
               TS ? "A in TMEM" : "SS distinct A", N, CH, per, s / h.size() / iters / per);
    }
    cudaFree(d);
}

// T6: cheap issue: descriptors fixed per 8-MMA group (compile-time offsets), ISSUERS warps each
// issue into their own accumulators
template <int N, bool TS, int ISSUERS, int CH = 1>
__global__ void __launch_bounds__(128) t6_kernel(long long* cyc, int iters)
{
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint32_t s_tmem;
    __shared__ __align__(8) uint64_t bar[4];
    for (int i = threadIdx.x; i < 65536 / 4; i += 128) reinterpret_cast<uint32_t*>(sm)[i] = 0x3c003c00u;
    if (threadIdx.x < 32) tc05::tmem_alloc(&s_tmem, 256);
    if (threadIdx.x == 0) { for (int k = 0; k < 4; ++k) tc05::mbar_init(&bar[k], 1); tc05::mbar_fence_init(); }
    tc05::fence_async_smem();
    tc05::fence_before();
    __syncthreads();
    tc05::fence_after();
    const uint32_t tm = s_tmem;
    const int w = threadIdx.x >> 5;
    if (w < ISSUERS && (threadIdx.x & 31) == 0) {
        const uint64_t bd = tc05::sdesc(tc05::smem_u32(sm + 49152), 4096, 128);
        const uint64_t ad = tc05::sdesc(tc05::smem_u32(sm), 4096, 128);
        const uint32_t id = tc05::idesc_f16(128, N);
        const uint32_t dbase = tm + w * 32;
        const long long t0 = clock64();
        for (int i = 0; i < iters; i += 8) {
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                if (TS) tc05::mma_f16_ts(dbase + (k % CH) * (32 / CH), tm + 128 + 8 * k, bd, id, 1);
                else tc05::mma_f16(dbase + (k % CH) * (32 / CH), ad + (uint64_t)(k * 128), bd, id, 1);
            }
        }
        tc05::commit(&bar[w]);
        tc05::mbar_wait(&bar[w], 0);
        cyc[blockIdx.x * 4 + w] = clock64() - t0;
    }
    tc05::fence_before();
    __syncthreads();
    tc05::fence_after();
    if (threadIdx.x < 32) tc05::tmem_dealloc(tm, 256);
}
template <int N, bool TS, int ISSUERS, int CH = 1>
static void run_t6(int sms)
{
    long long* d;
    CK(cudaMalloc(&d, sizeof(long long) * sms * 8 * 4));
    CK(cudaFuncSetAttribute(t6_kernel<N, TS, ISSUERS, CH>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536));
    for (int per = 1; per <= 2; ++per) {
        const int iters = 4096;
        t6_kernel<N, TS, ISSUERS, CH><<<sms * per, 128, 65536>>>(d, iters);
        CK(cudaDeviceSynchronize());
        std::vector<long long> h(sms * per * 4);
        CK(cudaMemcpy(h.data(), d, h.size() * 8, cudaMemcpyDeviceToHost));
        double mx = 0;
        for (int b = 0; b < sms * per; ++b) for (int w = 0; w < ISSUERS; ++w) mx += h[b * 4 + w];
        mx /= sms * per * ISSUERS;
        printf("{\"test\": \"T6 mma %s unrolled\", \"N\": %d, \"issuers\": %d, \"chains\": %d, \"ctas_per_sm\": %d, \"cycles_per_mma_per_sm\": %.2f}\n",
               TS ? "A in TMEM" : "SS", N, ISSUERS, CH, per, mx / (iters * ISSUERS * per));
    }
    cudaFree(d);
}

// T7: does issuing tcgen05.mma stall the issuing warp's other work?  Warp 0: lane 0 issues 8
// MMAs per iteration (if DO_MMA), then every lane runs FF dependent-free FFMAs (if FF > 0)
template <bool DO_MMA, int FF, bool ELECT>
__global__ void __launch_bounds__(128) t7_kernel(long long* cyc, float* sink, int iters)
{
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint32_t s_tmem;
    __shared__ __align__(8) uint64_t bar;
    for (int i = threadIdx.x; i < 65536 / 4; i += 128) reinterpret_cast<uint32_t*>(sm)[i] = 0x3c003c00u;
    if (threadIdx.x < 32) tc05::tmem_alloc(&s_tmem, 256);
    if (threadIdx.x == 0) { tc05::mbar_init(&bar, 1); tc05::mbar_fence_init(); }
    tc05::fence_async_smem();
    tc05::fence_before();
    __syncthreads();
    tc05::fence_after();
    const uint32_t tm = s_tmem;
    if (threadIdx.x < 32) {
        const uint64_t bd = tc05::sdesc(tc05::smem_u32(sm + 49152), 4096, 128);
        const uint32_t id = tc05::idesc_f16(128, 24);
        float f[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) f[k] = threadIdx.x * 1e-3f + k;
        const float wv = sink[0] + 1.0001f;
        const long long t0 = clock64();
        for (int i = 0; i < iters; i += 8) {
            if (DO_MMA) {
                if (ELECT) {
                    if (tc05::elect_one()) {
#pragma unroll
                        for (int k = 0; k < 8; ++k) tc05::mma_f16_ts(tm + 32 * (k & 3), tm + 128 + 8 * k, bd, id, 1);
                    }
                } else if (threadIdx.x == 0) {
#pragma unroll
                    for (int k = 0; k < 8; ++k) tc05::mma_f16_ts(tm + 32 * (k & 3), tm + 128 + 8 * k, bd, id, 1);
                }
            }
            __syncwarp();
#pragma unroll
            for (int k = 0; k < FF; ++k) f[k & 7] = fmaf(f[k & 7], wv, 1e-7f);
        }
        if (DO_MMA && threadIdx.x == 0) { tc05::commit(&bar); tc05::mbar_wait(&bar, 0); }
        __syncwarp();
        if (threadIdx.x == 0) cyc[blockIdx.x] = clock64() - t0;
        float t = 0.f;
#pragma unroll
        for (int k = 0; k < 8; ++k) t += f[k];
        if (t == 1234.f) sink[1 + threadIdx.x] = t;
    }
    tc05::fence_before();
    __syncthreads();
    tc05::fence_after();
    if (threadIdx.x < 32) tc05::tmem_dealloc(tm, 256);
}
template <bool DO_MMA, int FF, bool ELECT>
static void run_t7(int sms)
{
    long long* d;
    float* sink;
    CK(cudaMalloc(&d, sizeof(long long) * sms));
    CK(cudaMalloc(&sink, 4096));
    CK(cudaMemset(sink, 0, 4096));
    CK(cudaFuncSetAttribute(t7_kernel<DO_MMA, FF, ELECT>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536));
    const int iters = 4096;
    t7_kernel<DO_MMA, FF, ELECT><<<sms, 128, 65536>>>(d, sink, iters);
    CK(cudaDeviceSynchronize());
    std::vector<long long> h(sms);
    CK(cudaMemcpy(h.data(), d, h.size() * 8, cudaMemcpyDeviceToHost));
    double m = 0;
    for (long long x : h) m += x;
    printf("{\"test\": \"T7 issue stall\", \"mma\": %d, \"elect\": %d, \"ffma_per_8mma\": %d, \"cycles_per_8mma_iter\": %.1f}\n",
           (int)DO_MMA, (int)ELECT, FF, m / sms / (iters / 8));
    cudaFree(d); cudaFree(sink);
}

int main()
{
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    int fails = 0;
    fails += run_t1(RP, 32, "T1 two-row chunks");
    fails += run_t1(16, 32, "T1b overlapping chunks");
    fails += run_t1(RP, 24, "T1c N=24");
    fails += run_t1(RP, 16, "T1d N=16");
    fails += run_t4(24);
    fails += run_t4(32);
    run_t7<true, 0, false>(sms);
    run_t7<true, 0, true>(sms);
    run_t7<false, 256, true>(sms);
    run_t7<true, 256, true>(sms);
    printf("{\"fails\": %d}\n", fails);
    return 0;
}
