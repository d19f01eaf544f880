// tc2_probe.cu -- cta_group::2 (CTA-pair) tcgen05 building blocks for a paired stage-1 kernel:
//   P1  SS MMA M=256 (128 rows per CTA), N=32, K=16; B split along N between the two CTAs
//       (hypothesis H1: CTA r holds B rows [r N/2, (r+1) N/2) at the same smem offset);
//       the leader issues, the commit is multicast to both CTAs' mbarriers;
//   P2  the same with A in TMEM (each CTA's 128 rows written by tcgen05.st);
//   P3  issue throughput: cycles per paired MMA (SS / TS, N = 48 / 96), 1 or 2 pairs per TPC.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_1508_01292_b200/csrc -o tc2_probe tools/tc2_probe.cu
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include "tc05.cuh"

using namespace ccnn;

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("{\"error\": \"%s at %d: %s\"}\n", #x, __LINE__, cudaGetErrorString(e_)); exit(1); } } while (0)

__device__ __forceinline__ uint32_t cta_rank()
{
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync()
{
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void alloc2(uint32_t* dst, uint32_t ncols)
{
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" :: "r"(tc05::smem_u32(dst)), "r"(ncols) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void dealloc2(uint32_t taddr, uint32_t ncols)
{
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" :: "r"(taddr), "r"(ncols) : "memory");
}
__device__ __forceinline__ void mma2_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc)
{
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}"
                 :: "r"(d), "l"(a), "l"(b), "r"(idesc), "r"(acc) : "memory");
}
__device__ __forceinline__ void mma2_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, uint32_t acc)
{
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n\t}"
                 :: "r"(d), "r"(a), "l"(b), "r"(idesc), "r"(acc) : "memory");
}
__device__ __forceinline__ void commit2(uint64_t* bar)
{
    asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
                 :: "r"(tc05::smem_u32(bar)), "h"((uint16_t)3) : "memory");
}

// A: [k chunk 2][m 128][8] fp16 per CTA; B (this CTA's N/2 rows): [k chunk 2][n N/2][8]
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128) p1_kernel(const __half* A, const __half* B, float* out,
                                                                      int n, int ts)
{
    __shared__ __align__(1024) __half sA[2 * 128 * 8];
    __shared__ __align__(1024) __half sB[2 * 128 * 8];
    __shared__ uint32_t s_tmem;
    __shared__ __align__(8) uint64_t bar;
    const uint32_t r = cta_rank();
    const int nh = n / 2;
    for (int i = threadIdx.x; i < 2 * 128 * 8; i += 128) sA[i] = A[r * 2048 + i];
    for (int i = threadIdx.x; i < 2 * nh * 8; i += 128) {
        const int kc = i / (nh * 8), rem = i % (nh * 8), nn = rem / 8, kk = rem % 8;
        sB[i] = B[(kc * n + r * nh + nn) * 8 + kk];
    }
    if (threadIdx.x < 32) alloc2(&s_tmem, 128);
    if (threadIdx.x == 0) { tc05::mbar_init(&bar, 1); tc05::mbar_fence_init(); }
    tc05::fence_async_smem();
    tc05::fence_before();
    __syncthreads();
    tc05::fence_after();
    const uint32_t tm = s_tmem;
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31, m = threadIdx.x;
    if (ts) {   // A row m -> TMEM lane m, columns 112 .. 119 (K = 16 = 8 x 32-bit)
        uint32_t v[8];
        for (int c = 0; c < 8; ++c) {
            const int k0 = 2 * c;
            const __half lo = sA[(k0 / 8) * 1024 + m * 8 + (k0 % 8)];
            const __half hi = sA[((k0 + 1) / 8) * 1024 + m * 8 + ((k0 + 1) % 8)];
            v[c] = (uint32_t)__half_as_ushort(lo) | ((uint32_t)__half_as_ushort(hi) << 16);
        }
        const uint32_t ta = tm + ((uint32_t)(32 * w) << 16) + 112;
        tc05::st4(ta, v[0], v[1], v[2], v[3]);
        tc05::st4(ta + 4, v[4], v[5], v[6], v[7]);
        tc05::st_wait();
    }
    tc05::fence_before();
    cluster_sync();
    tc05::fence_after();
    if (r == 0 && threadIdx.x == 0) {
        const uint64_t bd = tc05::sdesc(tc05::smem_u32(sB), (uint32_t)(nh * 16), 128);
        const uint32_t idesc = tc05::idesc_f16(256, n);
        if (ts) mma2_ts(tm, tm + 112, bd, idesc, 0);
        else mma2_ss(tm, tc05::sdesc(tc05::smem_u32(sA), 2048, 128), bd, idesc, 0);
        commit2(&bar);
    }
    tc05::mbar_wait(&bar, 0);
    tc05::fence_after();
    float v[16];
    for (int h = 0; h < n / 16; ++h) {
        tc05::ld16(tm + ((uint32_t)(32 * w) << 16) + 16 * h, v);
        for (int i = 0; i < 16; ++i) out[(r * 128 + m) * n + 16 * h + i] = v[i];
    }
    (void)lane;
    tc05::fence_before();
    cluster_sync();
    if (threadIdx.x < 32) dealloc2(tm, 128);
}

// throughput: the leader issues `iters` MMAs (A in smem or TMEM, N), one commit at the end
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128) p3_kernel(long long* cyc, int iters, int n, int ts)
{
    __shared__ __align__(1024) __half sA[2 * 128 * 8];
    __shared__ __align__(1024) __half sB[2 * 128 * 8];
    __shared__ uint32_t s_tmem;
    __shared__ __align__(8) uint64_t bar;
    const uint32_t r = cta_rank();
    for (int i = threadIdx.x; i < 2 * 128 * 8; i += 128) { sA[i] = __float2half(0.f); sB[i] = __float2half(0.f); }
    if (threadIdx.x < 32) alloc2(&s_tmem, 128);
    if (threadIdx.x == 0) { tc05::mbar_init(&bar, 1); tc05::mbar_fence_init(); }
    tc05::fence_async_smem();
    tc05::fence_before();
    __syncthreads();
    tc05::fence_after();
    const uint32_t tm = s_tmem;
    cluster_sync();
    tc05::fence_after();
    if (r == 0 && threadIdx.x == 0) {
        const uint64_t bd = tc05::sdesc(tc05::smem_u32(sB), (uint32_t)(n / 2 * 16), 128);
        const uint64_t ad = tc05::sdesc(tc05::smem_u32(sA), 2048, 128);
        const uint32_t idesc = tc05::idesc_f16(256, n);
        const long long t0 = clock64();
        for (int i = 0; i < iters; ++i) {
            if (ts) mma2_ts(tm, tm + 100, bd, idesc, i != 0);
            else mma2_ss(tm, ad, bd, idesc, i != 0);
        }
        commit2(&bar);
        tc05::mbar_wait(&bar, 0);
        cyc[blockIdx.x / 2] = clock64() - t0;
    } else {
        tc05::mbar_wait(&bar, 0);
    }
    tc05::fence_before();
    cluster_sync();
    if (threadIdx.x < 32) dealloc2(tm, 128);
}

int main()
{
    // ---- P1 / P2 correctness ----
    for (int ts = 0; ts < 2; ++ts)
        for (int n : {32, 48, 96}) {
            std::vector<__half> A(2 * 2048), B(2 * n * 8);
            std::vector<float> ha(2 * 128 * 16), hb(n * 16);
            srand(7 + n + ts);
            for (int r = 0; r < 2; ++r)
                for (int kc = 0; kc < 2; ++kc)
                    for (int m = 0; m < 128; ++m)
                        for (int kk = 0; kk < 8; ++kk) {
                            const float v = (float)(rand() % 7 - 3);
                            A[r * 2048 + kc * 1024 + m * 8 + kk] = __float2half(v);
                            ha[(r * 128 + m) * 16 + kc * 8 + kk] = v;
                        }
            for (int kc = 0; kc < 2; ++kc)
                for (int nn = 0; nn < n; ++nn)
                    for (int kk = 0; kk < 8; ++kk) {
                        const float v = (float)(rand() % 5 - 2);
                        B[(kc * n + nn) * 8 + kk] = __float2half(v);
                        hb[nn * 16 + kc * 8 + kk] = v;
                    }
            __half *dA, *dB;
            float* dO;
            CK(cudaMalloc(&dA, A.size() * 2));
            CK(cudaMalloc(&dB, B.size() * 2));
            CK(cudaMalloc(&dO, 256 * n * 4));
            CK(cudaMemcpy(dA, A.data(), A.size() * 2, cudaMemcpyHostToDevice));
            CK(cudaMemcpy(dB, B.data(), B.size() * 2, cudaMemcpyHostToDevice));
            CK(cudaMemset(dO, 0, 256 * n * 4));
            p1_kernel<<<2, 128>>>(dA, dB, dO, n, ts);
            CK(cudaGetLastError());
            CK(cudaDeviceSynchronize());
            std::vector<float> o(256 * n);
            CK(cudaMemcpy(o.data(), dO, o.size() * 4, cudaMemcpyDeviceToHost));
            int bad = 0;
            double maxerr = 0;
            for (int m = 0; m < 256; ++m)
                for (int nn = 0; nn < n; ++nn) {
                    float ref = 0;
                    for (int k = 0; k < 16; ++k) ref += ha[m * 16 + k] * hb[nn * 16 + k];
                    const double e = fabs(ref - o[m * n + nn]);
                    if (e > 1e-3) ++bad;
                    if (e > maxerr) maxerr = e;
                }
            printf("{\"test\": \"P%d pair MMA %s\", \"n\": %d, \"bad\": %d, \"max_err\": %g, \"d00\": %g, \"d_last\": %g}\n",
                   ts ? 2 : 1, ts ? "TS" : "SS", n, bad, maxerr, o[0], o[255 * n + n - 1]);
            cudaFree(dA); cudaFree(dB); cudaFree(dO);
        }
    // ---- P3 throughput ----
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    long long* dc;
    CK(cudaMalloc(&dc, sizeof(long long) * 4 * sms));
    for (int ts = 0; ts < 2; ++ts)
        for (int n : {32, 48, 96})
            for (int pairs_per_tpc : {1, 2}) {
                const int clusters = sms / 2 * pairs_per_tpc;
                const int iters = 2048;
                p3_kernel<<<2 * clusters, 128>>>(dc, iters, n, ts);
                CK(cudaGetLastError());
                CK(cudaDeviceSynchronize());
                std::vector<long long> c(clusters);
                CK(cudaMemcpy(c.data(), dc, sizeof(long long) * clusters, cudaMemcpyDeviceToHost));
                double avg = 0;
                for (long long x : c) avg += (double)x;
                avg /= clusters;
                // per TPC: pairs_per_tpc pairs share the two SMs' tensor cores
                printf("{\"test\": \"P3 pair MMA issue\", \"ts\": %d, \"N\": %d, \"pairs_per_tpc\": %d, "
                       "\"cycles_per_mma_per_pair\": %.2f, \"cycles_per_mma_per_tpc\": %.2f}\n",
                       ts, n, pairs_per_tpc, avg / iters, avg / iters / pairs_per_tpc);
            }
    return 0;
}
