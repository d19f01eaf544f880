// selective.cu -- stage 3 of the cascade and the decision rule on every stage-1 survivor
// (K3), after selective_tc.cu has computed CNN2's 50 responses (resp2).
//
// PAPER.md §3.3: K = number of responses exceeding T2; Eq. 2 (strict) with the
// early stop of P:99 -- CNN3 runs only when the rule needs it -- or Eq. 3 (weak).
// Readings O7-O8: K pooled over both orientations, the score = the max response of
// the last net evaluated, the raw box = the stage-1 window mapped back.
//
// B200 design: a persistent kernel whose WARPS drain the survivor queue independently (one
// atomic claim per survivor, no block barriers): K2 from resp2 by two ballots and the stop
// decision (with few survivors -- at most 4 per CTA: small frames, sparse 4K -- a whole CTA
// takes each survivor instead, the same code over 6 warps: latency); otherwise CNN3 on the equalised patch E that selective_tc.cu left in epatch, on the
// FFMA pipe (2-map layers: no dense contraction for the tensor cores), in the warp's own
// shared-memory slice:
//  * layer 1 (C4x4 1->2, pool, act), one orientation at a time: a lane computes 4 adjacent
//    pooled outputs of both maps from a 5 x 11 pixel block; the mirrored patch
//    M(x, y) = E(50 - x, y) is read through mirrored addresses;
//  * layer 2 (C3x3 2->2, pool, act): a lane per pooled position;
//  * layer 3 (C7x8 2->25, act): a lane per map (25 lanes), one input channel at a time with its
//    7 x 8 kernel in registers (from a per-CTA shared copy), 5 response cells at a time from P2
//    rows broadcast as float4s -- 0.1 shared loads per FMA, no constant-cache traffic;
//  * layer 4 (C1x1 25->1, act): a lane per response cell.
// CNN3 = architecture R (R1): C4x4 1->2, P, C3x3 2->2, P, C7x8 2->25, C1x1 25->1.
#include <cstdlib>

#include "ccnn_internal.h"
#include "selective_common.cuh"

namespace ccnn {
namespace {

constexpr int kWarps = 6;                   // warps per CTA (each works alone)
constexpr int kW3S = 113;                   // layer-3 weights per map in shared memory: [ch*56 +
                                            // ky*7 + kx], bias at 112; odd stride: lanes = maps
                                            // read distinct banks
constexpr int kL3S = 51;                    // layer-3 sums per map: [cell], odd stride

constexpr size_t kW3Bytes = (25 * kW3S * 4 + 15) / 16 * 16;

struct WarpSmem {                           // one warp's slice
    uint32_t e[kEPatchBytes / 4];           // E, row-major 51 x 55 bytes (epatch's layout)
    union {
        float p1[2][26][24];                // pooled layer 1 of one orientation [map][y][x]
        float l3[25 * kL3S];                // layer 3 [map][cell] (after P1 is consumed)
    };
    alignas(16) float p2[2][2][12][12];     // pooled layer 2 [orientation][map][y][x] (12 x 11)
};

__device__ __forceinline__ float act(float x)      // Eq. 1, see stage1_tc.cu
{
    const float a = fabsf(x) * (2.0f / 3.0f);
    const float a2 = a * a;
    const float p = fmaf(a2, fmaf(a2, 1.41645f, 1.0f), a + 1.0f);
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(p));
    return copysignf(fmaf(-1.7159f, r, 1.7159f), x);
}

// CNN3 on both orientations of the group's patch, by a group of G warps (G = 1: one warp per
// survivor, the throughput form; G = kWarps: the whole CTA on one survivor, the latency form
// used when there are no more survivors than CTAs).  gt = thread index in the group; thread gt
// returns the responses of cells gt and gt + 32 G (cell c = orientation c / 25, position c % 25;
// -inf past 49)
template <int G>
__device__ __forceinline__ void group_sync()
{
    if constexpr (G == 1) __syncwarp();
    else __syncthreads();
}
template <int G>
__device__ __forceinline__ void cnn3_group(const Cnn3W& W, const float* __restrict__ w3s, WarpSmem& S,
                                           int gt, float (&r)[2])
{
    constexpr int NG = 32 * G;
    const int lane = gt & 31, wg = gt >> 5;
    const uint8_t* e = reinterpret_cast<const uint8_t*>(S.e);
#pragma unroll 1
    for (int o = 0; o < 2; ++o) {
        // ---- layer 1: item = (pooled row py, pooled columns 4q .. 4q+3): 26 x 6 items ----
#pragma unroll 1
        for (int it = gt; it < 26 * 6; it += NG) {
            const int py = it / 6, q = it - py * 6;
            // image column 8q + c is E column x0 + dx * c: M(x) = E(50 - x) for o = 1 (one code
            // path for both orientations keeps the kernel's instruction footprint small)
            const uint8_t* e0 = e + 2 * py * kPatchW + (o == 0 ? 8 * q : 50 - 8 * q);
            const int dx = o == 0 ? 1 : -1;
            float x[5][11];                        // image rows 2py .. +4, columns 8q .. 8q+10
#pragma unroll
            for (int rr = 0; rr < 5; ++rr)
#pragma unroll
                for (int c = 0; c < 11; ++c)
                    x[rr][c] = fmaf((float)e0[rr * kPatchW + dx * c], 1.0f / 127.5f, -1.0f);   // O3
#pragma unroll
            for (int a = 0; a < 2; ++a)
#pragma unroll
                for (int j = 0; j < 4; ++j) {       // pooled column 4q + j: conv columns 8q + 2j + {0,1}
                    float sv[4];
#pragma unroll
                    for (int p = 0; p < 4; ++p) {
                        sv[p] = W.b1[a];
#pragma unroll
                        for (int ky = 0; ky < 4; ++ky)
#pragma unroll
                            for (int kx = 0; kx < 4; ++kx)
                                sv[p] = fmaf(W.w1[a][ky * 4 + kx], x[(p >> 1) + ky][2 * j + (p & 1) + kx], sv[p]);
                    }
                    S.p1[a][py][4 * q + j] = act(fmaxf(fmaxf(sv[0], sv[1]), fmaxf(sv[2], sv[3])));  // pool, act
                }
        }
        group_sync<G>();
        // ---- layer 2: item = pooled position (12 rows x 11 columns) ----
#pragma unroll 1
        for (int it = gt; it < 12 * 11; it += NG) {
            const int py = it / 11, px = it - py * 11;
            float s2[2][4];
#pragma unroll
            for (int b = 0; b < 2; ++b)
#pragma unroll
                for (int k = 0; k < 4; ++k) s2[b][k] = W.b2[b];
#pragma unroll
            for (int a = 0; a < 2; ++a) {
                float v[4][4];
#pragma unroll
                for (int rr = 0; rr < 4; ++rr)
#pragma unroll
                    for (int c = 0; c < 4; ++c) v[rr][c] = S.p1[a][2 * py + rr][2 * px + c];
#pragma unroll
                for (int b = 0; b < 2; ++b)
#pragma unroll
                    for (int ky = 0; ky < 3; ++ky)
#pragma unroll
                        for (int kx = 0; kx < 3; ++kx)
#pragma unroll
                            for (int k = 0; k < 4; ++k)
                                s2[b][k] = fmaf(W.w2[b][a][ky * 3 + kx], v[(k >> 1) + ky][(k & 1) + kx], s2[b][k]);
            }
#pragma unroll
            for (int b = 0; b < 2; ++b)
                S.p2[o][b][py][px] = act(fmaxf(fmaxf(s2[b][0], s2[b][1]), fmaxf(s2[b][2], s2[b][3])));
        }
        group_sync<G>();                            // P2 complete; P1 free for the next orientation
    }
    // ---- layer 3: a lane per map m (lanes 25-31 idle), one input channel at a time with its
    //      7 x 8 kernel in registers; a pass walks the 10 response rows (orientation, y), the
    //      P2 rows broadcast to the warp as float4s; channel 0 leaves partial sums in l3; the
    //      group's warps split the response rows ----
    float* l3 = S.l3;                               // [m][kL3S] (P1 is dead by now)
    const int m = lane < 25 ? lane : 24;
#pragma unroll 1
    for (int ch = 0; ch < 2; ++ch) {
        float w[56];
#pragma unroll
        for (int k = 0; k < 56; ++k) w[k] = w3s[m * kW3S + ch * 56 + k];
        const float b = w3s[m * kW3S + 112];
#pragma unroll 1
        for (int oy = wg; oy < 10; oy += G) {
            const int o = oy / 5, y = oy - o * 5;
            float a[5];
#pragma unroll
            for (int xx = 0; xx < 5; ++xx) a[xx] = ch == 0 ? b : l3[m * kL3S + oy * 5 + xx];
#pragma unroll
            for (int ky = 0; ky < 8; ++ky) {
                const float4* rp4 = reinterpret_cast<const float4*>(&S.p2[o][ch][y + ky][0]);
                const float4 q0 = rp4[0], q1 = rp4[1], q2 = rp4[2];
                const float v[11] = {q0.x, q0.y, q0.z, q0.w, q1.x, q1.y, q1.z, q1.w, q2.x, q2.y, q2.z};
#pragma unroll
                for (int kx = 0; kx < 7; ++kx)
#pragma unroll
                    for (int xx = 0; xx < 5; ++xx) a[xx] = fmaf(w[ky * 7 + kx], v[xx + kx], a[xx]);
            }
            if (lane < 25) {
#pragma unroll
                for (int xx = 0; xx < 5; ++xx) l3[m * kL3S + oy * 5 + xx] = ch == 0 ? a[xx] : act(a[xx]);
            }
        }
    }
    group_sync<G>();
    // ---- layer 4 (C1x1 25->1, act): a thread per response cell ----
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const int c = gt + NG * h;
        float rr = W.b4;
        if (c < 2 * kResp) {
#pragma unroll
            for (int mm = 0; mm < 25; ++mm) rr = fmaf(W.w4[mm], l3[mm * kL3S + c], rr);
        }
        r[h] = c < 2 * kResp ? act(rr) : -INFINITY;
    }
    group_sync<G>();                                // l3 / P1 reused by the next survivor
}

__global__ void __launch_bounds__(32 * kWarps, 3) selective_kernel(
    const __grid_constant__ Cnn3W W3, const SelParams sp, const LevelInfo* __restrict__ lvinfo,
    const S1Cand* __restrict__ cands, const uint32_t cand_cap, const float* __restrict__ resp2,
    const uint8_t* __restrict__ epatch, SelOut* __restrict__ out, float* __restrict__ dbg_resp,
    AccBox* __restrict__ acc, Ctrl* __restrict__ ctrl, const uint32_t cta_max)
{
    extern __shared__ __align__(16) unsigned char sraw[];
    const int lane = (int)(threadIdx.x & 31);
    float* w3s = reinterpret_cast<float*>(sraw);                          // [25][kW3S]
    WarpSmem& S = reinterpret_cast<WarpSmem*>(sraw + kW3Bytes)[threadIdx.x >> 5];
    for (int i = threadIdx.x; i < 25 * kW3S; i += blockDim.x) {
        const int mm = i / kW3S, k = i - mm * kW3S;
        w3s[i] = k < 112 ? W3.w3[mm][k / 56][k % 56] : W3.b3[mm];
    }
    __syncthreads();
    const uint32_t n_cand = min(*(volatile uint32_t*)&ctrl->n_cand, cand_cap);
    auto warp_max = [](float v) {
#pragma unroll
        for (int d = 16; d >= 1; d >>= 1) v = fmaxf(v, __shfl_xor_sync(0xFFFFFFFFu, v, d));
        return v;
    };
    // the survivor's outcome (one thread): SelOut, Table-1 counters, the accepted-box list
    auto finish = [&](int ci, int K2, int K3, int delta, int ran3, float best) {
        const S1Cand cd = cands[ci];
        SelOut so;
        so.K2 = K2; so.K3 = K3; so.delta = delta; so.cnn3_ran = ran3; so.score = best;
        sel::raw_box(cd, lvinfo[cd.level].sigma, so);              // O8
        out[ci] = so;
        if (K2 > 0) atomicAdd(&ctrl->n_stage2, 1u);
        if (delta) {
            atomicAdd(&ctrl->n_stage3, 1u);
            const uint32_t k = atomicAdd(&ctrl->n_acc, 1u);
            AccBox b;
            b.frame = cd.frame; b.x = so.bx; b.y = so.by; b.w = so.bw; b.h = so.bh; b.score = best;
            acc[k] = b;                   // n_acc <= n_cand <= cand_cap slots
        }
    };
    if (n_cand <= cta_max) {
        // ---- latency form (few survivors): a whole CTA per survivor ----
        __shared__ int s_ci;
        __shared__ float s_wmax[kWarps];
        WarpSmem& S0 = reinterpret_cast<WarpSmem*>(sraw + kW3Bytes)[0];
        const int tid = (int)threadIdx.x;
        auto block_max = [&](float v) {
            v = warp_max(v);
            if (lane == 0) s_wmax[tid >> 5] = v;
            __syncthreads();
            float m = s_wmax[0];
#pragma unroll
            for (int k = 1; k < kWarps; ++k) m = fmaxf(m, s_wmax[k]);
            __syncthreads();
            return m;
        };
        for (;;) {
            if (tid == 0) s_ci = (int)atomicAdd(&ctrl->sel_next, 1u);
            __syncthreads();
            const int ci = s_ci;
            if ((uint32_t)ci >= n_cand) break;                  // CTA-uniform
            const float r2v = tid < 2 * kResp ? resp2[(int64_t)ci * 50 + tid] : -INFINITY;
            const int K2 = __syncthreads_count(r2v > sp.T2a);
            const bool stop = (sp.rule == 0) ? (K2 == 0) : (K2 >= sp.Tnn);
            int K3 = 0, delta, ran3 = 0;
            float best, r3[2] = {0.f, 0.f};
            if (stop) {
                delta = (sp.rule == 0) ? 0 : 1;
                best = block_max(r2v);
            } else {
                const uint4* src = reinterpret_cast<const uint4*>(epatch + (int64_t)ci * kEPatchBytes);
                uint4* dst = reinterpret_cast<uint4*>(S0.e);
                for (int w = tid; w < kEPatchBytes / 16; w += 32 * kWarps) dst[w] = __ldg(src + w);
                __syncthreads();
                cnn3_group<kWarps>(W3, w3s, S0, tid, r3);          // cells tid (< 50) only
                K3 = __syncthreads_count(r3[0] > sp.T2b);
                ran3 = 1;
                delta = (sp.rule == 0) ? (((K2 >= sp.Tnn) && K3 > 0) || (K2 > 0 && K3 >= sp.Tnn))
                                       : (K2 >= sp.Tnn || K3 >= sp.Tnn);
                best = block_max(r3[0]);
            }
            if (dbg_resp && tid < 2 * kResp) {
                dbg_resp[(int64_t)ci * 100 + tid] = r2v;
                dbg_resp[(int64_t)ci * 100 + 50 + tid] = r3[0];
            }
            if (tid == 0) finish(ci, K2, K3, delta, ran3, best);
            __syncthreads();                                    // s_ci / S0 reused
        }
        return;
    }
    // ---- throughput form: one warp per survivor ----
    for (;;) {
        int ci = 0;
        if (lane == 0) ci = (int)atomicAdd(&ctrl->sel_next, 1u);
        ci = __shfl_sync(0xFFFFFFFFu, ci, 0);
        if ((uint32_t)ci >= n_cand) break;
        // ---- CNN2's responses (selective_tc.cu): lane l holds cells l and l + 32; K2
        const float* rp = resp2 + (int64_t)ci * 50;
        const float r2a = rp[lane];
        const float r2b = lane + 32 < 2 * kResp ? rp[lane + 32] : -INFINITY;
        const int K2 = __popc(__ballot_sync(0xFFFFFFFFu, r2a > sp.T2a)) +
                       __popc(__ballot_sync(0xFFFFFFFFu, r2b > sp.T2a));
        const bool stop = (sp.rule == 0) ? (K2 == 0) : (K2 >= sp.Tnn);   // P:99 / S:358
        int K3 = 0, delta, ran3 = 0;
        float best, r3[2] = {0.f, 0.f};
        if (stop) {
            delta = (sp.rule == 0) ? 0 : 1;
            best = warp_max(fmaxf(r2a, r2b));
        } else {
            // ---- E (selective_tc.cu kept it for every survivor the rule sends here) ----
            const uint4* src = reinterpret_cast<const uint4*>(epatch + (int64_t)ci * kEPatchBytes);
            uint4* dst = reinterpret_cast<uint4*>(S.e);
            for (int w = lane; w < kEPatchBytes / 16; w += 32) dst[w] = __ldg(src + w);
            __syncwarp();
            // ---- CNN3 on both orientations, K3, the rule (P:95 / P:217) ----
            cnn3_group<1>(W3, w3s, S, lane, r3);
            K3 = __popc(__ballot_sync(0xFFFFFFFFu, r3[0] > sp.T2b)) +
                 __popc(__ballot_sync(0xFFFFFFFFu, r3[1] > sp.T2b));
            ran3 = 1;
            delta = (sp.rule == 0) ? (((K2 >= sp.Tnn) && K3 > 0) || (K2 > 0 && K3 >= sp.Tnn))
                                   : (K2 >= sp.Tnn || K3 >= sp.Tnn);
            best = warp_max(fmaxf(r3[0], r3[1]));
            __syncwarp();                           // S.e / S.p2 are reused by the next survivor
        }
        if (dbg_resp) {
            float* d = dbg_resp + (int64_t)ci * 100;
            d[lane] = r2a;
            d[50 + lane] = r3[0];
            if (lane + 32 < 2 * kResp) {
                d[lane + 32] = r2b;
                d[50 + lane + 32] = r3[1];
            }
        }
        if (lane == 0) finish(ci, K2, K3, delta, ran3, best);
    }
}

}  // namespace

void launch_selective(const Cnn3W& w3, SelParams sp, const LevelInfo* d_levels,
                      const S1Cand* cands, uint32_t cand_cap, const float* resp2,
                      const uint8_t* epatch, SelOut* out, float* dbg_resp, AccBox* acc, Ctrl* ctrl,
                      int sm_count, cudaStream_t s)
{
    const size_t smem = kW3Bytes + sizeof(WarpSmem) * kWarps;
    cudaFuncSetAttribute(selective_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, selective_kernel, 32 * kWarps, smem);
    if (occ < 1) occ = 1;
    // a lone warp needs ~40 us for one survivor's CNN3, a CTA ~10 us: below a few survivors
    // per CTA the CTA form finishes first (C4: 700 survivors -> 73 -> ~25 us), above it the
    // warp form's throughput wins (C5: 45k survivors)
    static const long env_max = [] {
        const char* e = std::getenv("CCNN_CNN3_CTA_PER_GRID");     // experiments only
        return e ? std::atol(e) : -1L;
    }();
    const int grid = sm_count * occ;
    const uint32_t cta_max = (uint32_t)(env_max >= 0 ? env_max * grid : 4L * grid);
    selective_kernel<<<grid, 32 * kWarps, smem, s>>>(w3, sp, d_levels, cands, cand_cap, resp2,
                                                     epatch, out, dbg_resp, acc, ctrl, cta_max);
}

}  // namespace ccnn
