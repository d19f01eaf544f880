// selective.cu -- stage 3 of the cascade and the decision rule on every stage-1 survivor
// (K3), after selective_tc.cu has computed CNN2's 50 responses (resp2).
//
// PAPER.md §3.3: K = number of responses exceeding T2; Eq. 2 (strict) with the
// early stop of P:99 -- CNN3 runs only when the rule needs it -- or Eq. 3 (weak).
// Readings O5-O8: the patch (O5 geometry, O2 sampling, O6 equalisation), K pooled
// over both orientations, the raw box.
//
// B200 design: a persistent kernel drains the survivor queue with a dynamic atomic counter.
// One CTA per survivor: K2 from resp2 (block count); when CNN3 is needed the CTA loads the
// equalised patch E selective_tc.cu left for it and runs CNN3 on both orientations on the FFMA
// pipe (2-map layers: no dense contraction for the tensor cores); only E is stored, the
// mirrored orientation M(x,y) = E(50-x,y) is read through mirrored
// addresses; every layer's work is split over data so the weights a warp uses are warp-uniform
// constant-bank kernel parameters.
#include <type_traits>

#include "ccnn_internal.h"
#include "selective_common.cuh"
#include <cuda_fp16.h>

namespace ccnn {
namespace {

constexpr int kSelThreads = 288;            // 9 warps: layer-2 items (264) in one round
constexpr int kEW = 48;                     // words per row of the fp16 patch plane (26 used;
                                            // 48 == 16 mod 32: rows y, y+1 on disjoint banks)
constexpr int kP1RS = 24;                   // pooled L1 row (24 wide): even [0,12), odd [12,24)
constexpr int kP1Odd = 12;

__device__ __forceinline__ float act(float x)      // Eq. 1, see stage1.cu
{
    const float a = fabsf(x) * (2.0f / 3.0f);
    const float a2 = a * a;
    const float p = fmaf(a2, fmaf(a2, 1.41645f, 1.0f), a + 1.0f);
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(p));
    return copysignf(fmaf(-1.7159f, r, 1.7159f), x);
}

struct SelSmem {
    uint32_t eh[kPatchH][kEW];              // E as raw fp16 pixel pairs: word j = pixels (2j, 2j+1),
                                            // pixel 51 = 0 (exact: equalised values <= 255)
    float p2[2][6][12][12];                 // pooled layer 2 [orient][map][y][x]
    float l3[25][2][25];                    // layer-3 activations [map][orient][cell]
    float w3s[25][3][56];                   // layer-3 weights [map][in][ky*7+kx]; [map][2][0] = bias
    float resp[2][kResp];
    float wmax[kSelThreads / 32];
    int cand;
};
// one P1 map plane: 26 rows + 4 floats of padding, so the planes of maps 2c and 2c+2 (the
// 4 lane groups of a layer-1 MMA epilogue store) start 8 banks apart: conflict-free stores
constexpr int kP1MS = 26 * kP1RS + 4;
constexpr size_t kP1Floats = 2 * 2 * kP1MS;    // pooled layer 1 of CNN3: [orient][map][y][row]

// E(x, y) normalised (O3), for the FFMA layer 1 of CNN3
__device__ __forceinline__ float img_at(const SelSmem& sm, int y, int x)
{
    const __half h = reinterpret_cast<const __half*>(&sm.eh[y][0])[x];
    return fmaf(__half2float(h), 1.0f / 127.5f, -1.0f);
}

// CNN3 (architecture R: C4x4 1->2, P, C3x3 2->2, P, C7x8 2->25, C1x1 25->1, Eq. 1 after every
// conv) on both orientations: 51x55 -> 2 x 5x5 responses in sm.resp.  Work items are register
// blocked (layer 1: 6 pooled columns per thread, layer 3: one 5-cell response row per thread)
// so the shared-memory loads per FMA stay low; layer 3's weights are in shared memory (w3s).
__device__ void run_cnn3(const Cnn3W& W, SelSmem& sm, float* p1)
{
    const int tid = threadIdx.x;
    // ---- layer 1: conv4x4 1->2, pool, act; item = (orientation, pooled row, 6 pooled columns)
    for (int it = tid; it < 2 * 26 * 4; it += kSelThreads) {
        const int o = it / 104, rem = it - o * 104, py0 = rem >> 2, g = rem & 3;
        float x[5][15];                             // image rows 2py0 .. +4, columns 12g .. +14
#pragma unroll
        for (int r = 0; r < 5; ++r)
#pragma unroll
            for (int c = 0; c < 15; ++c)            // M(x, y) = E(50 - x, y); column 51+ unused
                x[r][c] = img_at(sm, 2 * py0 + r, o == 0 ? min(12 * g + c, 50) : max(50 - 12 * g - c, 0));
#pragma unroll
        for (int j = 0; j < 6; ++j) {               // pooled column px0 = 6g + j
            const int px0 = 6 * g + j;
            const int col = (px0 & 1) ? kP1Odd + (px0 >> 1) : (px0 >> 1);
#pragma unroll
            for (int a = 0; a < 2; ++a) {
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
                p1[(o * 2 + a) * kP1MS + py0 * kP1RS + col] =
                    act(fmaxf(fmaxf(sv[0], sv[1]), fmaxf(sv[2], sv[3])));   // pool then act
            }
        }
    }
    __syncthreads();
    // ---- layer 2: conv3x3 2->2, pool, act; item = (orientation, pooled position) ----
    if (tid < 2 * 132) {
        const int o2 = tid / 132, pos2 = tid - o2 * 132, py2 = pos2 / 11, px2 = pos2 - py2 * 11;
        float s2[2][4];
#pragma unroll
        for (int b = 0; b < 2; ++b)
#pragma unroll
            for (int k = 0; k < 4; ++k) s2[b][k] = W.b2[b];
#pragma unroll
        for (int a = 0; a < 2; ++a) {
            const float* in = p1 + (o2 * 2 + a) * kP1MS + 2 * py2 * kP1RS;
            float v[4][4];
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                v[r][0] = in[r * kP1RS + px2];
                v[r][1] = in[r * kP1RS + kP1Odd + px2];
                v[r][2] = in[r * kP1RS + px2 + 1];
                v[r][3] = in[r * kP1RS + kP1Odd + px2 + 1];
            }
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
            sm.p2[o2][b][py2][px2] = act(fmaxf(fmaxf(s2[b][0], s2[b][1]), fmaxf(s2[b][2], s2[b][3])));
    }
    __syncthreads();
    // ---- layer 3: conv7x8 2->25, act; item = (map, orientation, response row): 250 items ----
    if (tid < 250) {
        const int m = tid / 10, o = (tid / 5) & 1, y = tid % 5;
        float acc[5];
#pragma unroll
        for (int xx = 0; xx < 5; ++xx) acc[xx] = sm.w3s[m][2][0];   // bias
#pragma unroll 1
        for (int ch = 0; ch < 2; ++ch) {
#pragma unroll 2
            for (int ky = 0; ky < 8; ++ky) {
                const float* row = &sm.p2[o][ch][y + ky][0];
                float v[11];
#pragma unroll
                for (int c = 0; c < 11; ++c) v[c] = row[c];
                const float* wr = &sm.w3s[m][ch][ky * 7];
#pragma unroll
                for (int kx = 0; kx < 7; ++kx) {
                    const float w = wr[kx];
#pragma unroll
                    for (int xx = 0; xx < 5; ++xx) acc[xx] = fmaf(w, v[xx + kx], acc[xx]);
                }
            }
        }
#pragma unroll
        for (int xx = 0; xx < 5; ++xx) sm.l3[m][o][y * 5 + xx] = act(acc[xx]);
    }
    __syncthreads();
    // ---- layer 4: C1x1 25->1, act ----
    if (tid < 2 * kResp) {
        const int o = tid / kResp, cell = tid - o * kResp;
        float r = W.b4;
#pragma unroll
        for (int c = 0; c < 25; ++c) r = fmaf(W.w4[c], sm.l3[c][o][cell], r);
        sm.resp[o][cell] = act(r);
    }
    __syncthreads();
}

__global__ void __launch_bounds__(kSelThreads, 3) selective_kernel(
    const __grid_constant__ Cnn3W W3, const SelParams sp, const LevelInfo* __restrict__ lvinfo,
    const S1Cand* __restrict__ cands, const uint32_t cand_cap, const float* __restrict__ resp2,
    const uint8_t* __restrict__ epatch, SelOut* __restrict__ out, float* __restrict__ dbg_resp,
    AccBox* __restrict__ acc, Ctrl* __restrict__ ctrl)
{
    extern __shared__ __align__(16) unsigned char sraw[];
    SelSmem& sm = *reinterpret_cast<SelSmem*>(sraw);
    float* const p1 = reinterpret_cast<float*>(sraw + ((sizeof(SelSmem) + 15) & ~size_t(15)));
    const int tid = threadIdx.x;
    const uint32_t n_cand = min(*(volatile uint32_t*)&ctrl->n_cand, cand_cap);
    // block max of the responses of the last net evaluated (threads < 50 hold them)
    auto block_max = [&](float v) {
        float m = (tid < 2 * kResp) ? v : -INFINITY;
#pragma unroll
        for (int d = 16; d >= 1; d >>= 1) m = fmaxf(m, __shfl_xor_sync(0xFFFFFFFFu, m, d));
        if ((tid & 31) == 0) sm.wmax[tid >> 5] = m;
        __syncthreads();
        float r = sm.wmax[0];
#pragma unroll
        for (int k = 1; k < kSelThreads / 32; ++k) r = fmaxf(r, sm.wmax[k]);
        __syncthreads();
        return r;
    };

    for (int i = tid; i < 25 * 3 * 56; i += kSelThreads) {
        const int m = i / 168, r = i - m * 168, ch = r / 56, k = r - ch * 56;
        sm.w3s[m][ch][k] = ch < 2 ? W3.w3[m][ch][k] : (k == 0 ? W3.b3[m] : 0.f);
    }
    for (;;) {
        if (tid == 0) sm.cand = (int)atomicAdd(&ctrl->sel_next, 1u);
        __syncthreads();
        const int ci = sm.cand;
        if ((uint32_t)ci >= n_cand) break;
        const S1Cand cd = cands[ci];
        const double sigma = lvinfo[cd.level].sigma;

        // ---- CNN2's responses (selective_tc.cu), K2 ----
        const float r2v = (tid < 2 * kResp) ? resp2[(int64_t)ci * 50 + tid] : 0.f;
        const int K2 = __syncthreads_count(tid < 2 * kResp && r2v > sp.T2a);
        const bool stop = (sp.rule == 0) ? (K2 == 0) : (K2 >= sp.Tnn);   // P:99 / S:358
        int K3 = 0, delta, ran3 = 0;
        float best, r3v = 0.f;
        if (stop) {
            delta = (sp.rule == 0) ? 0 : 1;
            best = block_max(r2v);
        } else {
            // ---- the equalised patch E (selective_tc.cu wrote it for every survivor the rule
            //      sends here) as fp16 pixel pairs (raw values; O3 is applied by the layers) ----
            const uint8_t* ep = epatch + (int64_t)ci * kEPatchBytes;
            for (int k = tid; k < kPatchH * 26; k += kSelThreads) {
                const int v = k / 26, j = k - v * 26;
                const uint32_t p0 = __ldg(ep + v * kPatchW + 2 * j);
                const uint32_t p1v = (2 * j + 1 < kPatchW) ? __ldg(ep + v * kPatchW + 2 * j + 1) : 0u;
                const __half2 h = __floats2half2_rn((float)p0, (float)p1v);
                sm.eh[v][j] = *reinterpret_cast<const uint32_t*>(&h);
            }
            __syncthreads();
            // ---- CNN3 on both orientations, K3, the rule (P:95 / P:217) ----
            run_cnn3(W3, sm, p1);
            if (tid < 2 * kResp) r3v = sm.resp[tid / kResp][tid % kResp];
            K3 = __syncthreads_count(tid < 2 * kResp && r3v > sp.T2b);
            ran3 = 1;
            delta = (sp.rule == 0) ? (((K2 >= sp.Tnn) && K3 > 0) || (K2 > 0 && K3 >= sp.Tnn))
                                   : (K2 >= sp.Tnn || K3 >= sp.Tnn);
            best = block_max(r3v);
        }
        if (dbg_resp && tid < 2 * kResp) {
            dbg_resp[(int64_t)ci * 100 + tid] = r2v;
            dbg_resp[(int64_t)ci * 100 + 50 + tid] = r3v;
        }
        if (tid == 0) {
            SelOut so;
            so.K2 = K2; so.K3 = K3; so.delta = delta; so.cnn3_ran = ran3; so.score = best;
            sel::raw_box(cd, sigma, so);              // O8
            out[ci] = so;
            if (K2 > 0) atomicAdd(&ctrl->n_stage2, 1u);
            if (delta) {
                atomicAdd(&ctrl->n_stage3, 1u);
                const uint32_t k = atomicAdd(&ctrl->n_acc, 1u);
                AccBox b;
                b.frame = cd.frame; b.x = so.bx; b.y = so.by; b.w = so.bw; b.h = so.bh; b.score = best;
                acc[k] = b;               // n_acc <= n_cand <= cand_cap slots
            }
        }
        __syncthreads();
    }
}

}  // namespace

size_t selective_smem_bytes()
{
    return ((sizeof(SelSmem) + 15) & ~size_t(15)) + sizeof(float) * kP1Floats;
}

void launch_selective(const Cnn3W& w3, SelParams sp, const LevelInfo* d_levels,
                      const S1Cand* cands, uint32_t cand_cap, const float* resp2,
                      const uint8_t* epatch, SelOut* out, float* dbg_resp, AccBox* acc, Ctrl* ctrl,
                      int sm_count, cudaStream_t s)
{
    const size_t smem = selective_smem_bytes();
    cudaFuncSetAttribute(selective_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, selective_kernel, kSelThreads, smem);
    if (occ < 1) occ = 1;
    selective_kernel<<<sm_count * occ, kSelThreads, smem, s>>>(w3, sp, d_levels, cands, cand_cap, resp2,
                                                              epatch, out, dbg_resp, acc, ctrl);
}

}  // namespace ccnn
