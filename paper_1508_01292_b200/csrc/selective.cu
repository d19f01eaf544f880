// selective.cu -- stage 3 of the cascade and the decision rule on every stage-1 survivor
// (K3), after selective_tc.cu has computed CNN2's 50 responses (resp2).
//
// PAPER.md §3.3: K = number of responses exceeding T2; Eq. 2 (strict) with the
// early stop of P:99 -- CNN3 runs only when the rule needs it -- or Eq. 3 (weak).
// Readings O5-O8: the patch (O5 geometry, O2 sampling, O6 equalisation), K pooled
// over both orientations, the raw box.
//
// B200 design: a persistent kernel drains the survivor queue with a dynamic atomic counter.
// One CTA per survivor: K2 from resp2 (block count); when CNN3 is needed the CTA rebuilds the
// equalised patch E (selective_common.cuh, bit-identical to selective_tc.cu's) and runs CNN3 on
// both orientations on the FFMA pipe (2-map layers: no dense contraction for the tensor
// cores); only E is stored, the mirrored orientation M(x,y) = E(50-x,y) is read through mirrored
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
    uint32_t colx[kPatchW], rowy[kPatchH];
    int hist[256];
    uint8_t lut[256];
    uint8_t patch[kPatchN + 3];
    uint32_t eh[kPatchH][kEW];              // E as raw fp16 pixel pairs: word j = pixels (2j, 2j+1),
                                            // pixel 51 = 0 (exact: equalised values <= 255)
    float p2[2][6][12][12];                 // pooled layer 2 [orient][map][y][x]
    float l3[25][2][25];                    // layer-3 activations [map][orient][cell]
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

// One selective CNN (architecture R: C4x4 1->A, P, C3x3 A->B, P, C7x8 B->C, C1x1 C->1,
// Eq. 1 after every conv) on both orientations: 51x55 -> 2 x 5x5 responses in sm.resp.
template <int A, int B, int C>
__device__ void run_net(const SelNetW<A, B, C>& W, SelSmem& sm, float* p1)
{
    const int tid = threadIdx.x;
    // layers 1-2 in chunks of AC input maps: P1 holds one chunk (both orientations), layer 2
    // accumulates over the chunks in registers
    constexpr int AC = A;
    constexpr int NCH = A / AC;
    const bool l2_item = tid < 2 * 132;
    const int o2 = tid / 132, pos2 = tid - o2 * 132, py2 = pos2 / 11, px2 = pos2 - py2 * 11;
    static_assert(B % 2 == 0, "layer 2 runs on map pairs");
    float2 s2[B / 2][4];                           // (map 2 bp, map 2 bp + 1) x pool position
#pragma unroll
    for (int bp = 0; bp < B / 2; ++bp)
#pragma unroll
        for (int k = 0; k < 4; ++k) s2[bp][k] = make_float2(W.b2[2 * bp], W.b2[2 * bp + 1]);
#pragma unroll 1
    for (int ch = 0; ch < NCH; ++ch) {
    // ---- layer 1: conv4x4 1->A, pool, act; item = (orientation, pooled pos), all A maps ----
    for (int it = tid; it < 1248; it += kSelThreads) {
        // a warp's lanes span two pooled rows (2 image rows apart); the mirrored orientation
        // walks its row backwards so its image words also increase with the lane
        const int o = it / 624, rem = it - o * 624, py0 = rem / 24;
        const int px0 = (o == 0) ? rem - py0 * 24 : 23 - (rem - py0 * 24);
        float x[5][5];
        if (o == 0) {
#pragma unroll
            for (int r = 0; r < 5; ++r)
#pragma unroll
                for (int c = 0; c < 5; ++c) x[r][c] = img_at(sm, 2 * py0 + r, 2 * px0 + c);
        } else {                                    // M(x, y) = E(50 - x, y)
#pragma unroll
            for (int r = 0; r < 5; ++r)
#pragma unroll
                for (int c = 0; c < 5; ++c) x[r][c] = img_at(sm, 2 * py0 + r, 50 - 2 * px0 - c);
        }
#pragma unroll
        for (int a = 0; a < A; ++a) {
            float sv[4];
#pragma unroll
            for (int p = 0; p < 4; ++p) {
                sv[p] = W.b1[a];
#pragma unroll
                for (int ky = 0; ky < 4; ++ky)
#pragma unroll
                    for (int kx = 0; kx < 4; ++kx)
                        sv[p] = fmaf(W.w1[a][ky * 4 + kx], x[(p >> 1) + ky][(p & 1) + kx], sv[p]);
            }
            const int col = (px0 & 1) ? kP1Odd + (px0 >> 1) : (px0 >> 1);
            p1[(o * AC + a) * kP1MS + py0 * kP1RS + col] =
                act(fmaxf(fmaxf(sv[0], sv[1]), fmaxf(sv[2], sv[3])));   // pool then act
        }
    }
    __syncthreads();
    // ---- layer 2 (partial over this chunk's maps): conv3x3 A->B; item = (orientation,
    //      pooled position), all output maps ----
    if (l2_item) {
#pragma unroll 1
        for (int a = 0; a < AC; ++a) {              // uniform counter: LDCU [UR+imm]
            const float* in = p1 + (o2 * AC + a) * kP1MS + 2 * py2 * kP1RS;
            float v[4][4];
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                v[r][0] = in[r * kP1RS + px2];
                v[r][1] = in[r * kP1RS + kP1Odd + px2];
                v[r][2] = in[r * kP1RS + px2 + 1];
                v[r][3] = in[r * kP1RS + kP1Odd + px2 + 1];
            }
            constexpr int NV = SelNetW<A, B, C>::W2V;
            float wv[NV];
            const float4* w4p = reinterpret_cast<const float4*>(W.w2v[ch * AC + a]);
#pragma unroll
            for (int k4 = 0; k4 < NV / 4; ++k4) {
                const float4 t4 = w4p[k4];
                wv[4 * k4] = t4.x; wv[4 * k4 + 1] = t4.y; wv[4 * k4 + 2] = t4.z; wv[4 * k4 + 3] = t4.w;
            }
#pragma unroll
            for (int bp = 0; bp < B / 2; ++bp)
#pragma unroll
                for (int ky = 0; ky < 3; ++ky)
#pragma unroll
                    for (int kx = 0; kx < 3; ++kx) {
                        const float2 w = make_float2(wv[(ky * 3 + kx) * B + 2 * bp], wv[(ky * 3 + kx) * B + 2 * bp + 1]);
#pragma unroll
                        for (int k = 0; k < 4; ++k) {
                            const float x = v[(k >> 1) + ky][(k & 1) + kx];
                            s2[bp][k] = __ffma2_rn(w, make_float2(x, x), s2[bp][k]);
                        }
                    }
        }
    }
    if (ch + 1 < NCH) __syncthreads();             // the next chunk overwrites P1
    }
    if (l2_item) {
#pragma unroll
        for (int bp = 0; bp < B / 2; ++bp) {
            sm.p2[o2][2 * bp][py2][px2] =
                act(fmaxf(fmaxf(s2[bp][0].x, s2[bp][1].x), fmaxf(s2[bp][2].x, s2[bp][3].x)));
            sm.p2[o2][2 * bp + 1][py2][px2] =
                act(fmaxf(fmaxf(s2[bp][0].y, s2[bp][1].y), fmaxf(s2[bp][2].y, s2[bp][3].y)));
        }
    }
    __syncthreads();
    // ---- layer 3: conv7x8 B->C, act; item = (map, orientation, cell) ----
    if constexpr (C == 2) {
        if (tid < 128) {                            // map = warp pair -> warp-uniform weights
            const int m = tid >> 6, idx = tid & 63;
            if (idx < 50) {
                const int o = idx / 25, cell = idx - o * 25, y = cell / 5, x = cell - y * 5;
                auto body = [&](auto Mc) {
                    constexpr int M = decltype(Mc)::value;
                    float s = W.b3[M];
#pragma unroll
                    for (int b = 0; b < B; ++b)
#pragma unroll
                        for (int ky = 0; ky < 8; ++ky)
#pragma unroll
                            for (int kx = 0; kx < 7; ++kx)
                                s = fmaf(W.w3[M][b][ky * 7 + kx], sm.p2[o][b][y + ky][x + kx], s);
                    sm.l3[M][o][cell] = act(s);
                };
                if (m == 0) body(std::integral_constant<int, 0>{});
                else body(std::integral_constant<int, 1>{});
            }
        }
    } else {
        // map-major items padded to 64 per map: every warp works on one map, so its weight
        // loads are one broadcast address (no serialised constant-cache accesses)
        for (int it = tid; it < C * 64; it += kSelThreads) {
            const int m = it >> 6, idx = it & 63;
            if (idx >= 50) continue;
            const int o = idx / 25, cell = idx - o * 25, y = cell / 5, x = cell - y * 5;
            float s = W.b3[m];
#pragma unroll
            for (int b = 0; b < B; ++b)
#pragma unroll
                for (int ky = 0; ky < 8; ++ky)
#pragma unroll
                    for (int kx = 0; kx < 7; ++kx)
                        s = fmaf(W.w3[m][b][ky * 7 + kx], sm.p2[o][b][y + ky][x + kx], s);
            sm.l3[m][o][cell] = act(s);
        }
    }
    __syncthreads();
    // ---- layer 4: C1x1 C->1, act ----
    if (tid < 2 * kResp) {
        const int o = tid / kResp, cell = tid - o * kResp;
        float r = W.b4;
#pragma unroll
        for (int c = 0; c < C; ++c) r = fmaf(W.w4[c], sm.l3[c][o][cell], r);
        sm.resp[o][cell] = act(r);
    }
    __syncthreads();
}

__global__ void __launch_bounds__(kSelThreads, 3) selective_kernel(
    const __grid_constant__ Cnn3W W3, const SelParams sp, const FrameInfo* __restrict__ frames,
    const LevelInfo* __restrict__ lvinfo, const S1Cand* __restrict__ cands, const uint32_t cand_cap,
    const float* __restrict__ resp2, SelOut* __restrict__ out, float* __restrict__ dbg_resp,
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
            const FrameInfo F = frames[lvinfo[cd.level].frame];
            // ---- the equalised patch E (O5, O2, O6; selective_common.cuh) ----
            if (tid < kPatchW) sm.colx[tid] = sel::patch_col(cd.ix, sigma, tid, F.w);
            else if (tid < kPatchW + kPatchH) sm.rowy[tid - kPatchW] = sel::patch_row(cd.iy, sigma, tid - kPatchW, F.h);
            if (tid < 256) sm.hist[tid] = 0;
            __syncthreads();
            for (int k0 = tid; k0 < kPatchN; k0 += 4 * kSelThreads) {
                uint32_t val[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int k = min(k0 + u * kSelThreads, kPatchN - 1);
                    const int v = k / kPatchW, uu = k - v * kPatchW;
                    val[u] = sel::sample(F.data, F.pitch, F.w, F.h, sm.colx[uu], sm.rowy[v]);
                }
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int k = k0 + u * kSelThreads;
                    if (k >= kPatchN) break;
                    sm.patch[k] = (uint8_t)val[u];
                    atomicAdd(&sm.hist[val[u]], 1);
                }
            }
            __syncthreads();
            if (tid < 32) sel::warp_lut(sm.hist, sm.lut);
            __syncthreads();
            // E as fp16 pixel pairs (raw equalised values; O3 is applied by the layers)
            for (int k = tid; k < kPatchH * 26; k += kSelThreads) {
                const int v = k / 26, j = k - v * 26;
                const uint32_t p0 = sm.lut[sm.patch[v * kPatchW + 2 * j]];
                const uint32_t p1v = (2 * j + 1 < kPatchW) ? sm.lut[sm.patch[v * kPatchW + 2 * j + 1]] : 0u;
                const __half2 h = __floats2half2_rn((float)p0, (float)p1v);
                sm.eh[v][j] = *reinterpret_cast<const uint32_t*>(&h);
            }
            __syncthreads();
            // ---- CNN3 on both orientations, K3, the rule (P:95 / P:217) ----
            run_net<2, 2, 25>(W3, sm, p1);
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

void launch_selective(const Cnn3W& w3, SelParams sp, const FrameInfo* d_frames,
                      const LevelInfo* d_levels, const S1Cand* cands, uint32_t cand_cap,
                      const float* resp2, SelOut* out, float* dbg_resp, AccBox* acc, Ctrl* ctrl,
                      int sm_count, cudaStream_t s)
{
    const size_t smem = selective_smem_bytes();
    cudaFuncSetAttribute(selective_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, selective_kernel, kSelThreads, smem);
    if (occ < 1) occ = 1;
    selective_kernel<<<sm_count * occ, kSelThreads, smem, s>>>(w3, sp, d_frames, d_levels, cands, cand_cap,
                                                              resp2, out, dbg_resp, acc, ctrl);
}

}  // namespace ccnn
