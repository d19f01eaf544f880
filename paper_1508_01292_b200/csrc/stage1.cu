// stage1.cu -- fused stage-1 CNN1 dense scan + threshold + compaction (K2).
//
// PAPER.md §3.3: "The first CNN densely scans in series each image of the
// pyramid.  The responses in the output network layer correspond to the positions of
// the scanning window with a size of 27x31 pixels during its uniform motion with a 4
// pixel step.  The coordinates of the windows, where the CNN response exceeded the
// predetermined threshold T1, are transmitted to the selective unit".  CNN1 is
// architecture R (R1): C4x4 1->6, pool, C3x3 6->6, pool, C5x6 6->2, C1x1 2->1,
// Eq. 1 activation after every conv, fp32.
//
// B200 design (not the paper's Kepler texture kernels):
//  * one persistent kernel over a flattened (frame, level, band, row-segment) task table,
//    longest tasks first, dynamic atomic task counter -> no per-level launches;
//  * a CTA owns a band of TW = NT/2-5 windows and marches down its rows with a
//    line-buffer pipeline in shared memory: input ring (fp32, even/odd de-interleaved
//    columns so every LDS is bank-conflict free), pooled-layer-1 ring, pooled-layer-2
//    ring; only ONE __syncthreads per window row, each phase reads rows written in
//    earlier steps; no vertical halo recompute inside a task;
//  * every MAC is an FFMA whose weight operand is a constant-bank kernel parameter
//    (fully unrolled, compile-time indices) -> two register operands per FFMA;
//  * max-pool BEFORE the activation (Eq. 1 is monotone: act(max) == max(act), 4x fewer
//    activations); layer 3 streams its 6 kernel rows through register accumulators;
//  * threshold + warp ballot/popc + ONE atomicAdd per warp into the survivor queue.
#include "ccnn_internal.h"

namespace ccnn {
namespace {

// Eq. 1: 1.7159 * sgn(y) * (1 - 1/(1 + |y| + y^2 + 1.41645 y^4)), y = 2x/3.
// (a+1) + a^2 (1 + k a^2) with a = |y|; MUFU reciprocal (|rel err| ~ 2^-23).
__device__ __forceinline__ float act(float x)
{
    const float a = fabsf(x) * (2.0f / 3.0f);
    const float a2 = a * a;
    const float p = fmaf(a2, fmaf(a2, 1.41645f, 1.0f), a + 1.0f);
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(p));
    return copysignf(fmaf(-1.7159f, r, 1.7159f), x);
}

template <int NT>
struct Cfg {
    static constexpr int TW = NT / 2 - 5;        // windows per band
    static constexpr int P2C = NT / 2 - 1;       // pooled layer-2 columns = TW + 4
    static constexpr int IN_WORDS = NT / 2 + 1;  // 32-bit words per input row (>= 2NT+3 B)
    static constexpr int IN_ODD = NT + 4;        // odd columns start inside an input row
    static constexpr int IN_RS = 2 * NT + 8;     // input ring row stride (floats)
    static constexpr int IN_RING = 12;
    static constexpr int P1_ODD = NT / 2 + 16;   // odd P1 columns start (bank offset 16)
    static constexpr int P1_RS = NT + 16;        // one (row, map) of the P1 ring
    static constexpr int P1_RING = 6;
    static constexpr int P2_RS = NT / 2 + 8;
    static constexpr int P2_RING = 2;
    static constexpr int SMEM_FLOATS = IN_RING * IN_RS + P1_RING * 6 * P1_RS + P2_RING * 6 * P2_RS;
    static constexpr int LOAD_SLOTS = (4 * IN_WORDS + NT - 1) / NT;
};

__device__ __forceinline__ float u8f(uint32_t v)
{
    return fmaf((float)v, 1.0f / 127.5f, -1.0f);   // O3: (v - 127.5) / 127.5
}

template <int NT>
__device__ __forceinline__ void store_word(float* ring, int slot, int w, uint32_t word)
{
    using C = Cfg<NT>;
    float* row = ring + slot * C::IN_RS;
    float2 ev = make_float2(u8f(word & 0xFFu), u8f((word >> 16) & 0xFFu));
    float2 od = make_float2(u8f((word >> 8) & 0xFFu), u8f(word >> 24));
    *reinterpret_cast<float2*>(row + 2 * w) = ev;
    *reinterpret_cast<float2*>(row + C::IN_ODD + 2 * w) = od;
}

template <int NT, bool DEBUG>
__global__ void __launch_bounds__(NT, 512 / NT) stage1_kernel(
    const __grid_constant__ Cnn1W W, const float T1,
    const uint8_t* __restrict__ levels, const int64_t level_frame_stride,
    const LevelInfo* __restrict__ lvinfo, const S1Task* __restrict__ tasks, const int n_tasks,
    S1Cand* __restrict__ cands, const uint32_t cand_cap, Ctrl* __restrict__ ctrl,
    float* __restrict__ dbg_map, const int64_t dbg_map_frame_stride)
{
    using C = Cfg<NT>;
    extern __shared__ __align__(16) float smem[];
    float* const in_ring = smem;
    float* const p1_ring = in_ring + C::IN_RING * C::IN_RS;
    float* const p2_ring = p1_ring + C::P1_RING * 6 * C::P1_RS;
    __shared__ int s_task;

    const int tid = threadIdx.x;
    const int lane = tid & 31;
    const int half = tid / (NT / 2);           // 0: L2 maps 0-1 + L3; 1: L2 maps 2-5
    const int q = tid & (NT / 2 - 1);          // P2 column (L2) / window column (L3)

    // loader slots: word k -> (row k / IN_WORDS, word k % IN_WORDS) of a 4-row group
    int ld_row[C::LOAD_SLOTS], ld_w[C::LOAD_SLOTS];
    bool ld_ok[C::LOAD_SLOTS];
#pragma unroll
    for (int k = 0; k < C::LOAD_SLOTS; ++k) {
        const int g = tid + k * NT;
        ld_ok[k] = g < 4 * C::IN_WORDS;
        ld_row[k] = g / C::IN_WORDS;
        ld_w[k] = g % C::IN_WORDS;
    }

    for (;;) {
        if (tid == 0) s_task = (int)atomicAdd(&ctrl->task_next, 1u);
        __syncthreads();
        const int ti = s_task;
        if (ti >= n_tasks) break;
        const S1Task T = tasks[ti];
        const LevelInfo L = lvinfo[T.level];
        const int nrows = T.nrows;
        const uint8_t* const band = levels + (int64_t)T.frame * level_frame_stride + L.offset +
                                    (int64_t)(4 * T.x0);
        const int row_base = 4 * T.y0;                 // first level row of the task
        const int wmax = (L.pitch - 4 * T.x0) / 4 - 1; // last readable word in a row
        auto gword = [&](int r, int w) -> uint32_t {
            const int lr = min(row_base + r, L.lh - 1);
            const int ww = min(w, wmax);
            return __ldg(reinterpret_cast<const uint32_t*>(band + (int64_t)lr * L.pitch) + ww);
        };

        // prologue: rows 0..6 straight to the ring, rows 7..10 into registers
        for (int g = tid; g < 7 * C::IN_WORDS; g += NT)
            store_word<NT>(in_ring, g / C::IN_WORDS, g % C::IN_WORDS,
                           gword(g / C::IN_WORDS, g % C::IN_WORDS));
        uint32_t pre[C::LOAD_SLOTS];
#pragma unroll
        for (int k = 0; k < C::LOAD_SLOTS; ++k)
            pre[k] = ld_ok[k] ? gword(7 + ld_row[k], ld_w[k]) : 0u;

        float acc3[2][6];
#pragma unroll
        for (int m = 0; m < 2; ++m)
#pragma unroll
            for (int i = 0; i < 6; ++i) acc3[m][i] = 0.f;
        __syncthreads();

        const int nsteps = nrows + 8;
        for (int s = 0; s < nsteps; ++s) {
            // ---- loader: commit rows 4s+7..4s+10, prefetch rows 4s+11..4s+14 ----
#pragma unroll
            for (int k = 0; k < C::LOAD_SLOTS; ++k)
                if (ld_ok[k]) store_word<NT>(in_ring, (4 * s + 7 + ld_row[k]) % C::IN_RING, ld_w[k], pre[k]);
#pragma unroll
            for (int k = 0; k < C::LOAD_SLOTS; ++k)
                pre[k] = ld_ok[k] ? gword(4 * s + 11 + ld_row[k], ld_w[k]) : 0u;

            // ---- L1: conv4x4 1->6 + pool + act -> P1 rows 2s, 2s+1 (input rows 4s..4s+6) ----
            if (s <= nrows + 5) {
                const int c = tid;                    // P1 column
                float x[7][5];
                const int s4 = (4 * s) % C::IN_RING;
#pragma unroll
                for (int rr = 0; rr < 7; ++rr) {
                    int slot = s4 + rr;
                    slot = slot >= C::IN_RING ? slot - C::IN_RING : slot;
                    const float* row = in_ring + slot * C::IN_RS;
                    x[rr][0] = row[c];
                    x[rr][1] = row[C::IN_ODD + c];
                    x[rr][2] = row[c + 1];
                    x[rr][3] = row[C::IN_ODD + c + 1];
                    x[rr][4] = row[c + 2];
                }
                const int pcol = (c & 1) ? C::P1_ODD + (c >> 1) : (c >> 1);
#pragma unroll
                for (int r = 0; r < 2; ++r) {
                    float mx[6];
#pragma unroll
                    for (int o = 0; o < 6; ++o) mx[o] = -INFINITY;
#pragma unroll
                    for (int py = 0; py < 2; ++py)
#pragma unroll
                        for (int px = 0; px < 2; ++px) {
                            float a[6];
#pragma unroll
                            for (int o = 0; o < 6; ++o) a[o] = W.b1[o];
#pragma unroll
                            for (int ky = 0; ky < 4; ++ky)
#pragma unroll
                                for (int kx = 0; kx < 4; ++kx) {
                                    const float v = x[2 * r + py + ky][px + kx];
#pragma unroll
                                    for (int o = 0; o < 6; ++o) a[o] = fmaf(W.w1[o][ky * 4 + kx], v, a[o]);
                                }
#pragma unroll
                            for (int o = 0; o < 6; ++o) mx[o] = fmaxf(mx[o], a[o]);
                        }
                    const int slot = (2 * s + r) % C::P1_RING;
#pragma unroll
                    for (int o = 0; o < 6; ++o)
                        p1_ring[(slot * 6 + o) * C::P1_RS + pcol] = act(mx[o]);
                }
            }

            // ---- L2: conv3x3 6->6 + pool + act -> P2 row s-2 (P1 rows 2s-4..2s-1) ----
            if (s >= 2 && s <= nrows + 6) {
                const int pslot = (s - 2) & 1;
                int rs[4];
#pragma unroll
                for (int rr = 0; rr < 4; ++rr) rs[rr] = (2 * s - 4 + rr) % C::P1_RING;
                auto l2 = [&](auto M0c, auto NMc) {
                    constexpr int M0 = decltype(M0c)::value, NM = decltype(NMc)::value;
                    float a[NM][4];
#pragma unroll
                    for (int o = 0; o < NM; ++o)
#pragma unroll
                        for (int k = 0; k < 4; ++k) a[o][k] = W.b2[M0 + o];
#pragma unroll
                    for (int ci = 0; ci < 6; ++ci) {
                        float v[4][4];
#pragma unroll
                        for (int rr = 0; rr < 4; ++rr) {
                            const float* row = p1_ring + (rs[rr] * 6 + ci) * C::P1_RS;
                            v[rr][0] = row[q];
                            v[rr][1] = row[C::P1_ODD + q];
                            v[rr][2] = row[q + 1];
                            v[rr][3] = row[C::P1_ODD + q + 1];
                        }
#pragma unroll
                        for (int o = 0; o < NM; ++o)
#pragma unroll
                            for (int py = 0; py < 2; ++py)
#pragma unroll
                                for (int px = 0; px < 2; ++px)
#pragma unroll
                                    for (int ky = 0; ky < 3; ++ky)
#pragma unroll
                                        for (int kx = 0; kx < 3; ++kx)
                                            a[o][py * 2 + px] = fmaf(W.w2[M0 + o][ci][ky * 3 + kx],
                                                                     v[py + ky][px + kx], a[o][py * 2 + px]);
                    }
#pragma unroll
                    for (int o = 0; o < NM; ++o) {
                        const float m = fmaxf(fmaxf(a[o][0], a[o][1]), fmaxf(a[o][2], a[o][3]));
                        p2_ring[(pslot * 6 + M0 + o) * C::P2_RS + q] = act(m);
                    }
                };
                if (half == 0) l2(std::integral_constant<int, 0>{}, std::integral_constant<int, 2>{});
                else           l2(std::integral_constant<int, 2>{}, std::integral_constant<int, 4>{});
            }

            // ---- L3 (+L4): conv5x6 6->2 streamed over P2 row s-3; C1x1 2->1; threshold ----
            if (half == 0 && s >= 3) {
                const int j = q;                       // window column in the band
                const float* p2 = p2_ring + ((s - 3) & 1) * 6 * C::P2_RS;
#pragma unroll
                for (int ci = 0; ci < 6; ++ci) {
                    float v[5];
#pragma unroll
                    for (int kx = 0; kx < 5; ++kx) v[kx] = p2[ci * C::P2_RS + j + kx];
#pragma unroll
                    for (int i = 0; i < 6; ++i)
#pragma unroll
                        for (int m = 0; m < 2; ++m)
#pragma unroll
                            for (int kx = 0; kx < 5; ++kx)
                                acc3[m][i] = fmaf(W.w3[m][ci][(5 - i) * 5 + kx], v[kx], acc3[m][i]);
                }
                const int o = s - 8;                   // finished window row (task-relative)
                if (o >= 0) {
                    const float a0 = act(acc3[0][0] + W.b3[0]);
                    const float a1 = act(acc3[1][0] + W.b3[1]);
                    const float score = act(fmaf(W.w4[1], a1, fmaf(W.w4[0], a0, W.b4)));
                    const bool valid = (j < T.bw) && (o < nrows);
                    if (DEBUG && valid)
                        dbg_map[(int64_t)T.frame * dbg_map_frame_stride + L.map_off +
                                (int64_t)(T.y0 + o) * L.nx + (T.x0 + j)] = score;
                    const bool pred = valid && (score > T1);     // "exceeded"
                    const unsigned mask = __ballot_sync(0xFFFFFFFFu, pred);
                    if (mask) {
                        uint32_t base = 0;
                        const int leader = __ffs(mask) - 1;
                        if (lane == leader) base = atomicAdd(&ctrl->n_cand, (uint32_t)__popc(mask));
                        base = __shfl_sync(0xFFFFFFFFu, base, leader);
                        if (pred) {
                            const uint32_t idx = base + __popc(mask & ((1u << lane) - 1u));
                            if (idx < cand_cap) {
                                S1Cand c;
                                c.frame = T.frame;
                                c.level = T.level;
                                c.pad = 0;
                                c.ix = (int16_t)(T.x0 + j);
                                c.iy = (int16_t)(T.y0 + o);
                                c.s1 = score;
                                cands[idx] = c;
                            }
                        }
                    }
                }
#pragma unroll
                for (int m = 0; m < 2; ++m) {
#pragma unroll
                    for (int i = 0; i < 5; ++i) acc3[m][i] = acc3[m][i + 1];
                    acc3[m][5] = 0.f;
                }
            }
            __syncthreads();
        }
    }
}

constexpr int kNT = 128;

template <bool DEBUG>
void launch_impl(const Cnn1W& w, float T1, const uint8_t* levels, int64_t lfs,
                 const LevelInfo* d_levels, const S1Task* d_tasks, int n_tasks, S1Cand* cands,
                 uint32_t cand_cap, Ctrl* ctrl, float* dbg_map, int64_t dbg_fs, int sm_count,
                 cudaStream_t s)
{
    using C = Cfg<kNT>;
    const size_t smem = sizeof(float) * C::SMEM_FLOATS;
    static bool attr_set = false;
    if (!attr_set) {
        cudaFuncSetAttribute(stage1_kernel<kNT, DEBUG>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem);
        attr_set = true;
    }
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, stage1_kernel<kNT, DEBUG>, kNT, smem);
    if (occ < 1) occ = 1;
    int grid = sm_count * occ;
    if (grid > n_tasks) grid = n_tasks;
    if (grid < 1) return;
    stage1_kernel<kNT, DEBUG><<<grid, kNT, smem, s>>>(w, T1, levels, lfs, d_levels, d_tasks, n_tasks,
                                                      cands, cand_cap, ctrl, dbg_map, dbg_fs);
}

}  // namespace

int stage1_band_width() { return Cfg<kNT>::TW; }

void launch_stage1(const Cnn1W& w, float T1, const uint8_t* levels, int64_t level_frame_stride,
                   const LevelInfo* d_levels, const S1Task* d_tasks, int n_tasks, S1Cand* cands,
                   uint32_t cand_cap, Ctrl* ctrl, float* dbg_map, int64_t dbg_map_frame_stride,
                   int sm_count, cudaStream_t s)
{
    if (n_tasks <= 0) return;
    if (dbg_map)
        launch_impl<true>(w, T1, levels, level_frame_stride, d_levels, d_tasks, n_tasks, cands,
                          cand_cap, ctrl, dbg_map, dbg_map_frame_stride, sm_count, s);
    else
        launch_impl<false>(w, T1, levels, level_frame_stride, d_levels, d_tasks, n_tasks, cands,
                           cand_cap, ctrl, nullptr, 0, sm_count, s);
}

}  // namespace ccnn
