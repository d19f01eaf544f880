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
//  * one persistent launch per batch; a CTA owns a band of TW = 59 windows of one level
//    (128 pooled-layer-1 columns, 63 pooled-layer-2 columns) and a segment of its rows;
//    the host assigns (frame, level, band, segment) tasks to CTAs longest-first (LPT),
//    so no per-level launches (the paper's small-level launch overhead);
//  * line-buffer pipeline in shared memory marching down the band, TWO window rows per
//    "super-step", two __syncthreads per super-step (layer 1 | loader + layers 2, 3):
//    input ring, pooled-layer-1 ring, pooled-layer-2 ring, 41 KB in all -> 5 CTAs per SM;
//  * layer 1 (half the FLOPs) on the tensor cores: mma.sync m16n8k16, A = 16 conv outputs
//    x 16 taps of raw pixels (exact in fp16; the input ring holds fp16 pairs in two copies
//    shifted by one pixel so every fragment pair is an aligned 32-bit load), B = the six
//    maps' weights / 127.5 * 2^s split into fp16 hi + lo parts (two MMAs, fp32 accumulate:
//    ~2^-22 relative weight error), bias and 2^-s applied after the pooling max;
//    S1_HMMA=0 builds the all-FFMA form;
//  * layers 2-4: work is split over DATA only (columns x rows), never over maps or taps, so
//    all 128 threads run one instruction stream whose weights are warp-uniform: every MAC is
//    an FFMA with a uniform-register (constant-bank kernel parameter) operand;
//  * max-pool BEFORE the activation (Eq. 1 is monotone: act(max) == max(act));
//    layer 3 streams P2 rows through register accumulators, the even/odd rows of a pair
//    on adjacent lanes, partial sums combined with one shfl per output;
//  * threshold + warp ballot/popc + ONE atomicAdd per warp into the survivor queue.
#include <algorithm>

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

#ifndef S1_MIN_BLOCKS
#define S1_MIN_BLOCKS 5
#endif

#ifndef S1_HMMA
#define S1_HMMA 1                       // layer 1 on the tensor cores (mma.sync m16n8k16)
#endif
#ifndef S1_L2_UNROLL
#define S1_L2_UNROLL 1                  // layer-2 input-map loop unrolled
#endif
#ifndef S1_L3_UNROLL
#define S1_L3_UNROLL 0
#endif

constexpr int NT = 128;                 // threads per CTA
constexpr int TW = NT / 2 - 5;          // 59 windows per band
constexpr int IN_WORDS = NT / 2 + 1;    // 65 32-bit words cover the 4*TW+23 = 259 input columns
constexpr int IN_ODD = NT + 4;          // odd input columns start inside a ring row
constexpr int IN_RS = 2 * NT + 8;       // input ring row stride (floats)
constexpr int IN_RING = 12;             // rows 8v .. 8v+10 (+ 8v+11 .. 8v+18 after the mid barrier)
constexpr int P1_ODD = NT / 2 + 16;     // odd P1 columns start (bank offset 16)
constexpr int P1_RS = NT + 18;          // one (row, map) of the P1 ring (L2 lane 63 reads [144]);
                                        // == 2 mod 16: layer-1 stores of maps 0/2/4 x even/odd hit disjoint banks
constexpr int P1_RING = 6;              // rows 4v-2 .. 4v+3
constexpr int P2_RS = NT / 2 + 8;
constexpr int P2_RING = 4;              // rows 2v-3 .. 2v
// S1_HMMA input ring: raw pixels as fp16 pairs, two copies per row -- copy0 word j = pixels
// (2j, 2j+1), copy1 word j = pixels (2j+1, 2j+2) -- so every A-fragment pair is one aligned
// 32-bit load; row stride 272 words (== 16 mod 32: rows y, y+1 of one load hit disjoint banks)
constexpr int IN_CW = 136;              // words per copy (130 used)
constexpr int IN_RSW = 2 * IN_CW;       // words per ring row
constexpr int IN_FLOATS = S1_HMMA ? IN_RING * IN_RSW : IN_RING * IN_RS;
constexpr int SMEM_FLOATS = IN_FLOATS + P1_RING * 6 * P1_RS + P2_RING * 6 * P2_RS;
// loader: 8 new input rows x 65 words per super-step = 520 loads on 128 threads.  Thread t
// owns ONE word column (t < 65: word t of rows 0-3; else word t-65 of rows 4-7) plus, for
// t < 8, one leftover (word 63 + (t&1) of row 4 + (t>>1)) -- so a thread's loads come from
// at most two source columns and its source descriptors stay in registers.
static_assert(IN_WORDS == 65 && NT == 128, "loader mapping");

__device__ __forceinline__ float u8f(uint32_t v)
{
    return fmaf((float)v, 1.0f / 127.5f, -1.0f);   // O3: (v - 127.5) / 127.5
}

#if !S1_HMMA
__device__ __forceinline__ void store_word(float* ring, int slot, int w, uint32_t word)
{
    float* row = ring + slot * IN_RS;
    const float2 ev = make_float2(u8f(word & 0xFFu), u8f((word >> 16) & 0xFFu));
    const float2 od = make_float2(u8f((word >> 8) & 0xFFu), u8f(word >> 24));
    *reinterpret_cast<float2*>(row + 2 * w) = ev;
    *reinterpret_cast<float2*>(row + IN_ODD + 2 * w) = od;
}
#else
// two bytes of `word` (selector) -> an fp16 pair of the exact pixel values: 0x64pp is the
// fp16 1024 + p, minus 1024
__device__ __forceinline__ uint32_t h2_of(uint32_t word, uint32_t sel)
{
    const uint32_t t = __byte_perm(word, 0x64646464u, sel);
    uint32_t r;
    asm("sub.rn.f16x2 %0, %1, %2;" : "=r"(r) : "r"(t), "r"(0x64006400u));
    return r;
}
// input word w (pixels 4w .. 4w+3) of ring row `slot`: copy0 words 2w, 2w+1; copy1 word 2w
// and the halves 4w-1 (upper half of word 2w-1) and 4w+2 (lower half of word 2w+1)
__device__ __forceinline__ void store_word(float* ring, int slot, int w, uint32_t word)
{
    uint32_t* row = reinterpret_cast<uint32_t*>(ring) + slot * IN_RSW;
    *reinterpret_cast<uint2*>(row + 2 * w) = make_uint2(h2_of(word, 0x4140), h2_of(word, 0x4342));
    uint32_t* c1 = row + IN_CW;
    const uint32_t mid = h2_of(word, 0x4241);                  // pixels (4w+1, 4w+2)
    const uint32_t edge = h2_of(word, 0x4340);                 // pixels (4w, 4w+3)
    c1[2 * w] = mid;
    uint16_t* c1h = reinterpret_cast<uint16_t*>(c1);
    if (w > 0) c1h[4 * w - 1] = (uint16_t)(edge & 0xFFFFu);
    c1h[4 * w + 2] = (uint16_t)(edge >> 16);
}

// P1 stores of a lane's two maps (rows 2c4, 2c4+1), skipped for the zero maps (c4 == 3)
__device__ __forceinline__ void st2_pred(uint32_t saddr, float v0, float v1, int c4)
{
    asm volatile("{\n\t.reg .pred p;\n\tsetp.lt.s32 p, %3, 3;\n\t"
                 "@p st.shared.f32 [%0], %1;\n\t@p st.shared.f32 [%0+%4], %2;\n\t}"
                 :: "r"(saddr), "f"(v0), "f"(v1), "r"(c4), "n"(4 * P1_RS) : "memory");
}

__device__ __forceinline__ void mma16816(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2,
                                         uint32_t a3, uint32_t b0, uint32_t b1)
{
    asm("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
#endif

__device__ __forceinline__ int pmod(int a, int m) { return ((a % m) + m) % m; }

template <bool DEBUG>
__global__ void __launch_bounds__(NT, S1_MIN_BLOCKS) stage1_kernel(
    const __grid_constant__ Cnn1W W, const float T1,
    const uint8_t* __restrict__ levels, const LevelInfo* __restrict__ lvinfo,
    const S1Task* __restrict__ tasks, const int32_t* __restrict__ cta_first,
    S1Cand* __restrict__ cands, const uint32_t cand_cap, Ctrl* __restrict__ ctrl,
    float* __restrict__ dbg_map)
{
    extern __shared__ __align__(16) float smem[];
    float* const in_ring = smem;
    float* const p1_ring = in_ring + IN_FLOATS;
    float* const p2_ring = p1_ring + P1_RING * 6 * P1_RS;

    const int tid = threadIdx.x;
    const int lane = tid & 31;
    const int warp = tid >> 5;
    // layer-2 thread -> (P2 column q2, row r2 of the super-step's pair)
    const int q2 = 32 * (warp & 1) + lane;
    const int r2 = warp >> 1;
    // layer-3 thread -> (window column j3, P2 row parity r3); pairs on adjacent lanes
    const int j3 = 16 * warp + (lane >> 1);
    const int r3 = lane & 1;

#if S1_HMMA
    // layer-1 MMA fragments: lane = (group m, thread-in-group c4); B (weights, hi / lo) and
    // the bias of this lane's two maps stay in registers for the whole kernel
    const int c4 = lane & 3, mg = lane >> 2;
    const uint32_t bh0 = W.l1frag[0][lane][0], bh1 = W.l1frag[0][lane][1];
    const uint32_t bl0 = W.l1frag[1][lane][0], bl1 = W.l1frag[1][lane][1];
    const float bias0 = W.b1h[2 * c4], bias1 = W.b1h[2 * c4 + 1];
    // P1 column of tile pair g: 32 * warp + 8 * g + mg (even / odd columns de-interleaved:
    // + 4 g in the store index); the lane's first map row 2 * c4
    const int p1_col0 = 32 * warp + mg;
    const int p1_lane = 2 * c4 * P1_RS + ((mg & 1) ? P1_ODD + (p1_col0 >> 1) : (p1_col0 >> 1));
    const int xw0 = 32 * warp + mg + (c4 & 1);                    // input word, tile pair 0
    const uint32_t p1_s = (uint32_t)__cvta_generic_to_shared(p1_ring + p1_lane);
#endif
    const int ld_w = tid < IN_WORDS ? tid : tid - IN_WORDS;      // primary word column
    const int ld_r0 = tid < IN_WORDS ? 0 : 4;                      // its rows ld_r0 .. +3
    const bool ld_x = tid < 8;                                     // leftover load
    const int ld_xw = 63 + (tid & 1), ld_xr = 4 + (tid >> 1);

    __shared__ int s_task;
    const int n_tasks = cta_first[gridDim.x];
    for (;;) {                                   // dynamic list scheduling, longest tasks first
        if (tid == 0) s_task = (int)atomicAdd(&ctrl->task_next, 1u);
        __syncthreads();
        const int ti = s_task;
        if (ti >= n_tasks) break;
        const S1Task T = tasks[ti];
        const int nrows = T.nrows;
        const int row_base = 4 * T.y0;
        // piece of a band window column j: the last piece starting at or before j (patchwork);
        // selected with predicated moves (no dynamic indexing -> no local memory)
        auto piece_of = [&](int j) -> S1Piece {
            S1Piece P = T.piece[0];
#pragma unroll
            for (int q = 1; q < kMaxPieces; ++q)
                if (q < T.npieces && T.piece[q].J <= j) P = T.piece[q];
            return P;
        };
        // input word w of the band (columns 4w .. 4w+3) of band row r: the piece's level,
        // clamped to its rows and its row pitch (gap columns read a neighbour: discarded)
        // (32-bit word offset from `levels`, pitch in words | rows << 16): two registers
        struct Src { uint32_t woff, pitch_lh; };
        auto src_of = [&](int w) -> Src {
            const S1Piece P = piece_of(w);
            const LevelInfo& L = lvinfo[P.level];
            const int lw = min(P.x0 + w - P.J, L.pitch / 4 - 1);
            const int64_t off = L.offset / 4 + lw;
            return Src{(uint32_t)off, (uint32_t)(L.pitch / 4) | ((uint32_t)L.lh << 16)};
        };
        auto gword = [&](const Src& sc, int r) -> uint32_t {
            const int row = min(row_base + r, (int)(sc.pitch_lh >> 16) - 1);
            return __ldg(reinterpret_cast<const uint32_t*>(levels) + sc.woff +
                         (uint32_t)row * (sc.pitch_lh & 0xFFFFu));
        };
        const Src lsrc = src_of(ld_w);
        const Src xsrc = src_of(ld_x ? ld_xw : 0);
        // the window column this thread emits (layer 3): its piece, level coordinates
        const S1Piece PE = piece_of(j3);
        const int e_level = PE.level;
        const int e_x = PE.x0 + j3 - PE.J;
        const bool e_col = (j3 >= PE.J) && (j3 < PE.J + PE.w);
        const LevelInfo& LE = lvinfo[e_level];
        const int e_rows = min(nrows, LE.ny - T.y0);       // rows of this piece in the segment

        // prologue: input rows 0..10 to the ring, rows 11..18 into registers
        for (int g = tid; g < 11 * IN_WORDS; g += NT)
            store_word(in_ring, g / IN_WORDS, g % IN_WORDS, gword(src_of(g % IN_WORDS), g / IN_WORDS));
        uint32_t pre[4], prex;
#pragma unroll
        for (int k = 0; k < 4; ++k) pre[k] = gword(lsrc, 11 + ld_r0 + k);
        prex = ld_x ? gword(xsrc, 11 + ld_xr) : 0u;

        float acc3[2][6], carry[2] = {0.f, 0.f};
#pragma unroll
        for (int m = 0; m < 2; ++m)
#pragma unroll
            for (int i = 0; i < 6; ++i) acc3[m][i] = 0.f;
        __syncthreads();

        const int nsteps = (nrows + 7) / 2 + 1;      // ceil((nrows + 6) / 2) + 1
        for (int v = 0; v < nsteps; ++v) {
            // ---- L1: conv4x4 1->6, pool, act -> P1 rows 4v .. 4v+3 (input rows 8v .. 8v+10);
            //      thread = P1 column, two row pairs ----
#if S1_HMMA
            // tensor-core form: a tile = 16 conv-1 outputs of one conv row (rows m / m+8 of the
            // MMA = columns xb+2m / xb+2m+1), K = the 16 taps, N = 8 maps (6 used); the tile
            // pair (conv rows 2p, 2p+1) holds whole 2x2 pool cells in each thread
            {
            const uint32_t* const ring32 = reinterpret_cast<const uint32_t*>(in_ring);
            const int rbase = (8 * v) % IN_RING + (c4 >> 1);          // ring row of input row 8v+ky0
#pragma unroll 1
            for (int pr = 0; pr < 4; ++pr) {
                int sl[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const int t = rbase + 2 * pr + q;                 // < 2 * IN_RING
                    sl[q] = (t >= IN_RING ? t - IN_RING : t) * IN_RSW;
                }
                // this lane's two maps of P1 row 4v+pr (lanes c4 = 3 hold the zero maps 6, 7:
                // predicated off inside one asm block -- no branch)
                const int p1slot = (4 * v + pr) % P1_RING;
                const uint32_t p1dst = p1_s + 4u * (uint32_t)(p1slot * 6 * P1_RS);
                // all four tile pairs' MMAs first, then their epilogues: the MMA latency of
                // one pair is covered by the others
                float dA[4][4], dB[4][4];
#pragma unroll
                for (int g = 0; g < 4; ++g) {
                    const int xw = xw0 + 8 * g;                          // word of pixel xb+2m+kx0
#pragma unroll
                    for (int k = 0; k < 4; ++k) { dA[g][k] = 0.f; dB[g][k] = 0.f; }
                    const uint32_t a0 = ring32[sl[0] + xw], a1 = ring32[sl[0] + IN_CW + xw];
                    const uint32_t a2 = ring32[sl[2] + xw], a3 = ring32[sl[2] + IN_CW + xw];
                    const uint32_t e0 = ring32[sl[1] + xw], e1 = ring32[sl[1] + IN_CW + xw];
                    const uint32_t e2 = ring32[sl[3] + xw], e3 = ring32[sl[3] + IN_CW + xw];
                    mma16816(dA[g], a0, a1, a2, a3, bh0, bh1);
                    mma16816(dB[g], e0, e1, e2, e3, bh0, bh1);
                    mma16816(dA[g], a0, a1, a2, a3, bl0, bl1);
                    mma16816(dB[g], e0, e1, e2, e3, bl0, bl1);
                }
#pragma unroll
                for (int g = 0; g < 4; ++g) {
                    const float m0 = fmaxf(fmaxf(dA[g][0], dA[g][2]), fmaxf(dB[g][0], dB[g][2]));
                    const float m1 = fmaxf(fmaxf(dA[g][1], dA[g][3]), fmaxf(dB[g][1], dB[g][3]));
                    st2_pred(p1dst + 16u * g, act(fmaf(m0, W.l1_inv_scale, bias0)),   // P1 column +8g
                             act(fmaf(m1, W.l1_inv_scale, bias1)), c4);
                }
            }
            }
#else
#pragma unroll 1
            for (int h = 0; h < 2; ++h) {
                const int c = tid;
                float x[7][5];
                const int r0 = (8 * v + 4 * h) % IN_RING;
#pragma unroll
                for (int rr = 0; rr < 7; ++rr) {
                    int slot = r0 + rr;
                    slot = slot >= IN_RING ? slot - IN_RING : slot;
                    const float* row = in_ring + slot * IN_RS;
                    x[rr][0] = row[c];
                    x[rr][1] = row[IN_ODD + c];
                    x[rr][2] = row[c + 1];
                    x[rr][3] = row[IN_ODD + c + 1];
                    x[rr][4] = row[c + 2];
                }
                const int pcol = (c & 1) ? P1_ODD + (c >> 1) : (c >> 1);
#pragma unroll
                for (int r = 0; r < 2; ++r) {
                    float a[4][6];                    // the 2x2 conv outputs of one pool cell
#pragma unroll
                    for (int p = 0; p < 4; ++p) {
                        const int py = p >> 1, px = p & 1;
#pragma unroll
                        for (int o = 0; o < 6; ++o) a[p][o] = W.b1[o];
#pragma unroll
                        for (int ky = 0; ky < 4; ++ky)
#pragma unroll
                            for (int kx = 0; kx < 4; ++kx) {
                                const float xv = x[2 * r + py + ky][px + kx];
#pragma unroll
                                for (int o = 0; o < 6; ++o) a[p][o] = fmaf(W.w1[o][ky * 4 + kx], xv, a[p][o]);
                            }
                    }
                    const int slot = (4 * v + 2 * h + r) % P1_RING;
#pragma unroll
                    for (int o = 0; o < 6; ++o)
                        p1_ring[(slot * 6 + o) * P1_RS + pcol] =
                            act(fmaxf(fmaxf(a[0][o], a[1][o]), fmaxf(a[2][o], a[3][o])));
                }
            }
#endif

            __syncthreads();   // P1 rows 4v..4v+3 visible; input rows 8v..8v+7 dead

            // ---- loader: input rows 8v+11 .. 8v+18 into the slots of 8v .. 8v+7 (fetched
            //      during the previous super-step), then prefetch rows 8v+19 .. 8v+26 ----
#pragma unroll
            for (int k = 0; k < 4; ++k)
                store_word(in_ring, (8 * v + 11 + ld_r0 + k) % IN_RING, ld_w, pre[k]);
            if (ld_x) store_word(in_ring, (8 * v + 11 + ld_xr) % IN_RING, ld_xw, prex);
#pragma unroll
            for (int k = 0; k < 4; ++k) pre[k] = gword(lsrc, 8 * v + 19 + ld_r0 + k);
            if (ld_x) prex = gword(xsrc, 8 * v + 19 + ld_xr);

            // ---- L2: conv3x3 6->6, pool, act -> P2 row p = 2v-1+r2 (P1 rows 2p .. 2p+3) ----
            {
                const int p = 2 * v - 1 + r2;
                int rs[4];
#pragma unroll
                for (int rr = 0; rr < 4; ++rr) rs[rr] = pmod(2 * p + rr, P1_RING);
                float a[6][4];
#pragma unroll
                for (int o = 0; o < 6; ++o)
#pragma unroll
                    for (int k = 0; k < 4; ++k) a[o][k] = W.b2[o];
#if S1_L2_UNROLL
#pragma unroll
#else
#pragma unroll 1
#endif
                for (int ci = 0; ci < 6; ++ci) {
                    float xv[4][4];
#pragma unroll
                    for (int rr = 0; rr < 4; ++rr) {
                        const float* row = p1_ring + (rs[rr] * 6 + ci) * P1_RS;
                        xv[rr][0] = row[q2];
                        xv[rr][1] = row[P1_ODD + q2];
                        xv[rr][2] = row[q2 + 1];
                        xv[rr][3] = row[P1_ODD + q2 + 1];
                    }
                    // explicit 16-byte loads of the parameter block -> LDCU [UR+imm]
                    float wv[56];
                    const float4* w4p = reinterpret_cast<const float4*>(W.w2v[ci]);
#pragma unroll
                    for (int k4 = 0; k4 < 14; ++k4) {
                        const float4 t4 = w4p[k4];
                        wv[4 * k4] = t4.x; wv[4 * k4 + 1] = t4.y; wv[4 * k4 + 2] = t4.z; wv[4 * k4 + 3] = t4.w;
                    }
#pragma unroll
                    for (int o = 0; o < 6; ++o)
#pragma unroll
                        for (int ky = 0; ky < 3; ++ky)
#pragma unroll
                            for (int kx = 0; kx < 3; ++kx) {
                                const float w = wv[o * 9 + ky * 3 + kx];
#pragma unroll
                                for (int k = 0; k < 4; ++k)
                                    a[o][k] = fmaf(w, xv[(k >> 1) + ky][(k & 1) + kx], a[o][k]);
                            }
                }
                const int pslot = pmod(p, P2_RING);
#pragma unroll
                for (int o = 0; o < 6; ++o)
                    p2_ring[(pslot * 6 + o) * P2_RS + q2] =
                        act(fmaxf(fmaxf(a[o][0], a[o][1]), fmaxf(a[o][2], a[o][3])));
            }

            // ---- L3: conv5x6 6->2 streamed over P2 row p = 2v-3+r3 (written in the previous
            //      super-step) -> outputs p-5 .. p ----
            {
                const int p = 2 * v - 3 + r3;
                const float* p2 = p2_ring + pmod(p, P2_RING) * 6 * P2_RS;
#if S1_L3_UNROLL
#pragma unroll
#else
#pragma unroll 1
#endif
                for (int ci = 0; ci < 6; ++ci) {
                    float xv[5];
#pragma unroll
                    for (int kx = 0; kx < 5; ++kx) xv[kx] = p2[ci * P2_RS + j3 + kx];
                    float wv[60];
                    const float4* w4p = reinterpret_cast<const float4*>(W.w3v[ci]);
#pragma unroll
                    for (int k4 = 0; k4 < 15; ++k4) {
                        const float4 t4 = w4p[k4];
                        wv[4 * k4] = t4.x; wv[4 * k4 + 1] = t4.y; wv[4 * k4 + 2] = t4.z; wv[4 * k4 + 3] = t4.w;
                    }
#pragma unroll
                    for (int i = 0; i < 6; ++i)
#pragma unroll
                        for (int m = 0; m < 2; ++m)
#pragma unroll
                            for (int kx = 0; kx < 5; ++kx)
                                acc3[m][i] = fmaf(wv[(i * 2 + m) * 5 + kx], xv[kx], acc3[m][i]);
                }
                // even/odd partial sums: lane r3=0 finalises output 2v-8 (its acc[0] + the odd
                // lane's carry), lane r3=1 output 2v-7 (its acc[0] + the even lane's acc[1])
                float fin[2];
#pragma unroll
                for (int m = 0; m < 2; ++m) {
                    const float send = r3 ? carry[m] : acc3[m][1];
                    fin[m] = acc3[m][0] + __shfl_xor_sync(0xFFFFFFFFu, send, 1);
                    carry[m] = acc3[m][1];
#pragma unroll
                    for (int i = 0; i < 4; ++i) acc3[m][i] = acc3[m][i + 2];
                    acc3[m][4] = 0.f;
                    acc3[m][5] = 0.f;
                }
                const int o = 2 * v - 8 + r3;                // finished window row (task-relative)
                const float a0 = act(fin[0] + W.b3[0]);
                const float a1 = act(fin[1] + W.b3[1]);
                const float score = act(fmaf(W.w4[1], a1, fmaf(W.w4[0], a0, W.b4)));
                const bool valid = (o >= 0) && (o < e_rows) && e_col;
                if (DEBUG && valid)
                    dbg_map[LE.map_off + (int64_t)(T.y0 + o) * LE.nx + e_x] = score;
                const bool pred = valid && (score > T1);             // "exceeded"
                const unsigned mask = __ballot_sync(0xFFFFFFFFu, pred);
                if (mask) {
                    uint32_t base = 0;
                    const int leader = __ffs(mask) - 1;
                    if (lane == leader) base = atomicAdd(&ctrl->n_cand, (uint32_t)__popc(mask));
                    base = __shfl_sync(0xFFFFFFFFu, base, leader);
                    if (pred) {
                        const uint32_t idx = base + __popc(mask & ((1u << lane) - 1u));
                        if (idx < cand_cap) {
                            S1Cand cd;
                            cd.frame = LE.frame;
                            cd.level = (int16_t)e_level;
                            cd.pad = 0;
                            cd.ix = (int16_t)e_x;
                            cd.iy = (int16_t)(T.y0 + o);
                            cd.s1 = score;
                            cands[idx] = cd;
                        }
                    }
                }
            }
#ifdef S1_PROFILE
            const long long t_bar0 = clock64();
#endif
            __syncthreads();
#ifdef S1_PROFILE
            if (lane == 0) atomicAdd(&ctrl->pad[0], (uint32_t)((clock64() - t_bar0) >> 6));
#endif
        }
    }
}

template <bool DEBUG>
int occupancy()
{
    const size_t smem = sizeof(float) * SMEM_FLOATS;
    cudaFuncSetAttribute(stage1_kernel<DEBUG>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, stage1_kernel<DEBUG>, NT, smem);
    return occ < 1 ? 1 : occ;
}

}  // namespace

int stage1_band_width() { return TW; }

int stage1_grid(int sm_count)
{
    // the production and debug instantiations must share one schedule
    return sm_count * std::min(occupancy<false>(), occupancy<true>());
}

int stage1_task_cost(int nrows) { return (nrows + 7) / 2 + 1 + 2; }   // super-steps + prologue

void launch_stage1(const Cnn1W& w, float T1, const uint8_t* levels, const LevelInfo* d_levels,
                   const S1Task* d_tasks, const int32_t* d_cta_first, int grid, S1Cand* cands,
                   uint32_t cand_cap, Ctrl* ctrl, float* dbg_map, cudaStream_t s)
{
    if (grid <= 0) return;
    const size_t smem = sizeof(float) * SMEM_FLOATS;
    if (dbg_map) {
        cudaFuncSetAttribute(stage1_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        stage1_kernel<true><<<grid, NT, smem, s>>>(w, T1, levels, d_levels, d_tasks, d_cta_first,
                                                   cands, cand_cap, ctrl, dbg_map);
    } else {
        cudaFuncSetAttribute(stage1_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        stage1_kernel<false><<<grid, NT, smem, s>>>(w, T1, levels, d_levels, d_tasks, d_cta_first,
                                                    cands, cand_cap, ctrl, nullptr);
    }
}

}  // namespace ccnn
