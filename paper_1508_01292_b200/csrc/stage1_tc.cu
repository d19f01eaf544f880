// stage1_tc.cu -- stage 1 (CNN1 dense scan + threshold + compaction) with the three conv
// layers on the 5th-generation tensor cores (tcgen05, accumulators in TMEM).  DESIGN.md K2 "v10".
//
// PAPER.md §3.3: CNN1 densely scans every pyramid level; its output cells are the 27x31
// windows at a 4-px step; windows whose response exceeds T1 go to the selective unit.
// CNN1 = architecture R (R1): C4x4 1->6, max-pool, C3x3 6->6, max-pool, C5x6 6->2,
// C1x1 2->1, Eq. 1 after every conv, fp32-accurate.
//
// Work unit: a band of 128 pooled-layer-2 (P2) columns of one level (TW = 123 windows; the
// patchwork pieces of stage1.cu's plan) x a segment of window rows, marched down one
// P2 row per step.  Cost model (measured, profiles/r1_tcgen05_probe.jsonl): an MMA costs ~28
// cycles with A in TMEM and ~40-44 with A in shared memory whatever its N up to ~64, so the
// design minimises the NUMBER of MMAs and the shared-memory A bytes.  Per step:
//  * layer 1 = implicit GEMM on the tensor core, A in TMEM: TMEM lane m (= P2 column X) holds,
//    per image row of an 8-row ring, the 8 raw pixels 4X .. 4X+7 (two aligned level words,
//    exact in fp16); one MMA (M=128, K=16 = two image rows, N=96 = 2 P1 rows x 2 P1 columns
//    (2X, 2X+1) x 4 pool positions x 6 maps) per image-row pair and weight part (w/127.5 * 2^s
//    split into fp16 hi + lo, both accumulated in fp32): 8 MMAs produce two P1 rows of the
//    band's 256 columns, the 2x2 pool cells of every map in one TMEM lane.  Row pair 0 only
//    reaches P1 row 0 and row pair 3 only P1 row 1: those MMAs run at N = 48;
//  * epilogue (4 warps, one TMEM lane each): max over the pool positions, bias, Eq. 1, split
//    into fp16 hi + lo, stored as 16-B entries (6 channels + 2 zero) in shared-memory planes,
//    even / odd columns de-interleaved;
//  * layer 2 = implicit GEMM from shared memory (no im2col), STREAMED: each P1 row is read
//    once and feeds the two P2 rows it belongs to -- row m = P2 column X, K = 16 = (P1 column
//    2X+2d, 8 channels) + (P1 column 2X+2d+1, 8 channels), two core matrices one plane apart
//    (LBO); N = 96 = {w hi, w lo} x {P2 row q, P2 row q+1} x 4 pool positions x 6 maps for
//    hi(A), N = 48 (w hi) for lo(A) (lo x lo dropped: ~2^-22): 4 MMAs per P1 row.  The two
//    accumulators alternate between TMEM halves (B matrices per half parity); a drained half
//    is zeroed with tcgen05.st before it starts the next P2 row;
//  * epilogue: hi + lo halves, max over positions, bias, Eq. 1 -> P2 row (fp16 hi / lo);
//  * layer 3 on tcgen05: row m = window column j, K = 16 = (P2 entry j+kx hi) + (its lo), one
//    MMA per kx (5), N = 24 = {w hi, w lo} x 6 kernel rows x 2 maps (lo(A) x lo(w) zero): the
//    contributions of the P2 row to the 6 window rows it reaches; the data warps keep 6 running
//    sums per map;
//  * layer 4 (1x1) on the FFMA pipe, threshold > T1, warp ballot / popc, one atomicAdd per
//    warp into the survivor queue.
// Warps 0-3 do all data work; warp 4 allocates TMEM and issues every MMA (elect.sync, so the
// operands stay warp-uniform); MMA completion is tracked with tcgen05.commit -> mbarrier.  The
// MMAs of layer 1 (one unit ahead) and layer 2 run while warps 0-3 do the epilogues.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cuda_fp16.h>

#include "ccnn_internal.h"
#include "tc05.cuh"

namespace ccnn {
namespace {

// Eq. 1, y = 1.7159 tanh(2x/3) via the paper's approximation, on x' = 2x/3 (the
// factor is folded into the preceding bias / scale, Cnn1W::tcx), two values per f32x2 op
__device__ __forceinline__ float2 act2(float2 x)
{
    const float2 a2 = __fmul2_rn(x, x);
    const float2 t = __ffma2_rn(a2, make_float2(1.41645f, 1.41645f), make_float2(1.0f, 1.0f));
    const float2 p = __ffma2_rn(a2, t, make_float2(fabsf(x.x) + 1.0f, fabsf(x.y) + 1.0f));
    float2 r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r.x) : "f"(p.x));
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r.y) : "f"(p.y));
    const float2 y = __ffma2_rn(make_float2(-1.7159f, -1.7159f), r, make_float2(1.7159f, 1.7159f));
    return make_float2(copysignf(y.x, x.x), copysignf(y.y, x.y));
}
__device__ __forceinline__ float act1(float x)           // x' = 2x/3, one value
{
    const float a2 = x * x;
    const float p = fmaf(a2, fmaf(a2, 1.41645f, 1.0f), fabsf(x) + 1.0f);
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(p));
    return copysignf(fmaf(-1.7159f, r, 1.7159f), x);
}

constexpr int NW = 4;                   // data warps of a pipeline
constexpr int PWT = 32 * (NW + 1);      // threads of a pipeline (+ its MMA warp)
constexpr int NPIPE = 2;                // independent band pipelines per CTA (one CTA per SM):
                                        // they share one copy of the B matrices, so the SM keeps
                                        // ~90 KB of L1 for the level loads and the overlapped pyramid
constexpr int NT = NPIPE * PWT;
constexpr int TW = 123;                 // windows per band (P2 columns 0..126 valid)
// shared memory (bytes)
constexpr int BMAT = 96 * 16 * 2;              // one layer-1 B (N = 96, K = 16): [k chunk 2][n 96][8]
constexpr int B1_BYTES = 8 * BMAT;             // layer-1 B: [pair 4][w part 2]
constexpr int BMAT2 = 96 * 16 * 2;             // one layer-2 B (N = 96): [k chunk 2][n 96][8]
constexpr int B2_BYTES = 8 * BMAT2;            // layer-2 B: [half parity 2][P1 row parity 2][d 2]
constexpr int BMAT3 = 24 * 16 * 2;             // one layer-3 B (N = 24): [k chunk 2][n 24][8]
constexpr int B3_BYTES = 5 * BMAT3;            // layer-3 B: [kx 5]
constexpr int PL_E = 132;                      // entries per (row, part, parity); 128 written
constexpr int PL_PAR = PL_E * 16;              // 2112 B == 64 mod 128: conflict-free stores
constexpr int PL_HL = 2 * PL_PAR;
constexpr int PL_SLOT = 2 * PL_HL;
constexpr int P1_RING = 4;                     // P1 rows 2q .. 2q+3 live (layer 2 streams them)
constexpr int P2_E = 136;                      // P2 entries per (buffer, part): 128 written + reach
constexpr int P2_HL = P2_E * 16;
constexpr int P2_BUF = 2 * P2_HL;
constexpr int OFF_B1 = 0, OFF_B2 = OFF_B1 + B1_BYTES, OFF_B3 = OFF_B2 + B2_BYTES;
constexpr int OFF_PL = OFF_B3 + B3_BYTES;      // per pipeline: P1 ring, then two P2 buffers
constexpr int OFF_P2_REL = P1_RING * PL_SLOT;
constexpr int PIPE_BYTES = OFF_P2_REL + 2 * P2_BUF;
constexpr int SMEM_BYTES = OFF_PL + NPIPE * PIPE_BYTES;
static_assert((B1_BYTES + B2_BYTES + B3_BYTES) / 2 == kStage1TcBmatHalves, "B matrix image size");
// TMEM columns
constexpr uint32_t TM_A = 0;                   // A ring: image row slot s at +4 s (32 columns)
constexpr uint32_t TM_D1 = 32;                 // layer-1 accumulator (96)
constexpr uint32_t TM_D2 = 128;                // layer-2 accumulators: [half 0 wh | half 1 wh | half 0 wl | half 1 wl]
constexpr uint32_t TM_D3 = 224;                // layer-3 accumulator (24)
constexpr uint32_t TM_PIPE = 256;              // TMEM columns per pipeline
constexpr uint32_t TM_COLS = TM_PIPE * NPIPE;
constexpr uint32_t IDESC = tc05::idesc_f16(128, 96);
constexpr uint32_t IDESC1_HALF = tc05::idesc_f16(128, 48);  // layer-1 row pairs 0 (P1 row 0), 3 (P1 row 1)
constexpr uint32_t IDESC2 = tc05::idesc_f16(128, 96);
constexpr uint32_t IDESC2_LO = tc05::idesc_f16(128, 48);    // lo(A): the w-hi columns only
constexpr uint32_t IDESC3 = tc05::idesc_f16(128, 24);

__device__ __forceinline__ uint32_t h2_of(uint32_t word, uint32_t sel)
{
    const uint32_t t = __byte_perm(word, 0x64646464u, sel);
    uint32_t r;
    asm("sub.rn.f16x2 %0, %1, %2;" : "=r"(r) : "r"(t), "r"(0x64006400u));
    return r;
}
__device__ __forceinline__ uint32_t pack_h2(float a, float b)
{
    const __half2 h = __floats2half2_rn(a, b);
    return *reinterpret_cast<const uint32_t*>(&h);
}
// fp32 pair -> fp16 hi pair + fp16 lo pair (v - hi), packed
__device__ __forceinline__ void split_h2(float2 v, uint32_t& hi, uint32_t& lo)
{
    const __half2 h = __float22half2_rn(v);
    const float2 d = __ffma2_rn(__half22float2(h), make_float2(-1.0f, -1.0f), v);   // exact
    hi = *reinterpret_cast<const uint32_t*>(&h);
    lo = pack_h2(d.x, d.y);
}
__device__ __forceinline__ void ld48(uint32_t taddr, float (&v)[48])
{
    uint32_t r[48];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%48];\n\t"
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%32,%33,%34,%35,%36,%37,%38,%39,%40,%41,%42,%43,%44,%45,%46,%47}, [%49];\n\t"
        "tcgen05.wait::ld.sync.aligned;"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31]),
          "=r"(r[32]), "=r"(r[33]), "=r"(r[34]), "=r"(r[35]), "=r"(r[36]), "=r"(r[37]), "=r"(r[38]), "=r"(r[39]),
          "=r"(r[40]), "=r"(r[41]), "=r"(r[42]), "=r"(r[43]), "=r"(r[44]), "=r"(r[45]), "=r"(r[46]), "=r"(r[47])
        : "r"(taddr), "r"(taddr + 32u)
        : "memory");
#pragma unroll
    for (int i = 0; i < 48; ++i) v[i] = __uint_as_float(r[i]);
}

// TMEM store of 24 zero columns (32 lanes of the warp's quadrant)
__device__ __forceinline__ void st_zero24(uint32_t taddr)
{
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%2,%2,%2,%2,%2,%2,%2,%2,%2,%2,%2,%2,%2,%2,%2,%2};\n\t"
        "tcgen05.st.sync.aligned.32x32b.x8.b32 [%1], {%2,%2,%2,%2,%2,%2,%2,%2};"
        :: "r"(taddr), "r"(taddr + 16u), "r"(0u) : "memory");
}

template <bool DEBUG>
#ifndef S1_MINB
#define S1_MINB 1
#endif
__global__ void __launch_bounds__(NT, S1_MINB) stage1_tc_kernel(
    const __grid_constant__ Cnn1W W, const float T1, const uint16_t* __restrict__ bmats,
    const uint8_t* __restrict__ levels, const LevelInfo* __restrict__ lvinfo,
    const S1Task* __restrict__ tasks, const int32_t* __restrict__ cta_first,
    S1Cand* __restrict__ cands, const uint32_t cand_cap, Ctrl* __restrict__ ctrl,
    float* __restrict__ dbg_map)
{
    extern __shared__ __align__(128) uint8_t smem[];
    __shared__ int s_task[NPIPE];
    __shared__ uint32_t s_tmem;
    __shared__ __align__(8) uint64_t bar_l1s[NPIPE], bar_l2s[NPIPE], bar_l3s[NPIPE];

    const int tid = threadIdx.x;
    // warp index through shfl: provably warp-uniform, so role branches stay on the uniform
    // datapath (constant-bank weights via LDCU [UR+imm], MMA descriptors in uniform registers)
    const int warp = __shfl_sync(0xFFFFFFFFu, tid >> 5, 0);
    const int lane = tid & 31;
    const int pipe = warp / (NW + 1);          // band pipeline of this warp
    const bool mma_warp = warp - pipe * (NW + 1) == NW;

    // ---- one-time setup: weights (B matrices) to shared memory, zeroed plane padding ----
    {
        const uint4* src = reinterpret_cast<const uint4*>(bmats);
        uint4* dst = reinterpret_cast<uint4*>(smem + OFF_B1);
        for (int i = tid; i < (B1_BYTES + B2_BYTES + B3_BYTES) / 16; i += NT) dst[i] = src[i];
        uint4* z = reinterpret_cast<uint4*>(smem + OFF_PL);
        for (int i = tid; i < (SMEM_BYTES - OFF_PL) / 16; i += NT) z[i] = make_uint4(0, 0, 0, 0);
    }
    if (warp == NW) tc05::tmem_alloc(&s_tmem, TM_COLS);
    if (tid == 0) {
        for (int p = 0; p < NPIPE; ++p) {
            tc05::mbar_init(&bar_l1s[p], 1);
            tc05::mbar_init(&bar_l2s[p], 1);
            tc05::mbar_init(&bar_l3s[p], 1);
        }
        tc05::mbar_fence_init();
    }
    tc05::fence_async_smem();
    tc05::fence_before();
    __syncthreads();
    tc05::fence_after();
    const uint32_t tm = s_tmem + TM_PIPE * (uint32_t)pipe;
    uint64_t& bar_l1 = bar_l1s[pipe];
    uint64_t& bar_l2 = bar_l2s[pipe];
    uint64_t& bar_l3 = bar_l3s[pipe];
    const int OFF_P1P = OFF_PL + pipe * PIPE_BYTES;            // this pipeline's P1 ring
    const int OFF_P2P = OFF_P1P + OFF_P2_REL;                  // ... and P2 buffers
    const uint32_t pbar = 1u + (uint32_t)pipe;                 // its named barrier
    auto pipe_sync = [pbar] { tc05::named_sync(pbar, PWT); };
    // completed phases of each mbarrier (the waiting side's count)
    uint32_t ph_l1 = 0, ph_l2 = 0, ph_l3 = 0;

    const uint32_t s_base = tc05::smem_u32(smem);
    const int m = 32 * (warp & 3) + lane;    // TMEM lane / P2 column / window column
    const uint32_t t_lane = (uint32_t)(32 * (warp & 3)) << 16;

    const int n_tasks = cta_first[gridDim.x];
    for (;;) {
        if (tid == pipe * PWT) s_task[pipe] = (int)atomicAdd(&ctrl->task_next, 1u);
        pipe_sync();
        const int ti = s_task[pipe];
        if (ti >= n_tasks) break;
        const S1Task T = tasks[ti];
        const int nrows = T.nrows;
        const int NQ = nrows + 5;                       // P2 rows of the task
        const int row_base = 4 * T.y0;                  // first image row of the task

        auto piece_of = [&](int j) -> S1Piece {
            S1Piece P = T.piece[0];
#pragma unroll
            for (int q = 1; q < kMaxPieces; ++q)
                if (q < T.npieces && T.piece[q].J <= j) P = T.piece[q];
            return P;
        };
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

        if (!mma_warp) {
            // ============================ data warps ============================
            // loader: lane m (P2 column X = m) loads band words X and X+1 (pixels 4X .. 4X+7) of
            // each image row and writes them as 4 fp16 pairs to its TMEM lane
            const Src ls0 = src_of(m);
            const Src ls1 = src_of(m + 1);
            auto fetch = [&](int r, uint32_t (&wv)[2]) {
                wv[0] = gword(ls0, r);
                wv[1] = gword(ls1, r);
            };
            auto put = [&](int r, const uint32_t (&wv)[2]) {      // image row r -> ring slot r % 8
                tc05::st4(tm + t_lane + TM_A + 4 * (r & 7), h2_of(wv[0], 0x4140), h2_of(wv[0], 0x4342),
                          h2_of(wv[1], 0x4140), h2_of(wv[1], 0x4342));
            };
            // layer-1 epilogue of unit k: P1 rows 2k + rr (task-relative), columns 2X + cx -> planes;
            // accumulator column rr * 48 + cx * 24 + pos * 6 + o
            auto l1_epilogue = [&](int k) {
#pragma unroll 1
                for (int rr = 0; rr < 2; ++rr) {
                    float d[48];
                    ld48(tm + t_lane + TM_D1 + 48 * rr, d);
#pragma unroll
                    for (int cx = 0; cx < 2; ++cx) {
                        uint32_t hi[3], lo[3];
#pragma unroll
                        for (int c = 0; c < 3; ++c) {
                            float mx[2];
#pragma unroll
                            for (int e = 0; e < 2; ++e) {
                                const float* q = d + cx * 24 + 2 * c + e;
                                mx[e] = fmaxf(fmaxf(q[0], q[6]), fmaxf(q[12], q[18]));
                            }
                            const float2 x = __ffma2_rn(make_float2(mx[0], mx[1]), make_float2(W.tcx[14], W.tcx[14]),
                                                        make_float2(W.tcx[2 * c], W.tcx[2 * c + 1]));
                            split_h2(act2(x), hi[c], lo[c]);
                        }
                        const int slot = (2 * k + rr) % P1_RING;
                        uint8_t* e = smem + OFF_P1P + slot * PL_SLOT + cx * PL_PAR + m * 16;
                        *reinterpret_cast<uint4*>(e) = make_uint4(hi[0], hi[1], hi[2], 0u);
                        *reinterpret_cast<uint4*>(e + PL_HL) = make_uint4(lo[0], lo[1], lo[2], 0u);
                    }
                }
            };
            // layer-2 epilogue of P2 row q (TMEM half q & 1) -> P2 buffer q & 1 as fp16 hi / lo
            // entries (column m); the half is zeroed for P2 row q + 2
            auto l2_epilogue = [&](int q) {
                const uint32_t h = (uint32_t)(q & 1);
                float dh[24], dl[24];
                tc05::ld24(tm + t_lane + TM_D2 + 24 * h, dh);
                tc05::ld24(tm + t_lane + TM_D2 + 48 + 24 * h, dl);
                st_zero24(tm + t_lane + TM_D2 + 24 * h);
                st_zero24(tm + t_lane + TM_D2 + 48 + 24 * h);
                uint32_t hi[3], lo[3];
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    float2 s4[4];
#pragma unroll
                    for (int p = 0; p < 4; ++p)
                        s4[p] = __fadd2_rn(make_float2(dh[p * 6 + 2 * c], dh[p * 6 + 2 * c + 1]),
                                           make_float2(dl[p * 6 + 2 * c], dl[p * 6 + 2 * c + 1]));
                    const float m0 = fmaxf(fmaxf(s4[0].x, s4[1].x), fmaxf(s4[2].x, s4[3].x));
                    const float m1 = fmaxf(fmaxf(s4[0].y, s4[1].y), fmaxf(s4[2].y, s4[3].y));
                    const float2 x = __ffma2_rn(make_float2(m0, m1), make_float2(W.tcx[15], W.tcx[15]),
                                                make_float2(W.tcx[6 + 2 * c], W.tcx[7 + 2 * c]));
                    split_h2(act2(x), hi[c], lo[c]);
                }
                uint8_t* e = smem + OFF_P2P + (q & 1) * P2_BUF + m * 16;
                *reinterpret_cast<uint4*>(e) = make_uint4(hi[0], hi[1], hi[2], 0u);
                *reinterpret_cast<uint4*>(e + P2_HL) = make_uint4(lo[0], lo[1], lo[2], 0u);
            };

            // the window column this thread emits
            const int j3 = m;
            const S1Piece PE = piece_of(j3);
            const int e_level = PE.level;
            const int e_x = PE.x0 + j3 - PE.J;
            const bool e_col = (j3 < TW) && (j3 >= PE.J) && (j3 < PE.J + PE.w);
            const LevelInfo& LE = lvinfo[e_level];
            const int e_rows = min(nrows, LE.ny - T.y0);
            // acc3[mm][i]: layer-3 map mm of window row (P2 row p) - 5 + i, in B-matrix scale
            float acc3[2][6];
#pragma unroll
            for (int mm = 0; mm < 2; ++mm)
#pragma unroll
                for (int i = 0; i < 6; ++i) acc3[mm][i] = 0.f;
            // layer-3 epilogue of P2 row p: its contributions to the 6 window rows it reaches
            // (TMEM column (w part) * 12 + ky * 2 + mm), then the finished window row p - 5
            auto l3_epilogue = [&](int p) {
                float d[24];
                tc05::ld24(tm + t_lane + TM_D3, d);
#pragma unroll
                for (int i = 0; i < 6; ++i) {
                    const int n = (5 - i) * 2;
                    const float2 c2 = __fadd2_rn(make_float2(d[n], d[n + 1]), make_float2(d[12 + n], d[13 + n]));
                    const float2 a2 = __fadd2_rn(make_float2(acc3[0][i], acc3[1][i]), c2);
                    acc3[0][i] = a2.x;
                    acc3[1][i] = a2.y;
                }
                const int o = p - 5;                        // finished window row (task-relative)
                const float2 a = act2(__ffma2_rn(make_float2(acc3[0][0], acc3[1][0]),
                                                 make_float2(W.tcx[16], W.tcx[16]),
                                                 make_float2(W.tcx[12], W.tcx[13])));
#pragma unroll
                for (int mm = 0; mm < 2; ++mm) {
#pragma unroll
                    for (int i = 0; i < 5; ++i) acc3[mm][i] = acc3[mm][i + 1];
                    acc3[mm][5] = 0.f;
                }
                const float score = act1(fmaf(W.tcx[18], a.y, fmaf(W.tcx[17], a.x, W.tcx[19])));
                const bool valid = (o >= 0) && (o < e_rows) && e_col;
                if (DEBUG && valid) dbg_map[LE.map_off + (int64_t)(T.y0 + o) * LE.nx + e_x] = score;
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
            };
            auto sync_for_mma = [&]() {
                tc05::fence_async_smem();
                tc05::fence_before();
                pipe_sync();
            };
            auto wait_l1 = [&]() {
                tc05::mbar_wait(&bar_l1, ph_l1 & 1); ++ph_l1;
                tc05::fence_after();
            };

            // prologue: image rows 0..7 -> L1(0); rows 8..11 once unit 0 is drained; both
            // layer-2 halves zeroed before the first streamed MMAs
            {
                uint32_t wv[8][2];
#pragma unroll
                for (int r = 0; r < 8; ++r) fetch(r, wv[r]);
#pragma unroll
                for (int r = 0; r < 8; ++r) put(r, wv[r]);
                tc05::st_wait();
                sync_for_mma();                                // -> MMA warp issues L1(0)
                uint32_t wx[4][2];
#pragma unroll
                for (int r = 0; r < 4; ++r) fetch(8 + r, wx[r]);
                wait_l1();
                l1_epilogue(0);
                st_zero24(tm + t_lane + TM_D2);
                st_zero24(tm + t_lane + TM_D2 + 24);
                st_zero24(tm + t_lane + TM_D2 + 48);
                st_zero24(tm + t_lane + TM_D2 + 72);
#pragma unroll
                for (int r = 0; r < 4; ++r) put(8 + r, wx[r]);
                tc05::st_wait();
                sync_for_mma();                                // -> L1(1), L2s(0)
            }
            // iteration q: drain L3(q-2), L1(q+1), L2s(q) (-> P2 row q-1, half zeroed); the MMA
            // warp then issues L3(q-1), L1(q+2), L2s(q+1)
#pragma unroll 1
            for (int q = 0; q <= NQ + 1; ++q) {
                const bool more = q + 2 <= NQ;                 // unit q+2 exists
                uint32_t wx[4][2];
                if (more) {
#pragma unroll
                    for (int r = 0; r < 4; ++r) fetch(4 * q + 12 + r, wx[r]);
                }
                if (q >= 2) {
                    tc05::mbar_wait(&bar_l3, ph_l3 & 1); ++ph_l3;      // L3(q-2) done
                    tc05::fence_after();
                    l3_epilogue(q - 2);
                }
                if (q + 1 <= NQ) {
                    wait_l1();
                    l1_epilogue(q + 1);
                }
                if (q <= NQ) {
                    tc05::mbar_wait(&bar_l2, ph_l2 & 1); ++ph_l2;      // L2s(q) done
                    tc05::fence_after();
                    if (q >= 1) {
                        l2_epilogue(q - 1);
                    } else {                                   // half 1 took unit 0's dy 2, 3 junk
                        st_zero24(tm + t_lane + TM_D2 + 24);
                        st_zero24(tm + t_lane + TM_D2 + 72);
                    }
                }
                if (more) {
#pragma unroll
                    for (int r = 0; r < 4; ++r) put(4 * q + 12 + r, wx[r]);
                }
                tc05::st_wait();
                sync_for_mma();                                // -> L3(q-1), L1(q+2), L2s(q+1)
            }
        } else {
            // ============================ MMA warp ============================
            const uint64_t bd1 = tc05::sdesc(s_base + OFF_B1, 96 * 16, 128);
            const uint64_t bd2 = tc05::sdesc(s_base + OFF_B2, 96 * 16, 128);
            const uint64_t ad2 = tc05::sdesc(s_base + OFF_P1P, PL_PAR, 128);
            const uint64_t bd3 = tc05::sdesc(s_base + OFF_B3, 24 * 16, 128);
            const uint64_t ad3 = tc05::sdesc(s_base + OFF_P2P, P2_HL, 128);
            // layer 1 of unit k: row pair 1 first (N = 96, initialises the accumulator), then
            // pairs 2 (N = 96), 0 (P1 row 0 only) and 3 (P1 row 1 only) at N = 48
            auto issue_l1 = [&](int k) {
                if (tc05::elect_one()) {
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        const int p = i == 0 ? 1 : i == 1 ? 2 : i == 2 ? 0 : 3;
                        const uint32_t n0 = p == 3 ? 48u : 0u;          // first accumulator column
#pragma unroll
                        for (int hl = 0; hl < 2; ++hl) {
                            const uint32_t a = tm + TM_A + 4 * ((4 * k + 2 * p) & 7);
                            tc05::mma_f16_ts(tm + TM_D1 + n0, a,
                                             bd1 + (uint64_t)(((p * 2 + hl) * BMAT + n0 * 16) >> 4),
                                             (p == 0 || p == 3) ? IDESC1_HALF : IDESC, (i | hl) != 0);
                        }
                    }
                    tc05::commit(&bar_l1);
                }
                __syncwarp();
            };
            // layer 2, streamed: the P1 rows of unit u (2u, 2u+1) into P2 row u-1 (kernel rows
            // dy 2, 3; TMEM half (u-1) & 1) and P2 row u (dy 0, 1; half u & 1)
            auto issue_l2s = [&](int u) {
                if (tc05::elect_one()) {
                    const int par = (u - 1) & 1;               // half of P2 row u-1
#pragma unroll
                    for (int rp = 0; rp < 2; ++rp) {
                        const uint32_t slot_off = (uint32_t)(((2 * u + rp) % P1_RING) * PL_SLOT);
#pragma unroll
                        for (int d = 0; d < 2; ++d) {
                            const uint64_t b = bd2 + (uint64_t)((((par * 2 + rp) * 2 + d) * BMAT2) >> 4);
                            const uint64_t a = ad2 + (uint64_t)((slot_off + d * 16) >> 4);
                            tc05::mma_f16(tm + TM_D2, a, b, IDESC2, 1u);
                            tc05::mma_f16(tm + TM_D2, a + (uint64_t)(PL_HL >> 4), b, IDESC2_LO, 1u);
                        }
                    }
                    tc05::commit(&bar_l2);
                }
                __syncwarp();
            };
            // layer 3 of P2 row p: row m = window column j, K = 16 = P2 entry j+kx hi + lo
            // (LBO = the hi -> lo plane distance), N = 24 = {w hi, w lo} x 6 kernel rows x 2 maps
            auto issue_l3 = [&](int p) {
                if (tc05::elect_one()) {
#pragma unroll
                    for (int kx = 0; kx < 5; ++kx) {
                        const uint64_t a = ad3 + (uint64_t)(((p & 1) * P2_BUF + kx * 16) >> 4);
                        const uint64_t b = bd3 + (uint64_t)((kx * BMAT3) >> 4);
                        tc05::mma_f16(tm + TM_D3, a, b, IDESC3, kx != 0);
                    }
                    tc05::commit(&bar_l3);
                }
                __syncwarp();
            };
            pipe_sync();                                       // rows 0..7 in TMEM
            tc05::fence_after();
            issue_l1(0);
            pipe_sync();                                       // rows 8..11, P1 rows 0, 1, D2 zeroed
            tc05::fence_after();
            issue_l1(1);
            issue_l2s(0);
#pragma unroll 1
            for (int q = 0; q <= NQ + 1; ++q) {
                pipe_sync();
                tc05::fence_after();
                if (q >= 1 && q <= NQ) issue_l3(q - 1);
                if (q + 2 <= NQ) issue_l1(q + 2);
                if (q + 1 <= NQ) issue_l2s(q + 1);
            }
        }
    }
    tc05::fence_before();
    __syncthreads();
    tc05::fence_after();
    if (warp == NW) tc05::tmem_dealloc(s_tmem, TM_COLS);
}

// shared-memory carveout: one CTA of two pipelines (135 KB) fits the 164 KB configuration (72% of
// 228 KB); the rest of the unified L1 (~90 KB) stays cache for the level loads and the
// overlapped pyramid's byte gathers (K1)
#ifndef S1_CARVEOUT                            // experiments: -DS1_CARVEOUT=50 -DS1_MAX_CTAS=1
#define S1_CARVEOUT 72
#endif
#ifndef S1_MAX_CTAS
#define S1_MAX_CTAS 1
#endif
constexpr int kCarveoutPct = S1_CARVEOUT;

template <bool DEBUG>
int occupancy()
{
    cudaFuncSetAttribute(stage1_tc_kernel<DEBUG>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
    cudaFuncSetAttribute(stage1_tc_kernel<DEBUG>, cudaFuncAttributePreferredSharedMemoryCarveout,
                         kCarveoutPct);
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, stage1_tc_kernel<DEBUG>, NT, SMEM_BYTES);
    if (const char* v = std::getenv("CCNN_VERBOSE"))
        if (v[0] == '1') std::fprintf(stderr, "ccnn: stage1_tc<%d> occupancy %d (smem %d)\n", (int)DEBUG, occ, SMEM_BYTES);
    // the occupancy API reports 1 for this kernel although ncu's launch limits (registers 3,
    // shared memory 2) allow 2; use the shared-memory bound directly (a CTA that finds no
    // task simply exits: the schedule is an atomic task counter)
    int dev = 0, smem_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
    occ = std::max(occ, smem_sm / (SMEM_BYTES + 128 + 1024));
    occ = std::min(occ, S1_MAX_CTAS);        // TMEM: 512 columns per CTA (two pipelines)
    return occ < 1 ? 1 : occ;
}

}  // namespace

int stage1_tc_band_width() { return TW; }
int stage1_tc_grid(int sm_count) { return sm_count * std::min(occupancy<false>(), occupancy<true>()); }
int stage1_tc_task_cost(int nrows) { return nrows + 5 + 2; }
int stage1_tc_pipes_per_cta() { return NPIPE; }
// tensor-core FLOPs (2 M N K per MMA) the kernel issues for a task of nrows window rows:
// NQ + 1 layer-1 units and streamed layer-2 P1-row pairs, NQ layer-3 P2 rows (NQ = nrows + 5)
double stage1_tc_task_mma_flops(int nrows)
{
    constexpr double mk = 2.0 * 128 * 16;                            // 2 M K of one MMA
    constexpr double l1 = mk * (4 * 96 + 4 * 48);                    // row pairs 1, 2 / 0, 3, hi + lo
    constexpr double l2 = mk * 2 * 2 * (96 + 48);                    // 2 P1 rows x 2 d x (hi(A), lo(A))
    constexpr double l3 = mk * 5 * 24;                               // 5 kx
    const int nq = nrows + 5;
    return (nq + 1) * (l1 + l2) + nq * l3;
}

// B matrices of the three tensor-core layers (fp16 bit patterns, the kernel's shared-memory
// image); returns the fp16 count.  K-major canonical layout of one B (N rows, K = 16):
// [k chunk 2][n N][8].
int stage1_tc_bmats(const Cnn1W& w, uint16_t* out)
{
    const int total = (B1_BYTES + B2_BYTES + B3_BYTES) / 2;
    std::fill(out, out + total, (uint16_t)0);
    auto put = [&](uint16_t* mat, int N, int n, int kk, float v) {
        mat[(kk >> 3) * N * 8 + n * 8 + (kk & 7)] = __half_as_ushort(__float2half_rn(v));
    };
    auto split = [](float wp, int part) {
        const float hi = __half2float(__float2half_rn(wp));
        return part ? wp - hi : wp;
    };
    // layer 1: mat = pair p * 2 + part; n = rr * 48 + cx * 24 + pos * 6 + o (P1 column 2X + cx);
    // kk = e * 8 + c: image row 2p + e of the unit, pixel 4X + c
    const double sc1 = 1.0 / (double)w.l1_inv_scale;
    for (int p = 0; p < 4; ++p)
        for (int part = 0; part < 2; ++part)
            for (int cx = 0; cx < 2; ++cx)
                for (int rr = 0; rr < 2; ++rr)
                    for (int pos = 0; pos < 4; ++pos)
                        for (int o = 0; o < 6; ++o)
                            for (int kk = 0; kk < 16; ++kk) {
                                const int py = pos >> 1, px = pos & 1;
                                const int d = 2 * p + (kk >> 3), c = kk & 7;
                                const int ky = d - 2 * rr - py, kx = c - 2 * cx - px;
                                if (ky < 0 || ky > 3 || kx < 0 || kx > 3) continue;
                                const float wp = (float)((double)w.w1[o][ky * 4 + kx] / 127.5 * sc1);
                                put(out + (p * 2 + part) * (BMAT / 2), 96, rr * 48 + cx * 24 + pos * 6 + o, kk,
                                    split(wp, part));
                            }
    // layer 2 (streamed): mat = (par * 2 + rp) * 2 + d, for P1 row 2u + rp of unit u with
    // P2 row u-1 in TMEM half par (kernel row dy = 2 + rp) and P2 row u in half 1 - par
    // (dy = rp); n = wpart * 48 + half * 24 + pos * 6 + o; kk = c * 8 + ch, P1 column 2X+2d+c
    uint16_t* out2 = out + B1_BYTES / 2;
    const double sc2 = 1.0 / (double)w.l2_inv_scale;
    for (int par = 0; par < 2; ++par)
        for (int rp = 0; rp < 2; ++rp)
            for (int d = 0; d < 2; ++d)
                for (int wh = 0; wh < 2; ++wh)
                    for (int half = 0; half < 2; ++half) {
                        const int dy = half == par ? 2 + rp : rp;
                        for (int pos = 0; pos < 4; ++pos)
                            for (int o = 0; o < 6; ++o)
                                for (int kk = 0; kk < 16; ++kk) {
                                    const int py = pos >> 1, px = pos & 1;
                                    const int dx = 2 * d + (kk >> 3), ch = kk & 7;
                                    const int ky = dy - py, kx = dx - px;
                                    if (ch >= 6 || ky < 0 || ky > 2 || kx < 0 || kx > 2) continue;
                                    const float wp = (float)((double)w.w2[o][ch][ky * 3 + kx] * sc2);
                                    put(out2 + ((par * 2 + rp) * 2 + d) * (BMAT2 / 2), 96,
                                        wh * 48 + half * 24 + pos * 6 + o, kk, split(wp, wh));
                                }
                    }
    // layer 3: mat = kx; n = wpart * 12 + ky * 2 + mm; kk = A part * 8 + ch (A part 0 = the
    // P2 entry's hi, 1 = its lo; lo(A) x lo(w) stays zero)
    uint16_t* out3 = out + (B1_BYTES + B2_BYTES) / 2;
    const double sc3 = 1.0 / (double)w.l3_inv_scale;
    for (int kx = 0; kx < 5; ++kx)
        for (int wh = 0; wh < 2; ++wh)
            for (int ky = 0; ky < 6; ++ky)
                for (int mm = 0; mm < 2; ++mm)
                    for (int kk = 0; kk < 16; ++kk) {
                        const int ha = kk >> 3, ch = kk & 7;
                        if (ch >= 6 || (ha && wh)) continue;
                        const float wp = (float)((double)w.w3[mm][ch][ky * 5 + kx] * sc3);
                        put(out3 + kx * (BMAT3 / 2), 24, wh * 12 + ky * 2 + mm, kk, split(wp, wh));
                    }
    return total;
}

void launch_stage1_tc(const Cnn1W& w, float T1, const uint16_t* d_bmats, const uint8_t* levels,
                      const LevelInfo* d_levels, const S1Task* d_tasks, const int32_t* d_cta_first, int grid,
                      S1Cand* cands, uint32_t cand_cap, Ctrl* ctrl, float* dbg_map, cudaStream_t s)
{
    if (grid <= 0) return;
    if (dbg_map) {
        cudaFuncSetAttribute(stage1_tc_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
        cudaFuncSetAttribute(stage1_tc_kernel<true>, cudaFuncAttributePreferredSharedMemoryCarveout,
                             kCarveoutPct);
        stage1_tc_kernel<true><<<grid, NT, SMEM_BYTES, s>>>(w, T1, d_bmats, levels, d_levels, d_tasks, d_cta_first,
                                                            cands, cand_cap, ctrl, dbg_map);
    } else {
        cudaFuncSetAttribute(stage1_tc_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
        cudaFuncSetAttribute(stage1_tc_kernel<false>, cudaFuncAttributePreferredSharedMemoryCarveout,
                             kCarveoutPct);
        stage1_tc_kernel<false><<<grid, NT, SMEM_BYTES, s>>>(w, T1, d_bmats, levels, d_levels, d_tasks, d_cta_first,
                                                             cands, cand_cap, ctrl, nullptr);
    }
}

}  // namespace ccnn
