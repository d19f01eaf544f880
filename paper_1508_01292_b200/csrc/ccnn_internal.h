// ccnn_internal.h -- device data layout and launcher declarations shared by the
// runtime (runtime.cu) and the sm_100a kernels.  Not part of the ABI.
//
// Architecture R (R1; §3.1, Fig. 1 missing) is compiled in:
//   CNN1: C4x4 1->6, P, C3x3 6->6, P, C5x6 6->2, C1x1 2->1     (27x31 window, stride 4)
//   CNN2: C4x4 1->16, P, C3x3 16->6, P, C7x8 6->2, C1x1 2->1   (51x55 -> 5x5)
//   CNN3: C4x4 1->2, P, C3x3 2->2, P, C7x8 2->25, C1x1 25->1   (51x55 -> 5x5)
#pragma once
#include <algorithm>
#include <cstdint>
#include <cuda_runtime.h>

namespace ccnn {

constexpr int kWinW = 27, kWinH = 31;           // stage-1 window
constexpr int kStep = 4;                        // window step
constexpr int kPatchW = 51, kPatchH = 55;       // selective patch
constexpr int kPatchN = kPatchW * kPatchH;      // 2805
constexpr int kResp = 25;                       // 5x5 response map

// ---- weights, laid out for compile-time indexing (kernel parameters = constant bank) ----
struct __align__(16) Cnn1W {   // 797 weights + re-arranged copies for the stage-1 kernel
    float w2v[6][56];          // layer 2 per input map ci: [o*9 + ky*3 + kx] (54 used), float4 blocks
    float w3v[6][60];          // layer 3 per input map ci: [i][m][kx], i = 5 - ky (streaming order)
    float w1[6][16], b1[6];    // [out][ky*4+kx]
    float w2[6][6][9], b2[6];  // [out][in][ky*3+kx]
    float w3[2][6][30], b3[2]; // [out][in][ky*5+kx]
    float w4[2], b4;
    // layer 1 on the tensor cores (stage1.cu, S1_HMMA): per lane the mma.m16n8k16 B fragments
    // of W' = w1 / 127.5 * 2^s (raw pixel inputs, the O3 normalisation folded in) split into
    // fp16 hi + lo parts, [hi/lo][lane][reg] (maps 6, 7 zero); b1h = b1 - sum_k w1; the
    // accumulator is scaled back by l1_inv_scale = 2^-s
    uint32_t l1frag[2][32][2];
    float b1h[8];
    float l1_inv_scale;
    // layer 2 on the tensor cores (stage1_tc.cu): w2 * 2^s2 (max |w'| in [8, 16)) as fp16
    // hi + lo; the accumulator is scaled back by l2_inv_scale = 2^-s2
    float l2_inv_scale;
    float l3_inv_scale;        // likewise for layer 3 (w3)
    // stage1_tc.cu epilogue constants with Eq. 1's inner factor 2/3 folded in (the kernel
    // evaluates Eq. 1 on x' = 2x/3): [0..5] b1h, [6..11] b2, [12..13] b3, [14] l1_inv_scale,
    // [15] l2_inv_scale, [16] l3_inv_scale, [17..18] w4, [19] b4, all x 2/3
    float tcx[20];
};
template <int A, int B, int C>
struct __align__(16) SelNetW { // CNN2: <16,6,2>, CNN3: <2,2,25>
    float w1[A][16], b1[A];
    float w2[B][A][9], b2[B];
    float w3[C][B][56], b3[C]; // [out][in][ky*7+kx], 7 wide x 8 tall
    float w4[C], b4;
    // O3 folded into layer 1 (raw equalised pixels in): b1h = b1 - sum_k w1, and the power of
    // two that scales w1 / 127.5 into fp16 range for the tensor-core copies (selective_tc.cu)
    float b1h[A];
    float l1_inv_scale;
};
using Cnn2W = SelNetW<16, 6, 2>;
using Cnn3W = SelNetW<2, 2, 25>;

// ---- per-call geometry ----
struct FrameInfo {             // one frame of a batch, as the kernels read it
    const uint8_t* data;       // device pointer
    int64_t pitch;             // row pitch in bytes
    int32_t w, h;
    int32_t level0, nlevels;   // its levels: LevelInfo[level0 .. level0 + nlevels)
    int32_t tiles, tile_off;   // pyramid tiles of all its levels; their descriptors at
                               // tiles[tile_off ..] (shared by equally-sized frames), in
                               // kernel classes: [gather | quad]
    int32_t tiles_g, pad_t;    // tiles of the gather class (quad = the rest)
    unsigned long long tex;    // pitch-2D uint8 texture object over data (0 = none)
};
struct GrayJob {               // one interleaved R,G,B frame -> its gray copy (ingest.cu)
    const uint8_t* src;
    int64_t src_pitch;
    uint8_t* dst;              // 16-B aligned rows
    int64_t dst_pitch;
    int32_t w, h;
};
struct LevelInfo {             // one pyramid level of one frame of the batch
    double sigma;
    int64_t offset;            // byte offset of the level in the level arena
    int64_t map_off;           // offset of the level in the dense stage-1 map (debug)
    int32_t lw, lh, pitch;     // level size, row pitch (multiple of 16 B)
    int32_t nx, ny;            // window grid
    int32_t tab_off;           // offset of the level's x table (pitch entries) then y table
                               // (lh rounded up to kPyrTileRows entries); multiple of 4
    int32_t frame;             // the frame this level belongs to
    int32_t pad0;
    int32_t pad;
};
// pyramid CTA tile: kPyrCols output columns x kPyrGroups groups of kPyrRows rows of one
// level; descriptor = level-in-frame | tile column << 8 | tile row << 16
#ifndef PYR_ROWS
#define PYR_ROWS 8
#endif
constexpr int kPyrCols = 128, kPyrRows = PYR_ROWS, kPyrGroups = 32 / PYR_ROWS;
constexpr int kPyrTileRows = kPyrRows * kPyrGroups;
// levels with sigma >= kPyrQuadSigma are resampled 4 adjacent columns per thread
// (pyramid_quad_kernel), the rest by byte gathers (pyramid_gather4_kernel); frames narrower or
// shorter than 2 px: the clamped byte-gather form only.  (A third class, source rows staged in
// shared memory by cp.async for 0.25 <= sigma < 0.7, was measured and removed: DESIGN.md K1.)
constexpr double kPyrQuadSigma = 0.7;
enum PyrClass { kPyrGather = 0, kPyrQuad = 1, kPyrClasses = 2 };

// One stage-1 CTA task: a band of TW = 59 window columns x a segment of rows.  Patchwork
// (SURVEY §8(f) NEXT #1): a band holds up to kMaxPieces pieces of levels
// side by side -- piece p = window columns [x0, x0+w) of `level` (a global level id: levels of
// different frames may share a band), placed at band window
// column J; consecutive pieces are kPieceGap windows apart so no valid window straddles
// two pieces (the windows in the gap are computed and discarded).
constexpr int kMaxPieces = 4;
constexpr int kPieceGap = 6;       // 4*6 = 24 > 23 = input columns a window reaches past 4j
struct S1Piece { int16_t level, x0, w, J; };
struct S1Task {
    int32_t frame;                 // frame of the first piece (informational)
    int16_t y0, nrows;             // first window row / window rows (shared by all pieces)
    int16_t npieces, pad0;
    int32_t pad1;
    S1Piece piece[kMaxPieces];
};
struct S1Cand {                // stage-1 survivor record (16 B)
    int32_t frame;
    int16_t level, pad;
    int16_t ix, iy;            // window column j / row i
    float s1;
};
struct SelOut {                // selective-unit outcome per survivor
    int32_t K2, K3, delta, cnn3_ran;
    float score;
    int32_t bx, by, bw, bh;
};
struct AccBox {                // accepted raw box (O8)
    int32_t frame, x, y, w, h;
    float score;
};
struct OutBox { int32_t frame, x, y, w, h; float score; int32_t neighbors; };

// device control block, zeroed at the start of every detect
struct Ctrl {
    uint32_t task_next;        // stage-1 dynamic task counter
    uint32_t n_cand;           // stage-1 survivors (may exceed capacity -> error)
    uint32_t sel_next;         // selective dynamic work counter
    uint32_t n_stage2, n_stage3;
    uint32_t n_acc;            // accepted raw boxes
    uint32_t nms_done;         // NMS last-block ticket
    uint32_t n_out;            // boxes after NMS
    uint32_t nms_overflow;     // a frame exceeded the NMS capacity
    uint32_t strip_next;       // selective CNN2 (tcgen05) dynamic strip counter
    uint32_t pad[6];
};

constexpr int kMaxLevels = 256;   // pyramid levels per frame (scale_step 1.02 spans 11 octaves)
constexpr int kNmsCap = 4096;  // raw boxes per frame handled by one NMS CTA

// ---- launchers (stream-ordered, no sync) ----
// pyramid: every level of every frame, from the original frames
void launch_to_gray(const GrayJob* d_jobs, int n_jobs, int sm_count, cudaStream_t s);
// use_tex: every frame has a texture object (FrameInfo.tex): 2x2 footprints by tex2Dgather
// max_tiles: the most tiles any frame has, in all classes / per class (PyrClass order);
// returns the number of kernels launched
int launch_pyramid(const FrameInfo* d_frames, int n_frames, int max_tiles, const int (&max_class)[kPyrClasses],
                   bool safe, bool use_tex, uint8_t* levels, const LevelInfo* d_levels,
                   const uint32_t* d_tiles, const uint32_t* d_tabs, cudaStream_t s);
// stage 1 (fused CNN1 + threshold + compaction): a persistent grid of stage1_grid() CTAs
// taking tasks[0 .. cta_first[grid]) from an atomic counter, longest first
void launch_stage1(const Cnn1W& w, float T1, const uint8_t* levels, const LevelInfo* d_levels,
                   const S1Task* d_tasks, const int32_t* d_cta_first, int grid, S1Cand* cands,
                   uint32_t cand_cap, Ctrl* ctrl, float* dbg_map, cudaStream_t s);
int stage1_band_width();          // TW of the compiled stage-1 kernel
int stage1_grid(int sm_count);    // CTAs of the persistent stage-1 launch
int stage1_task_cost(int nrows);  // relative cost of a task (super-steps)
// stage 1 with layers 1-2 on tcgen05 (stage1_tc.cu, the default): same task list format,
// band width stage1_tc_band_width(); d_bmats = the B matrices built by stage1_tc_bmats
void launch_stage1_tc(const Cnn1W& w, float T1, const uint16_t* d_bmats, const uint8_t* levels,
                      const LevelInfo* d_levels, const S1Task* d_tasks, const int32_t* d_cta_first, int grid,
                      S1Cand* cands, uint32_t cand_cap, Ctrl* ctrl, float* dbg_map, cudaStream_t s);
int stage1_tc_band_width();
int stage1_tc_grid(int sm_count);
int stage1_tc_task_cost(int nrows);
int stage1_tc_pipes_per_cta();    // band pipelines per CTA (each takes its own tasks)
double stage1_tc_task_mma_flops(int nrows);
int stage1_tc_bmats(const Cnn1W& w, uint16_t* out);   // fills out (kStage1TcBmatHalves), returns count
constexpr int kStage1TcBmatHalves = 8 * 96 * 16 + 8 * 96 * 16 + 5 * 24 * 16;   // layers 1, 2, 3
// selective unit (stage 2/3), persistent over the survivor queue
struct SelParams { float T2a, T2b; int32_t Tnn, rule; };
// CNN2 on the tensor cores (selective_tc.cu): epilogue constants with Eq. 1's inner factor 2/3
// folded in (the kernel evaluates Eq. 1 on x' = 2x/3): per layer the accumulator scale
// (2^-s of the split weights) and biases, layer 4's weights and bias, all x 2/3
struct Cnn2Tc {
    float l1s, l1b[16];        // layer 1: b1 - sum_k w1 (O3 folded), scale of w1/127.5 * 2^s
    float l2s, l2b[6];
    float l3s, l3b[2];
    float w4[2], b4;
};
int selective_tc_bmats(const Cnn2W& w, uint16_t* out, Cnn2Tc* consts);   // returns the fp16 count
constexpr int kSelTcBmatHalves = (6 * 128 * 16) + (16 * 96 * 16) + (7 * 32 * 16);
// stage 2 over strips of kSelTcCands survivors: patch preparation (O5, O2, O6), CNN2 layers
// 1-3 on tcgen05, layer 4 -> resp2[cand][50] (orientation E then M, 5x5 row-major); the
// equalised patch of every survivor the rule sends to CNN3 -> epatch[cand][kEPatchBytes]
// (rows of 51 pixels, row-major)
constexpr int kSelTcCands = 5;
constexpr int kEPatchBytes = 2816;             // 55 x 51 = 2805, padded to 16 B
void launch_selective_cnn2_tc(const Cnn2Tc& k, SelParams sp, const uint16_t* d_bmats,
                              const FrameInfo* d_frames, const LevelInfo* d_levels,
                              const S1Cand* cands, uint32_t cand_cap, float* resp2, uint8_t* epatch,
                              Ctrl* ctrl, int sm_count, cudaStream_t s);
// stage 3 + the decision per survivor, after launch_selective_cnn2_tc: K2 from resp2; CNN3 on
// the survivor's equalised patch (epatch) only where the rule needs it (P:99 early stop)
void launch_selective(const Cnn3W& w3, SelParams sp, const LevelInfo* d_levels,
                      const S1Cand* cands, uint32_t cand_cap, const float* resp2,
                      const uint8_t* epatch, SelOut* out, float* dbg_resp, AccBox* acc, Ctrl* ctrl,
                      int sm_count, cudaStream_t s);
// grouping / NMS per frame + compaction of the results
void launch_nms(const AccBox* acc, Ctrl* ctrl, int n_frames, int min_cluster, OutBox* staging,
                int32_t* frame_counts, OutBox* out, cudaStream_t s);

}  // namespace ccnn
