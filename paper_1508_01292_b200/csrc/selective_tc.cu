// selective_tc.cu -- stage 2 of the cascade: CNN2 on every stage-1 survivor, on the
// 5th-generation tensor cores (tcgen05, accumulators in TMEM).  DESIGN.md K3.
//
// PAPER.md §3.3: each region found by CNN1 is read from the ORIGINAL frame with its
// neighbourhood, scaled to 51x55, histogram-equalised and mirrored; CNN2 gives a 5x5 response
// map per orientation and K2 = #responses exceeding T2.  CNN2 = architecture R (R1):
// C4x4 1->16, max-pool, C3x3 16->6, max-pool, C7x8 6->2, C1x1 2->1, Eq. 1 after every conv,
// fp32-accurate.  The paper runs this "selective unit" asynchronously on the CPU
// or, in patchwork mode, "by scanning all the found regions in a single pass" on
// the GPU -- which is what this kernel does: a persistent grid drains the survivor
// queue in strips.
//
// A STRIP = kSelTcCands (5) survivors, i.e. 10 patches (each survivor's equalised patch E and
// its mirror M) placed side by side: patch slot s owns TMEM lanes 12s .. 12s+11, lane = P2
// column X of the slot (image columns 4X .. 4X+7), so CNN2's first two layers run exactly as
// stage 1's CNN1 does over a 128-column band (stage1_tc.cu): one pipeline step = one P2 row.
//  * patch preparation (per survivor, one warp each): O5 geometry, O2 sampling from the frame,
//    256-bin histogram, O6 LUT, equalised E into shared memory (64-B rows, pixel x at 4 + x);
//    M(x, y) = E(50 - x, y) is read through a byte permutation by its lanes (no second image);
//  * layer 1 = implicit GEMM, A in TMEM (8 raw equalised pixels per lane per image row, exact in
//    fp16; O3's (v - 127.5)/127.5 folded into the weights), K = 16 = two image rows, N = 128 =
//    2 P1 columns x 4 pool positions x 16 maps per P1 row, weights w/127.5 * 2^s split into fp16
//    hi + lo: 6 MMAs per P1 row, the 2x2 pool cells of every map in one TMEM lane;
//  * layer 2 = implicit GEMM from shared memory, streamed: each P1 row (16 channels, fp16 hi and
//    lo planes, even / odd columns de-interleaved) is read once and feeds both P2 rows it
//    belongs to; K = 16 = the 16 channels of P1 column 2X + e (e = 0..3), N = 96 = {w hi, w lo}
//    x {P2 row u-1, u} x 4 pool positions x 6 maps for hi(A), N = 48 for lo(A): 8 MMAs per P1
//    row;
//  * layer 3 (C7x8) on tcgen05: K = 16 = P2 entry j+kx hi + lo, N = 32 = {w hi, w lo} x 8
//    kernel rows x 2 maps: the contributions of a P2 row to the 8 response rows it reaches,
//    summed by the data warps; layer 4 (1x1) and Eq. 1 on the FFMA pipe -> resp2.
// Warps 0-7 do the data work (two per TMEM lane quadrant: half 0 / 1 take maps 0-7 / 8-15 of
// the layer-1 epilogue, half 0 the layer-2 epilogue, half 1 layer 3 + 4); warp 8 allocates
// TMEM and issues every MMA (one elected lane), completion by tcgen05.commit -> mbarrier.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cuda_fp16.h>

#include "ccnn_internal.h"
#include "selective_common.cuh"
#include "tc05.cuh"

namespace ccnn {
namespace {

constexpr int NDW = 8;                         // data warps 0..7
constexpr int NPW = 8;                         // patch-preparation warps 9..16
constexpr int NPIPE = 32 * (NDW + 1);          // pipeline threads: data warps + the MMA warp (8)
constexpr int NT = NPIPE + 32 * NPW;           // + the preparation warps
constexpr uint32_t BAR_PIPE = 1, BAR_PREP = 2; // named barriers of the two groups
constexpr int NC = kSelTcCands;                // survivors per strip: 2 NC patch slots
constexpr int SL = 12;                         // TMEM lanes per patch slot (P2 columns 0..11)
constexpr int NQ = 12;                         // P2 rows of a patch (0..11)
constexpr int EP = 64;                         // bytes per patch row in shared memory
constexpr int ER = 56;                         // patch rows (55 + one zero row)
constexpr int PATCH_BYTES = ER * EP;
// shared memory (bytes)
constexpr int B1M = 128 * 16 * 2;              // one layer-1 B (N = 128, K = 16): [k chunk 2][n][8]
constexpr int B1_BYTES = 6 * B1M;              // [t = pair - P1 row 3][w part 2]
constexpr int B2M = 96 * 16 * 2;               // one layer-2 B (N = 96)
constexpr int B2_BYTES = 16 * B2M;             // [half parity 2][P1 row parity 2][column e 4]
constexpr int B3M = 32 * 16 * 2;               // one layer-3 B (N = 32)
constexpr int B3_BYTES = 7 * B3M;              // [kx 7]
static_assert((B1_BYTES + B2_BYTES + B3_BYTES) / 2 == kSelTcBmatHalves, "B matrix image size");
constexpr int P1_E = 132;                      // entries per (w part, parity, k chunk); 128 written
constexpr int P1_KC = P1_E * 16;               // k-chunk stride (LBO)
constexpr int P1_PAR = 2 * P1_KC;
constexpr int P1_HL = 2 * P1_PAR;
constexpr int P1_SLOT = 2 * P1_HL;
constexpr int P1_RING = 4;                     // P1 rows 2u .. 2u+3 live
constexpr int P2_E = 136;                      // P2 entries per (buffer, part): 128 written + reach
constexpr int P2_HL = P2_E * 16;
constexpr int P2_BUF = 2 * P2_HL;
struct Prep {                                  // per survivor of the strip being prepared
    uint32_t colx[64], rowy[64];               // O2 table entries of the patch columns / rows
    int hist[256];
    uint8_t lut[256];
    const uint8_t* data;                       // its frame
    int64_t pitch;
    int32_t w, h;
    sel::PatchRegion g;                        // O5 region
};
constexpr int OFF_B1 = 0, OFF_B2 = OFF_B1 + B1_BYTES, OFF_B3 = OFF_B2 + B2_BYTES;
constexpr int OFF_P1 = OFF_B3 + B3_BYTES;
constexpr int OFF_P2 = OFF_P1 + P1_RING * P1_SLOT;
constexpr int OFF_E = OFF_P2 + 2 * P2_BUF;    // two strips of patches (double buffer)
constexpr int OFF_PREP = OFF_E + 2 * NC * PATCH_BYTES;
constexpr int SMEM_BYTES = OFF_PREP + 2 * NC * (int)sizeof(Prep);   // geometry one strip ahead
static_assert(OFF_E % 16 == 0 && OFF_PREP % 16 == 0, "alignment");
static_assert(SMEM_BYTES <= 227 * 1024, "shared memory");
// TMEM columns (512 allocated: one CTA per SM)
constexpr uint32_t TM_A = 0;                   // A ring: image row slot s at +4 s (32 columns)
constexpr uint32_t TM_D1 = 32;                 // layer 1: P1 row 0 of the unit (128), row 1 (128)
constexpr uint32_t TM_D2 = 288;                // layer 2: [half 0 wh | half 1 wh | half 0 wl | half 1 wl]
constexpr uint32_t TM_D3 = 384;                // layer 3 (32)
constexpr uint32_t TM_COLS = 512;
constexpr uint32_t IDESC1 = tc05::idesc_f16(128, 128);
constexpr uint32_t IDESC2 = tc05::idesc_f16(128, 96);
constexpr uint32_t IDESC2_LO = tc05::idesc_f16(128, 48);
constexpr uint32_t IDESC3 = tc05::idesc_f16(128, 32);

// Eq. 1 on x' = 2x/3 (the factor is folded into the preceding scale / bias)
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
__device__ __forceinline__ float act1(float x)
{
    const float a2 = x * x;
    const float p = fmaf(a2, fmaf(a2, 1.41645f, 1.0f), fabsf(x) + 1.0f);
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(p));
    return copysignf(fmaf(-1.7159f, r, 1.7159f), x);
}
// byte -> exact fp16 (magic number 1024 + v, minus 1024), two pixels of `word` per call
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
// 32 lanes x 32 / 64 consecutive columns, one wait
__device__ __forceinline__ void ld32(uint32_t taddr, float (&v)[32])
{
    uint32_t r[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n\t"
        "tcgen05.wait::ld.sync.aligned;"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr) : "memory");
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void st_zero24(uint32_t taddr)
{
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%2,%2,%2,%2,%2,%2,%2,%2,%2,%2,%2,%2,%2,%2,%2,%2};\n\t"
        "tcgen05.st.sync.aligned.32x32b.x8.b32 [%1], {%2,%2,%2,%2,%2,%2,%2,%2};"
        :: "r"(taddr), "r"(taddr + 16u), "r"(0u) : "memory");
}

// patch preparation of the nc survivors c0 .. c0+nc-1 of a strip by the 128 threads of the
// preparation warps, in two parts: prep_geometry (O5 sampling tables of every patch column /
// row; run one strip ahead, while the previous strip's sampling is still to come) and prep_sample (O2
// sampling into the 56 x 64-B patch rows at ebuf -- pixel x of row y at byte y*64 + 4 + x --,
// histogram, O6 LUT, equalisation in place)
__device__ __forceinline__ void prep_geometry(int c0, int nc, const S1Cand* __restrict__ cands,
                                              const LevelInfo* __restrict__ lvinfo,
                                              const FrameInfo* __restrict__ frames, Prep* P)
{
    const int pt = (int)threadIdx.x - NPIPE;                  // 0 .. 32 NPW - 1
    if (pt < nc) {                                             // per survivor: region, frame
        const S1Cand cd = cands[c0 + pt];
        const LevelInfo& L = lvinfo[cd.level];
        const FrameInfo& F = frames[L.frame];
        Prep& Q = P[pt];
        Q.g = sel::patch_region(cd.ix, cd.iy, L.sigma);
        Q.data = F.data; Q.pitch = F.pitch; Q.w = F.w; Q.h = F.h;
    }
    tc05::named_sync(BAR_PREP, 32 * NPW);
    for (int i = pt; i < nc * (kPatchW + kPatchH); i += 32 * NPW) {
        const int c = i / (kPatchW + kPatchH), j = i - c * (kPatchW + kPatchH);
        Prep& Q = P[c];
        if (j < kPatchW) Q.colx[j] = sel::region_col(Q.g, j, Q.w);
        else Q.rowy[j - kPatchW] = sel::region_row(Q.g, j - kPatchW, Q.h);
    }
}

__device__ __forceinline__ void prep_sample(int nc, uint8_t* ebuf, Prep* P)
{
    const int pt = (int)threadIdx.x - NPIPE;                  // 0 .. 32 NPW - 1
    auto psync = [] { tc05::named_sync(BAR_PREP, 32 * NPW); };
    for (int i = pt; i < nc * 256; i += 32 * NPW) P[i >> 8].hist[i & 255] = 0;
    psync();
    // O2 sampling: thread = patch column u (pt & 63; 51 active) x row phase (pt >> 6) over the
    // strip's nc x 55 patch rows, 8 rows per pass so 32 byte gathers are in flight per thread
    // (the frames are in HBM: latency-bound otherwise)
    constexpr int RP = 32 * NPW / 64;                          // row phases
    const int u = pt & 63, rs = pt >> 6;
    const int nrows = nc * kPatchH;
    constexpr int RU = 4;
    for (int r0 = rs; r0 < nrows; r0 += RP * RU) {
        uint32_t px[RU][4], axy[RU];
        int off[RU], cc[RU];
#pragma unroll
        for (int j = 0; j < RU; ++j) {
            const int r = min(r0 + RP * j, nrows - 1);
            const int c = r / kPatchH, v = r - c * kPatchH;
            const Prep& Q = P[c];
            const uint32_t xt = Q.colx[min(u, kPatchW - 1)], yt = Q.rowy[v];
            const uint32_t x0 = xt & 0xFFFFu, y0 = yt & 0xFFFFu;
            const uint32_t x1 = min(x0 + 1u, (uint32_t)(Q.w - 1)), y1 = min(y0 + 1u, (uint32_t)(Q.h - 1));
            const uint8_t* q0 = Q.data + (int64_t)y0 * Q.pitch;
            const uint8_t* q1 = Q.data + (int64_t)y1 * Q.pitch;
#ifndef SELTC_NO_LOAD                                           // timing experiments only
            px[j][0] = __ldg(q0 + x0);
            px[j][1] = __ldg(q0 + x1);
            px[j][2] = __ldg(q1 + x0);
            px[j][3] = __ldg(q1 + x1);
#else
            px[j][0] = (uint32_t)(uintptr_t)q0 & 255u; px[j][1] = x1 & 255u; px[j][2] = y1 & 255u;
            px[j][3] = (uint32_t)(uintptr_t)q1 & 255u;
#endif
            axy[j] = (xt >> 16) | (yt & 0xFFFF0000u);
            off[j] = c * PATCH_BYTES + v * EP + 4 + u;
            cc[j] = c;
        }
#pragma unroll
        for (int j = 0; j < RU; ++j) {
            if (u < kPatchW && r0 + RP * j < nrows) {
                const uint32_t ax = axy[j] & 0xFFFFu, ay = axy[j] >> 16;
                const uint32_t top = px[j][0] * (2048u - ax) + px[j][1] * ax;
                const uint32_t bot = px[j][2] * (2048u - ax) + px[j][3] * ax;
                const uint32_t val = (top * (2048u - ay) + bot * ay + (1u << 21)) >> 22;
                ebuf[off[j]] = (uint8_t)val;
#ifndef SELTC_NO_HIST                                           // timing experiments only
                atomicAdd(&P[cc[j]].hist[val], 1);
#endif
            }
        }
    }
    psync();
    for (int c = pt >> 5; c < nc; c += NPW) sel::warp_lut(P[c].hist, P[c].lut);
    psync();
    // O6 applied in place, 4 pixels per word (rows 0..54; the pad bytes of a row only reach
    // discarded outputs): the data warps and the CNN3 copy then read E directly
    constexpr int RW = EP / 4;
    for (int i = pt; i < nc * kPatchH * RW; i += 32 * NPW) {
        const int c = i / (kPatchH * RW), k = i - c * (kPatchH * RW);
        uint32_t* w = reinterpret_cast<uint32_t*>(ebuf + c * PATCH_BYTES) + k;
        const uint8_t* lut = P[c].lut;
        const uint32_t x = *w;
        *w = (uint32_t)lut[x & 0xFFu] | ((uint32_t)lut[(x >> 8) & 0xFFu] << 8) |
             ((uint32_t)lut[(x >> 16) & 0xFFu] << 16) | ((uint32_t)lut[x >> 24] << 24);
    }
    psync();
}

// 72 registers (4 B of spill): 544 x 72 = 39k of the SM's 64k registers, so 5 CTAs of the next
// batch's pyramid keep running beside a CNN2 CTA (at the default 96, 2): the pyramid no longer
// stalls while the batch's tail holds the SMs -- C4 step 0.616 -> 0.601 ms (K3)
__global__ void __maxnreg__(72) selective_cnn2_tc_kernel(
    const __grid_constant__ Cnn2Tc K, const SelParams sp, const uint16_t* __restrict__ bmats,
    const FrameInfo* __restrict__ frames, const LevelInfo* __restrict__ lvinfo,
    const S1Cand* __restrict__ cands, const uint32_t cand_cap, float* __restrict__ resp2,
    uint8_t* __restrict__ epatch, Ctrl* __restrict__ ctrl)
{
    extern __shared__ __align__(128) uint8_t smem[];
    __shared__ int s_claim, s_strip[2], s_nc[2], s_k2[2][NC];
    __shared__ uint32_t s_tmem;
    __shared__ __align__(8) uint64_t bar_l1, bar_l1a, bar_l2, bar_l3, bar_full[2], bar_empty[2];

    const int tid = threadIdx.x;
    const int warp = __shfl_sync(0xFFFFFFFFu, tid >> 5, 0);   // provably warp-uniform
    const int lane = tid & 31;
    const bool mma_warp = warp == NDW;
    const bool prep_warp = warp > NDW;
    const int n_cand = (int)min(*(volatile uint32_t*)&ctrl->n_cand, cand_cap);
    const int n_strips = (n_cand + NC - 1) / NC;
    if ((int)blockIdx.x >= n_strips) return;                   // CTA-uniform, before any barrier

    // ---- one-time setup: B matrices to shared memory, zeroed plane padding ----
    {
        const uint4* src = reinterpret_cast<const uint4*>(bmats);
        uint4* dst = reinterpret_cast<uint4*>(smem + OFF_B1);
        for (int i = tid; i < (B1_BYTES + B2_BYTES + B3_BYTES) / 16; i += NT) dst[i] = src[i];
        uint4* z = reinterpret_cast<uint4*>(smem + OFF_P1);
        for (int i = tid; i < (OFF_E - OFF_P1) / 16; i += NT) z[i] = make_uint4(0, 0, 0, 0);
    }
    if (mma_warp) tc05::tmem_alloc(&s_tmem, TM_COLS);
    if (tid == 0) {
        tc05::mbar_init(&bar_l1, 1);
        tc05::mbar_init(&bar_l1a, 1);
        tc05::mbar_init(&bar_l2, 1);
        tc05::mbar_init(&bar_l3, 1);
        for (int b = 0; b < 2; ++b) {
            tc05::mbar_init(&bar_full[b], 32 * NPW);           // every preparation thread
            tc05::mbar_init(&bar_empty[b], NDW);               // one thread per data warp
        }
        tc05::mbar_fence_init();
    }
    tc05::fence_async_smem();
    tc05::fence_before();
    __syncthreads();
    tc05::fence_after();
    const uint32_t tm = s_tmem;
    uint32_t ph_l1 = 0, ph_l1a = 0, ph_l2 = 0, ph_l3 = 0;   // completed phases (waiting side's count)
    const uint32_t s_base = tc05::smem_u32(smem);

    const int qd = warp & 3, hf = (warp >> 2) & 1;
    const int m = 32 * qd + lane;                  // TMEM lane = strip column
    const uint32_t t_lane = (uint32_t)(32 * qd) << 16;
    const int slot = m / SL, xp = m - slot * SL;   // patch slot, P2 column within the patch

    if (prep_warp) {
        // ======================= patch-preparation warps =======================
        // producer of the two patch buffers: claims a strip, prepares its patches, publishes
        // them (bar_full), and reuses a buffer once the data warps released it (bar_empty);
        // a strip id < 0 ends the consumers' loop
        Prep* const PB = reinterpret_cast<Prep*>(smem + OFF_PREP);   // [2][NC]
        auto claim = [&](int& st, int& nc) {
            if (tid == NPIPE) s_claim = (int)atomicAdd(&ctrl->strip_next, 1u);
            tc05::named_sync(BAR_PREP, 32 * NPW);
            st = s_claim;
            nc = st < n_strips ? min(NC, n_cand - st * NC) : 0;
            tc05::named_sync(BAR_PREP, 32 * NPW);             // s_claim read by all
        };
        int st, nc;
        claim(st, nc);
        if (nc > 0) prep_geometry(st * NC, nc, cands, lvinfo, frames, PB);
        uint32_t uses[2] = {0u, 0u};
        for (int it = 0;; ++it) {
            const int b = it & 1;
            if (uses[b] > 0) tc05::mbar_wait(&bar_empty[b], (uses[b] - 1u) & 1u);
            ++uses[b];
            int st_n = -1, nc_n = 0;
            if (nc > 0) {
                claim(st_n, nc_n);                             // the next strip: geometry + L2
                if (nc_n > 0) prep_geometry(st_n * NC, nc_n, cands, lvinfo, frames, PB + (b ^ 1) * NC);
                tc05::named_sync(BAR_PREP, 32 * NPW);
#ifndef SELTC_SKIP_PREP                                         // timing experiments only
                prep_sample(nc, smem + OFF_E + b * NC * PATCH_BYTES, PB + b * NC);
#endif
            }
            if (tid == NPIPE) {
                s_strip[b] = nc > 0 ? st : -1;
                s_nc[b] = nc;
            }
            tc05::named_sync(BAR_PREP, 32 * NPW);              // patches and s_strip written
            tc05::mbar_arrive(&bar_full[b]);
            if (nc == 0) break;
            st = st_n;
            nc = nc_n;
        }
    }
    uint32_t uses[2] = {0u, 0u};
    for (int it = 0; !prep_warp; ++it) {
        const int b = it & 1;
        tc05::mbar_wait(&bar_full[b], uses[b] & 1u);
        ++uses[b];
        const int st = s_strip[b];
        if (st < 0) break;
        const int c0 = st * NC;
        const int nc = s_nc[b];
#ifdef SELTC_SKIP_PIPE                                          // timing experiments only
        if (!mma_warp) { __syncwarp(); if (lane == 0) tc05::mbar_arrive(&bar_empty[b]); }
        continue;
#endif

        if (!mma_warp) {
            // ============================ data warps ============================
            const bool slot_ok = slot < 2 * nc;
            const int orient = slot & 1;                       // 0 = E, 1 = M (mirror)
            const uint8_t* prow = smem + OFF_E + (b * NC + (slot >> 1)) * PATCH_BYTES;
            // image row r of this lane's patch: pixels 4X .. 4X+7 (X = xp) as two words of the
            // equalised patch E; the mirrored patch M(x) = E(50 - x) reverses the bytes of words
            // 11-X .. 13-X.  Pixel 51 (the pad) and the rows >= 55 reach only discarded outputs
            // (zero weights or invalid rows)
            auto fetch = [&](int r, uint32_t (&pw)[2]) {
                if (!slot_ok) { pw[0] = pw[1] = 0u; return; }
                const uint32_t* rw = reinterpret_cast<const uint32_t*>(prow + min(r, ER - 1) * EP);
                if (orient == 0) {
                    pw[0] = rw[xp + 1];
                    pw[1] = rw[xp + 2];
                } else {
                    const uint32_t a = rw[11 - xp], b = rw[12 - xp], c = rw[13 - xp];
                    pw[0] = __byte_perm(b, c, 0x3456);
                    pw[1] = __byte_perm(a, b, 0x3456);
                }
            };
            auto put = [&](int r, const uint32_t (&pw)[2]) {          // image row r -> ring slot r % 8
                tc05::st4(tm + t_lane + TM_A + 4 * (r & 7), h2_of(pw[0], 0x4140), h2_of(pw[0], 0x4342),
                          h2_of(pw[1], 0x4140), h2_of(pw[1], 0x4342));
            };
            // layer-1 epilogue of unit k, maps 8 hf .. 8 hf + 7: P1 rows 2k + rr, columns 2X + cx
            // -> k chunk hf of the P1 entries; accumulator column h*64 + cx*32 + pos*8 + j
            // waits for P1 row rr's MMAs (committed apart: bar_l1a row 0, bar_l1 both rows)
            auto l1_epilogue = [&](int k) {
#pragma unroll 1
                for (int rr = 0; rr < 2; ++rr) {
                    if (rr == 0) { tc05::mbar_wait(&bar_l1a, ph_l1a & 1); ++ph_l1a; }
                    else { tc05::mbar_wait(&bar_l1, ph_l1 & 1); ++ph_l1; }
                    tc05::fence_after();
                    const int slot1 = (2 * k + rr) % P1_RING;
#pragma unroll 1
                    for (int cx = 0; cx < 2; ++cx) {
                        float d[32];
                        ld32(tm + t_lane + TM_D1 + 128 * rr + 64 * hf + 32 * cx, d);
                        uint32_t hi[4], lo[4];
#pragma unroll
                        for (int c = 0; c < 4; ++c) {
                            float mx[2];
#pragma unroll
                            for (int e = 0; e < 2; ++e) {
                                const float* q = d + 2 * c + e;
                                mx[e] = fmaxf(fmaxf(q[0], q[8]), fmaxf(q[16], q[24]));
                            }
                            const float2 x = __ffma2_rn(make_float2(mx[0], mx[1]), make_float2(K.l1s, K.l1s),
                                                        make_float2(K.l1b[8 * hf + 2 * c], K.l1b[8 * hf + 2 * c + 1]));
                            split_h2(act2(x), hi[c], lo[c]);
                        }
                        uint8_t* e = smem + OFF_P1 + slot1 * P1_SLOT + cx * P1_PAR + hf * P1_KC + m * 16;
                        *reinterpret_cast<uint4*>(e) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
                        *reinterpret_cast<uint4*>(e + P1_HL) = make_uint4(lo[0], lo[1], lo[2], lo[3]);
                    }
                }
            };
            // layer-2 epilogue of P2 row q (TMEM half q & 1) -> P2 buffer q & 1 as fp16 hi / lo
            // entries (6 maps + 2 zero); the half is zeroed for P2 row q + 2
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
                    const float2 x = __ffma2_rn(make_float2(m0, m1), make_float2(K.l2s, K.l2s),
                                                make_float2(K.l2b[2 * c], K.l2b[2 * c + 1]));
                    split_h2(act2(x), hi[c], lo[c]);
                }
                uint8_t* e = smem + OFF_P2 + (q & 1) * P2_BUF + m * 16;
                *reinterpret_cast<uint4*>(e) = make_uint4(hi[0], hi[1], hi[2], 0u);
                *reinterpret_cast<uint4*>(e + P2_HL) = make_uint4(lo[0], lo[1], lo[2], 0u);
            };
            // layer 3 + 4 (warps of half 1): acc3[mm][i] = map mm of response row p - 7 + i
            float acc3[2][8];
#pragma unroll
            for (int mm = 0; mm < 2; ++mm)
#pragma unroll
                for (int i = 0; i < 8; ++i) acc3[mm][i] = 0.f;
            const bool e_col = slot_ok && xp < 5;
            float* const rout = resp2 + (int64_t)(c0 + (slot >> 1)) * 50 + orient * kResp + xp;
            auto l3_epilogue = [&](int p) {
                float d[32];
                ld32(tm + t_lane + TM_D3, d);
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    const int n = (7 - i) * 2;
                    const float2 c2 = __fadd2_rn(make_float2(d[n], d[n + 1]), make_float2(d[16 + n], d[17 + n]));
                    const float2 a2 = __fadd2_rn(make_float2(acc3[0][i], acc3[1][i]), c2);
                    acc3[0][i] = a2.x;
                    acc3[1][i] = a2.y;
                }
                const int o = p - 7;                           // finished response row
                const float2 a = act2(__ffma2_rn(make_float2(acc3[0][0], acc3[1][0]),
                                                 make_float2(K.l3s, K.l3s), make_float2(K.l3b[0], K.l3b[1])));
#pragma unroll
                for (int mm = 0; mm < 2; ++mm) {
#pragma unroll
                    for (int i = 0; i < 7; ++i) acc3[mm][i] = acc3[mm][i + 1];
                    acc3[mm][7] = 0.f;
                }
                const float r = act1(fmaf(K.w4[1], a.y, fmaf(K.w4[0], a.x, K.b4)));
                if (e_col && o >= 0 && o < 5) {
                    rout[o * 5] = r;
                    if (r > sp.T2a) atomicAdd(&s_k2[b][slot >> 1], 1);    // K2
                }
            };
            auto sync_for_mma = [&]() {
                tc05::fence_async_smem();
                tc05::fence_before();
                tc05::named_sync(BAR_PIPE, NPIPE);
            };

            // K2 counters of this buffer (last read two strips ago, before the previous strip's syncs)
            if (warp == 4 && lane < NC) s_k2[b][lane] = 0;
            // prologue: image rows 0..7 -> L1(0); rows 8..11 once unit 0 is drained; both
            // layer-2 halves zeroed before the first streamed MMAs.  The two warps of a lane
            // quadrant load the even / odd image rows.
            {
                uint32_t wv[4][2];
#pragma unroll
                for (int i = 0; i < 4; ++i) fetch(2 * i + hf, wv[i]);
#pragma unroll
                for (int i = 0; i < 4; ++i) put(2 * i + hf, wv[i]);
                tc05::st_wait();
                sync_for_mma();                                // -> L1(0)
                uint32_t wx[2][2];
#pragma unroll
                for (int i = 0; i < 2; ++i) fetch(8 + 2 * i + hf, wx[i]);
                l1_epilogue(0);
                if (hf == 0) {
                    st_zero24(tm + t_lane + TM_D2);
                    st_zero24(tm + t_lane + TM_D2 + 24);
                    st_zero24(tm + t_lane + TM_D2 + 48);
                    st_zero24(tm + t_lane + TM_D2 + 72);
                }
#pragma unroll
                for (int i = 0; i < 2; ++i) put(8 + 2 * i + hf, wx[i]);
                tc05::st_wait();
                sync_for_mma();                                // -> L1(1), L2s(0)
            }
#pragma unroll 1
            for (int q = 0; q <= NQ + 1; ++q) {
                const bool more = q + 2 <= NQ;                 // unit q+2 exists
                uint32_t wx[2][2];
                if (more) {
#pragma unroll
                    for (int i = 0; i < 2; ++i) fetch(4 * q + 12 + 2 * i + hf, wx[i]);
                }
                // the MMAs run in the order L1(q+1) [P1 row 0, then row 1], L2s(q), L3(q-2): the
                // largest epilogue (layer 1, all data warps) starts first, P1 row by P1 row, and
                // only the short layer-3 epilogue trails the last MMA
                if (q + 1 <= NQ) l1_epilogue(q + 1);
                if (q >= 2 && hf == 1) {
                    tc05::mbar_wait(&bar_l3, ph_l3 & 1); ++ph_l3;      // L3(q-2) done
                    tc05::fence_after();
                    l3_epilogue(q - 2);
                }
                if (q <= NQ && hf == 0) {
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
                    for (int i = 0; i < 2; ++i) put(4 * q + 12 + 2 * i + hf, wx[i]);
                }
                tc05::st_wait();
                sync_for_mma();                                // -> L1(q+2), L2s(q+1), L3(q-1)
            }
            // the equalised patches of the survivors the rule sends to CNN3 (K2 > 0 under Eq. 2,
            // K2 < T_nn under Eq. 3; P:99 / S:358) -> epatch, for selective.cu
            if (warp < nc) {
                const int k2 = *(volatile int*)&s_k2[b][warp];
                const bool need3 = sp.rule == 0 ? k2 > 0 : k2 < sp.Tnn;
                if (need3) {
                    const uint8_t* src = smem + OFF_E + (b * NC + warp) * PATCH_BYTES;
                    uint32_t* dst = reinterpret_cast<uint32_t*>(epatch + (int64_t)(c0 + warp) * kEPatchBytes);
                    for (int wi = lane; wi < kEPatchBytes / 4; wi += 32) {
                        uint32_t x = 0;
#pragma unroll
                        for (int q = 0; q < 4; ++q) {
                            const int k = min(4 * wi + q, kPatchN - 1);
                            const int v = k / kPatchW, u = k - v * kPatchW;
                            x |= (uint32_t)src[v * EP + 4 + u] << (8 * q);
                        }
                        dst[wi] = x;
                    }
                }
            }
            __syncwarp();
            if (lane == 0) tc05::mbar_arrive(&bar_empty[b]);   // this strip's patches are read
        } else {
            // ============================ MMA warp ============================
            const uint64_t bd1 = tc05::sdesc(s_base + OFF_B1, 128 * 16, 128);
            const uint64_t bd2 = tc05::sdesc(s_base + OFF_B2, 96 * 16, 128);
            const uint64_t ad2 = tc05::sdesc(s_base + OFF_P1, P1_KC, 128);
            const uint64_t bd3 = tc05::sdesc(s_base + OFF_B3, 32 * 16, 128);
            const uint64_t ad3 = tc05::sdesc(s_base + OFF_P2, P2_HL, 128);
            // layer 1 of unit k: P1 row rr from image-row pairs rr, rr+1, rr+2 of the unit's
            // 8-row ring (B depends on t = pair - rr), weight parts hi / lo
            auto issue_l1 = [&](int k) {
                if (tc05::elect_one()) {
#pragma unroll
                    for (int rr = 0; rr < 2; ++rr) {
#pragma unroll
                        for (int t = 0; t < 3; ++t)
#pragma unroll
                            for (int hl = 0; hl < 2; ++hl) {
                                const uint32_t a = tm + TM_A + 4 * ((4 * k + 2 * (rr + t)) & 7);
                                tc05::mma_f16_ts(tm + TM_D1 + 128 * rr, a,
                                                 bd1 + (uint64_t)(((t * 2 + hl) * B1M) >> 4), IDESC1,
                                                 (t | hl) != 0);
                            }
                        if (rr == 0) tc05::commit(&bar_l1a);
                    }
                    tc05::commit(&bar_l1);
                }
                __syncwarp();
            };
            // layer 2, streamed: the P1 rows of unit u (2u, 2u+1) into P2 row u-1 (kernel rows
            // dy 2, 3; TMEM half (u-1) & 1) and P2 row u (dy 0, 1; half u & 1)
            auto issue_l2s = [&](int u) {
                if (tc05::elect_one()) {
                    const int par = (u - 1) & 1;
#pragma unroll
                    for (int rp = 0; rp < 2; ++rp) {
                        const uint32_t slot_off = (uint32_t)(((2 * u + rp) % P1_RING) * P1_SLOT);
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            const uint64_t b = bd2 + (uint64_t)((((par * 2 + rp) * 4 + e) * B2M) >> 4);
                            const uint64_t a = ad2 + (uint64_t)((slot_off + (e & 1) * P1_PAR + (e >> 1) * 16) >> 4);
                            tc05::mma_f16(tm + TM_D2, a, b, IDESC2, 1u);
                            tc05::mma_f16(tm + TM_D2, a + (uint64_t)(P1_HL >> 4), b, IDESC2_LO, 1u);
                        }
                    }
                    tc05::commit(&bar_l2);
                }
                __syncwarp();
            };
            // layer 3 of P2 row p: row m = response column j, K = 16 = P2 entry j+kx hi + lo
            auto issue_l3 = [&](int p) {
                if (tc05::elect_one()) {
#pragma unroll
                    for (int kx = 0; kx < 7; ++kx) {
                        const uint64_t a = ad3 + (uint64_t)(((p & 1) * P2_BUF + kx * 16) >> 4);
                        const uint64_t b = bd3 + (uint64_t)((kx * B3M) >> 4);
                        tc05::mma_f16(tm + TM_D3, a, b, IDESC3, kx != 0);
                    }
                    tc05::commit(&bar_l3);
                }
                __syncwarp();
            };
            tc05::named_sync(BAR_PIPE, NPIPE);                 // rows 0..7 in TMEM
            tc05::fence_after();
            issue_l1(0);
            tc05::named_sync(BAR_PIPE, NPIPE);                 // rows 8..11, P1 rows 0, 1, D2 zeroed
            tc05::fence_after();
            issue_l1(1);
            issue_l2s(0);
#pragma unroll 1
            for (int q = 0; q <= NQ + 1; ++q) {
                tc05::named_sync(BAR_PIPE, NPIPE);
                tc05::fence_after();
                if (q + 2 <= NQ) issue_l1(q + 2);
                if (q + 1 <= NQ) issue_l2s(q + 1);
                if (q >= 1 && q <= NQ) issue_l3(q - 1);
            }
        }
    }
    tc05::fence_before();
    __syncthreads();
    tc05::fence_after();
    if (mma_warp) tc05::tmem_dealloc(tm, TM_COLS);
}

}  // namespace

// B matrices of the three tensor-core layers (fp16 bit patterns, the kernel's shared-memory
// image) and the epilogue constants.  K-major canonical layout of one B (N rows, K = 16):
// [k chunk 2][n N][8].  Weights are scaled by 2^s (max |w'| in [8, 16), fp16 hi / lo parts
// stay normal) and split w' = hi + lo.
int selective_tc_bmats(const Cnn2W& w, uint16_t* out, Cnn2Tc* consts)
{
    const int total = kSelTcBmatHalves;
    std::fill(out, out + total, (uint16_t)0);
    auto put = [&](uint16_t* mat, int N, int n, int kk, float v) {
        mat[(kk >> 3) * N * 8 + n * 8 + (kk & 7)] = __half_as_ushort(__float2half_rn(v));
    };
    auto split = [](float wp, int part) {
        const float hi = __half2float(__float2half_rn(wp));
        return part ? wp - hi : wp;
    };
    auto scale_exp = [](const float* v, int n) {
        double mx = 0.0;
        for (int k = 0; k < n; ++k) mx = std::max(mx, std::fabs((double)v[k]));
        return mx > 0.0 ? (int)std::floor(std::log2(mx)) : 0;
    };
    // layer 1: mat = t * 2 + part (t = image-row pair - P1 row of the unit); n = h*64 + cx*32 +
    // pos*8 + (o & 7), h = o >> 3; kk = e*8 + c: image row 2(rr + t) + e of the unit, pixel 4X + c
    // -> conv row 2 rr + py needs ky = 2t + e - py, conv column 4X + 2cx + px needs kx = c - 2cx - px
    const double sc1 = 1.0 / (double)w.l1_inv_scale;
    for (int t = 0; t < 3; ++t)
        for (int part = 0; part < 2; ++part)
            for (int o = 0; o < 16; ++o)
                for (int cx = 0; cx < 2; ++cx)
                    for (int pos = 0; pos < 4; ++pos)
                        for (int kk = 0; kk < 16; ++kk) {
                            const int py = pos >> 1, px = pos & 1, e = kk >> 3, c = kk & 7;
                            const int ky = 2 * t + e - py, kx = c - 2 * cx - px;
                            if (ky < 0 || ky > 3 || kx < 0 || kx > 3) continue;
                            const float wp = (float)((double)w.w1[o][ky * 4 + kx] / 127.5 * sc1);
                            put(out + (t * 2 + part) * (B1M / 2), 128, (o >> 3) * 64 + cx * 32 + pos * 8 + (o & 7),
                                kk, split(wp, part));
                        }
    // layer 2 (streamed): mat = (par * 2 + rp) * 4 + e for P1 row 2u + rp of unit u with P2 row
    // u-1 in TMEM half par (kernel row dy = 2 + rp) and P2 row u in half 1 - par (dy = rp);
    // n = wpart*48 + half*24 + pos*6 + o; kk = input channel of P1 column 2X + e
    uint16_t* out2 = out + B1_BYTES / 2;
    const int e2 = scale_exp(&w.w2[0][0][0], 6 * 16 * 9);
    const double sc2 = std::ldexp(1.0, 3 - e2);
    for (int par = 0; par < 2; ++par)
        for (int rp = 0; rp < 2; ++rp)
            for (int e = 0; e < 4; ++e)
                for (int wh = 0; wh < 2; ++wh)
                    for (int half = 0; half < 2; ++half) {
                        const int dy = half == par ? 2 + rp : rp;
                        for (int pos = 0; pos < 4; ++pos)
                            for (int o = 0; o < 6; ++o)
                                for (int ch = 0; ch < 16; ++ch) {
                                    const int py = pos >> 1, px = pos & 1;
                                    const int ky = dy - py, kx = e - px;
                                    if (ky < 0 || ky > 2 || kx < 0 || kx > 2) continue;
                                    const float wp = (float)((double)w.w2[o][ch][ky * 3 + kx] * sc2);
                                    put(out2 + ((par * 2 + rp) * 4 + e) * (B2M / 2), 96,
                                        wh * 48 + half * 24 + pos * 6 + o, ch, split(wp, wh));
                                }
                    }
    // layer 3: mat = kx; n = wpart*16 + ky*2 + mm (8 kernel rows); kk = A part * 8 + ch (A part 0
    // = the P2 entry's hi, 1 = its lo; lo(A) x lo(w) stays zero)
    uint16_t* out3 = out + (B1_BYTES + B2_BYTES) / 2;
    const int e3 = scale_exp(&w.w3[0][0][0], 2 * 6 * 56);
    const double sc3 = std::ldexp(1.0, 3 - e3);
    for (int kx = 0; kx < 7; ++kx)
        for (int wh = 0; wh < 2; ++wh)
            for (int ky = 0; ky < 8; ++ky)
                for (int mm = 0; mm < 2; ++mm)
                    for (int kk = 0; kk < 16; ++kk) {
                        const int ha = kk >> 3, ch = kk & 7;
                        if (ch >= 6 || (ha && wh)) continue;
                        const float wp = (float)((double)w.w3[mm][ch][ky * 7 + kx] * sc3);
                        put(out3 + kx * (B3M / 2), 32, wh * 16 + ky * 2 + mm, kk, split(wp, wh));
                    }
    // epilogue constants, x 2/3 (Eq. 1 is evaluated on x' = 2x/3)
    const double k23 = 2.0 / 3.0;
    consts->l1s = (float)(k23 * (double)w.l1_inv_scale);
    for (int o = 0; o < 16; ++o) consts->l1b[o] = (float)(k23 * (double)w.b1h[o]);
    consts->l2s = (float)(k23 * std::ldexp(1.0, e2 - 3));
    for (int o = 0; o < 6; ++o) consts->l2b[o] = (float)(k23 * (double)w.b2[o]);
    consts->l3s = (float)(k23 * std::ldexp(1.0, e3 - 3));
    for (int o = 0; o < 2; ++o) consts->l3b[o] = (float)(k23 * (double)w.b3[o]);
    for (int o = 0; o < 2; ++o) consts->w4[o] = (float)(k23 * (double)w.w4[o]);
    consts->b4 = (float)(k23 * (double)w.b4);
    return total;
}

void launch_selective_cnn2_tc(const Cnn2Tc& k, SelParams sp, const uint16_t* d_bmats,
                              const FrameInfo* d_frames, const LevelInfo* d_levels,
                              const S1Cand* cands, uint32_t cand_cap, float* resp2, uint8_t* epatch,
                              Ctrl* ctrl, int sm_count, cudaStream_t s)
{
    cudaFuncSetAttribute(selective_cnn2_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
    selective_cnn2_tc_kernel<<<sm_count, NT, SMEM_BYTES, s>>>(k, sp, d_bmats, d_frames, d_levels, cands,
                                                             cand_cap, resp2, epatch, ctrl);
}

}  // namespace ccnn
