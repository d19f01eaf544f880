// pyramid.cu -- image pyramid construction on sm_100a (DESIGN.md kernel K1).
//
// PAPER.md P:87 ("The first CNN densely scans in series each image of the pyramid"),
// P:121 (GPU pyramid), P:156 (minSize / scaleFactor); reading O2: every level is a
// bilinear resample of the ORIGINAL frame with half-pixel centres, clamp-to-edge and
// 11-bit fixed-point weights, so CPU and GPU levels are bit-identical.  The sampling
// coordinates (x0, ax) / (y0, ay) are IEEE-double geometry evaluated on the host
// (runtime.cu, -ffp-contract=off) and uploaded as packed tables; this kernel is pure
// integer arithmetic.
//
// Roofline: HBM-bound in principle (the frame read once + 1 B written per level pixel;
// DESIGN.md K1), in practice bound by the L1 / load-store path of the byte gathers.  Tiles of
// 128 output columns x 32 rows of one level, described by host-built descriptors grouped by
// kernel class (runtime.cu build_plan): grid.y = frame, grid.x = the most tiles any frame has
// in the class (surplus CTAs of smaller frames exit).
//  * gather class (sigma < 0.7; pyramid_gather4_kernel): warp w owns tile rows 8w .. 8w+7 and
//    lane l the columns l, l+32, l+64, l+96, so the per-row work (y-table decode, row offset,
//    weights) is shared by 4 pixels and every store instruction writes 32 consecutive bytes;
//    16 byte gathers per row are in flight before any blend;
//  * quad class (sigma >= 0.7, upscaled / mildly scaled levels): 4 adjacent columns per
//    thread, one 32-bit store per row (pyramid_quad_kernel);
//  * frames narrower or shorter than 2 px: the clamped form (pyramid_kernel<false>).
// The O2 blend is 6 integer multiply-adds.  Optional tld4 texture gathers (the 2x2 footprint
// in one instruction, hardware 2-D addressing -- the paper's texture pyramid) on
// request (CCNN_DEBUG_PYR_TEX): identical results, measured slower (tex_throttle-bound).
#include "ccnn_internal.h"

namespace ccnn {
namespace {

struct PyrTile {
    const LevelInfo* L;
    int xo, y_beg, nr;     // output column, first row, rows of this tile (<= kPyrTileRows)
};

// decode this CTA's tile (descriptor `first` + blockIdx.x of the frame's list); false if the
// thread has no column
__device__ __forceinline__ bool pyr_tile(const FrameInfo& F, const LevelInfo* __restrict__ lv,
                                         const uint32_t* __restrict__ tiles, int first, PyrTile& T)
{
    const uint32_t d = __ldg(tiles + F.tile_off + first + blockIdx.x);
    T.L = lv + F.level0 + (int)(d & 0xFFu);
    T.xo = (int)((d >> 8) & 0xFFu) * kPyrCols + threadIdx.x;
    T.y_beg = (int)(d >> 16) * kPyrTileRows;
    T.nr = min(kPyrTileRows, T.L->lh - T.y_beg);
    return T.xo < T.L->pitch;
}

// O2: ((p00 (2048-ax) + p01 ax) (2048-ay) + (p10 (2048-ax) + p11 ax) ay + 2^21) >> 22, as
// 6 integer multiply-adds (every partial sum < 2^31)
__device__ __forceinline__ uint8_t blend(int p00, int p01, int p10, int p11, int ax, int ay)
{
    const int top = p00 * (2048 - ax) + p01 * ax;
    const int bot = p10 * (2048 - ax) + p11 * ax;
    return (uint8_t)((top * (2048 - ay) + bot * ay + (1 << 21)) >> 22);
}

// predicated byte store (the blend above it runs unconditionally: no branch per pixel)
__device__ __forceinline__ void st_u8_if(uint8_t* p, uint32_t v, bool ok)
{
    asm volatile("{ .reg .pred q; setp.ne.b32 q, %2, 0; @q st.global.u8 [%0], %1; }"
                 :: "l"(p), "r"(v), "r"((uint32_t)ok) : "memory");
}

// the y-table entries of a row group: 16-B loads (the table is padded and aligned,
// runtime.cu build_plan), the same address across the CTA
__device__ __forceinline__ void load_rows(const uint32_t* __restrict__ yt, uint32_t (&ye)[kPyrRows])
{
    if constexpr (kPyrRows % 4 == 0) {
#pragma unroll
        for (int k = 0; k < kPyrRows / 4; ++k) {
            const uint4 a = __ldg(reinterpret_cast<const uint4*>(yt) + k);
            ye[4 * k + 0] = a.x; ye[4 * k + 1] = a.y; ye[4 * k + 2] = a.z; ye[4 * k + 3] = a.w;
        }
    } else {
#pragma unroll
        for (int k = 0; k < kPyrRows; ++k) ye[k] = __ldg(yt + k);
    }
}

// SAFE form for the mildly scaled levels (sigma >= kQuadSigma, e.g. the upscaled levels of
// small min_face): a thread owns 4 consecutive output columns xo .. xo+3 (one x-table load of
// 4 entries, one 32-bit store per row) of 8 rows; the CTA's 128 threads cover the same
// 128 x 32 tile as pyramid_kernel (lane -> column quad, warp -> 8-row group).  The row offset
// is shared by the 4 columns and 16 byte gathers are in flight before any blend: ~25
// instructions per pixel instead of ~35, for levels whose 4-column quads stay within a few
// source sectors per warp (at small sigma the lane stride 4/sigma multiplies the L1
// wavefronts per gather, and the one-column form wins; K1).
constexpr double kQuadSigma = kPyrQuadSigma;

__device__ __forceinline__ void quad_tile(const FrameInfo& F, const LevelInfo& L, int tx0, int ty0,
                                          uint8_t* __restrict__ levels, const uint32_t* __restrict__ tabs)
{
    const int pitch = L.pitch;
    const int xo = tx0 + 4 * (int)(threadIdx.x & 31);
    const int y_beg = ty0 + 8 * (int)(threadIdx.x >> 5);
    const int nr = min(8, L.lh - y_beg);
    if (xo >= pitch || nr <= 0) return;                  // pitch % 16 == 0: xo + 3 < pitch
    const uint4 xe = __ldg(reinterpret_cast<const uint4*>(tabs + L.tab_off + xo));
    const uint32_t xs[4] = {xe.x, xe.y, xe.z, xe.w};
    uint32_t ye[8];
    {
        const uint4* yt = reinterpret_cast<const uint4*>(tabs + L.tab_off + pitch + y_beg);
        const uint4 a = __ldg(yt), b = __ldg(yt + 1);   // padded to kPyrTileRows: no clamp
        ye[0] = a.x; ye[1] = a.y; ye[2] = a.z; ye[3] = a.w;
        ye[4] = b.x; ye[5] = b.y; ye[6] = b.z; ye[7] = b.w;
    }
    const uint32_t fp = (uint32_t)F.pitch;
    const uint8_t* __restrict__ src = F.data;
    uint8_t* dst = levels + L.offset + xo + (int64_t)y_beg * pitch;
#pragma unroll
    for (int h = 0; h < 8; h += 2) {
        int p[2][4][4];
#pragma unroll
        for (int r = 0; r < 2; ++r) {
            const uint32_t row0 = (ye[h + r] & 0xFFFFu) * fp;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const uint32_t o = row0 + (xs[k] & 0xFFFFu);
                p[r][k][0] = __ldg(src + o);
                p[r][k][1] = __ldg(src + o + 1u);
                p[r][k][2] = __ldg(src + o + fp);
                p[r][k][3] = __ldg(src + o + fp + 1u);
            }
        }
#pragma unroll
        for (int r = 0; r < 2; ++r) {
            const int ay = (int)(ye[h + r] >> 16);
            uint32_t w = 0;
#pragma unroll
            for (int k = 0; k < 4; ++k)
                w |= (uint32_t)blend(p[r][k][0], p[r][k][1], p[r][k][2], p[r][k][3], (int)(xs[k] >> 16), ay) << (8 * k);
            if (h + r < nr) *reinterpret_cast<uint32_t*>(dst + (int64_t)(h + r) * pitch) = w;
        }
    }
}

// the quad class: the tiles of the levels with sigma >= kQuadSigma (the last class of the list)
__global__ void __launch_bounds__(kPyrCols) pyramid_quad_kernel(
    const FrameInfo* __restrict__ frames, uint8_t* __restrict__ levels,
    const LevelInfo* __restrict__ lv, const uint32_t* __restrict__ tiles,
    const uint32_t* __restrict__ tabs)
{
    const FrameInfo F = frames[blockIdx.y];
    const int first = F.tiles_g;
    if ((int)blockIdx.x >= F.tiles - first) return;
    const uint32_t d = __ldg(tiles + F.tile_off + first + blockIdx.x);
    const LevelInfo& L = lv[F.level0 + (int)(d & 0xFFu)];
    quad_tile(F, L, (int)((d >> 8) & 0xFFu) * kPyrCols, (int)(d >> 16) * kPyrTileRows, levels, tabs);
}

// the gather class with clamped sampling (every tile of a frame narrower or shorter than 2 px:
// its tables do not encode the edge)
template <bool SAFE>
__global__ void __launch_bounds__(kPyrCols) pyramid_kernel(
    const FrameInfo* __restrict__ frames, uint8_t* __restrict__ levels,
    const LevelInfo* __restrict__ lv, const uint32_t* __restrict__ tiles,
    const uint32_t* __restrict__ tabs)
{
    const FrameInfo F = frames[blockIdx.y];
    if ((int)blockIdx.x >= F.tiles_g) return;
    PyrTile T;
    if (!pyr_tile(F, lv, tiles, 0, T)) return;
    const LevelInfo& L = *T.L;
    // SAFE (every frame W, H >= 2): the tables encode the edge so that i1 = i0 + 1 always
    // (runtime.cu sample_entry); otherwise the clamped form
    const uint32_t e = __ldg(tabs + L.tab_off + T.xo);          // padding = edge column
    const uint32_t x0 = e & 0xFFFFu;
    const uint32_t x1 = SAFE ? x0 + 1u : min(x0 + 1u, (uint32_t)(F.w - 1));
    const int ax = (int)(e >> 16);
    const int pitch = L.pitch;
    uint8_t* dst = levels + L.offset + T.xo + (int64_t)T.y_beg * pitch;
    const uint32_t* yt = tabs + L.tab_off + pitch + T.y_beg;   // padded: no clamp
    // frames are < 4 GB: 32-bit row offsets from this column's base pointer (SAFE: the
    // second row is one pitch further, the second column one byte)
    const uint32_t fp = (uint32_t)F.pitch;
    const uint8_t* __restrict__ col = F.data + x0;
    for (int g0 = 0; g0 < T.nr; g0 += kPyrRows) {             // CTA-uniform
        const int nr = T.nr - g0;
        uint32_t ye[kPyrRows];
        load_rows(yt + g0, ye);
        int p[kPyrRows][4];
#pragma unroll
        for (int r = 0; r < kPyrRows; ++r) {
            const uint32_t y0 = ye[r] & 0xFFFFu;
            if (SAFE) {
                const uint8_t* r0 = col + y0 * fp;
                const uint8_t* r1 = r0 + fp;
                p[r][0] = __ldg(r0);
                p[r][1] = __ldg(r0 + 1);
                p[r][2] = __ldg(r1);
                p[r][3] = __ldg(r1 + 1);
            } else {
                const uint32_t y1 = min(y0 + 1u, (uint32_t)(F.h - 1));
                const uint8_t* r0 = F.data + (int64_t)y0 * F.pitch;
                const uint8_t* r1 = F.data + (int64_t)y1 * F.pitch;
                p[r][0] = __ldg(r0 + x0);
                p[r][1] = __ldg(r0 + x1);
                p[r][2] = __ldg(r1 + x0);
                p[r][3] = __ldg(r1 + x1);
            }
        }
        uint8_t* d = dst + (int64_t)g0 * pitch;
        if (nr >= kPyrRows) {
#pragma unroll
            for (int r = 0; r < kPyrRows; ++r)
                d[r * pitch] = blend(p[r][0], p[r][1], p[r][2], p[r][3], ax, (int)(ye[r] >> 16));
        } else {
#pragma unroll
            for (int r = 0; r < kPyrRows; ++r)
                if (r < nr) d[r * pitch] = blend(p[r][0], p[r][1], p[r][2], p[r][3], ax, (int)(ye[r] >> 16));
        }
    }
}

// Thread mapping of the gather kernel (SAFE tables): warp w owns the tile rows
// 8w .. 8w+7, lane l the columns l, l+32, l+64, l+96 -- the per-row work (y-table decode, row
// offsets, weights) is shared by 4 pixels, and every store instruction of a warp writes 32
// consecutive bytes.  Columns at or past the level pitch (the last tile column) are clamped
// for the loads and not stored.
struct ColSet {
    uint32_t x0[4];            // source column of each of the 4 output columns
    int wa[4], wb[4];          // their x weights 2048 - ax, ax
    bool ok[4];                // column < pitch
};
__device__ __forceinline__ void load_cols(const uint32_t* __restrict__ xt, int tx0, int pitch, ColSet& C)
{
    const int lane = (int)(threadIdx.x & 31);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const int xo = tx0 + lane + 32 * k;
        C.ok[k] = xo < pitch;
        const uint32_t e = __ldg(xt + min(xo, pitch - 1));
        C.x0[k] = e & 0xFFFFu;
        C.wb[k] = (int)(e >> 16);
        C.wa[k] = 2048 - C.wb[k];
    }
}

// GATHER class, SAFE tables (W, H >= 2: x0 + 1, y0 + 1 always inside): 4 byte gathers per
// pixel from the frame through L1.  Register cap 48 (10 CTAs of 128 threads per SM; 56 uncapped),
// no spills: beside the resident stage-1 CTA (320 threads x 120 registers) or a CNN2 CTA (544 x
// 72) the register file holds 4 pyramid CTAs instead of 3 (56) -- and each keeps more loads in
// flight than at 40 registers (5 CTAs), which measured best: pipelined C4 step 0.650 (56) ->
// 0.616 (40) -> 0.605 ms (48) (K1)
#ifndef PYR_MINB
#define PYR_MINB 10
#endif
__global__ void __launch_bounds__(kPyrCols, PYR_MINB) pyramid_gather4_kernel(
    const FrameInfo* __restrict__ frames, uint8_t* __restrict__ levels,
    const LevelInfo* __restrict__ lv, const uint32_t* __restrict__ tiles,
    const uint32_t* __restrict__ tabs)
{
    const FrameInfo F = frames[blockIdx.y];
    if ((int)blockIdx.x >= F.tiles_g) return;
    const uint32_t d = __ldg(tiles + F.tile_off + blockIdx.x);
    const LevelInfo& L = lv[F.level0 + (int)(d & 0xFFu)];
    const int pitch = L.pitch;
    const int tx0 = (int)((d >> 8) & 0xFFu) * kPyrCols;
    const int ry = (int)(d >> 16) * kPyrTileRows + 8 * (int)(threadIdx.x >> 5);
    const int nrw = min(8, L.lh - ry);
    if (nrw <= 0) return;
    const uint32_t* __restrict__ xt = tabs + L.tab_off;
    ColSet C;
    load_cols(xt, tx0, pitch, C);
    uint32_t ye[8];
    {
        const uint4* yt = reinterpret_cast<const uint4*>(xt + pitch + ry);   // padded, aligned
        const uint4 a = __ldg(yt), b = __ldg(yt + 1);
        ye[0] = a.x; ye[1] = a.y; ye[2] = a.z; ye[3] = a.w;
        ye[4] = b.x; ye[5] = b.y; ye[6] = b.z; ye[7] = b.w;
    }
    const uint32_t fp = (uint32_t)F.pitch;
    const uint8_t* __restrict__ col[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) col[k] = F.data + C.x0[k];
    uint8_t* dst = levels + L.offset + tx0 + (int)(threadIdx.x & 31) + (int64_t)ry * pitch;
#pragma unroll
    for (int r = 0; r < 8; ++r) {
        if (r < nrw) {                                          // warp-uniform
            const uint32_t o = (ye[r] & 0xFFFFu) * fp;
            const int wd = (int)(ye[r] >> 16), wc = 2048 - wd;
            int p[4][4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const uint8_t* q0 = col[k] + o;
                const uint8_t* q1 = q0 + fp;
                p[k][0] = __ldg(q0);
                p[k][1] = __ldg(q0 + 1);
                p[k][2] = __ldg(q1);
                p[k][3] = __ldg(q1 + 1);
            }
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int top = p[k][0] * C.wa[k] + p[k][1] * C.wb[k];
                const int bot = p[k][2] * C.wa[k] + p[k][3] * C.wb[k];
                st_u8_if(dst + 32 * k, (uint32_t)((top * wc + bot * wd + (1 << 21)) >> 22), C.ok[k]);
            }
            dst += pitch;
        }
    }
}

// tld4 (texture gather, red channel) with an integer destination type: the four texels of
// the 2x2 footprint at unnormalised (u, v) as zero-extended u32 -- order (i0, j1), (i1, j1),
// (i1, j0), (i0, j0) for the footprint at (i0 + 1, j0 + 1); clamp addressing supplies
// i1 = min(i0 + 1, W - 1)
__device__ __forceinline__ void gather4(cudaTextureObject_t tex, float u, float v, uint32_t& a,
                                        uint32_t& b, uint32_t& c, uint32_t& d)
{
    asm volatile("tld4.r.2d.v4.u32.f32 {%0, %1, %2, %3}, [%4, {%5, %6}];"
                 : "=r"(a), "=r"(b), "=r"(c), "=r"(d)
                 : "l"(tex), "f"(u), "f"(v));
}

__global__ void __launch_bounds__(kPyrCols) pyramid_tex_kernel(
    const FrameInfo* __restrict__ frames, uint8_t* __restrict__ levels,
    const LevelInfo* __restrict__ lv, const uint32_t* __restrict__ tiles,
    const uint32_t* __restrict__ tabs)
{
    const FrameInfo F = frames[blockIdx.y];
    if ((int)blockIdx.x >= F.tiles) return;
    PyrTile T;
    if (!pyr_tile(F, lv, tiles, 0, T)) return;
    const LevelInfo& L = *T.L;
    const uint32_t e = __ldg(tabs + L.tab_off + T.xo);
    const float u = (float)(e & 0xFFFFu) + 1.0f;
    const int ax = (int)(e >> 16);
    const cudaTextureObject_t tex = (cudaTextureObject_t)F.tex;
    const int pitch = L.pitch;
    uint8_t* dst = levels + L.offset + T.xo + (int64_t)T.y_beg * pitch;
    const uint32_t* yt = tabs + L.tab_off + pitch + T.y_beg;
    for (int g0 = 0; g0 < T.nr; g0 += kPyrRows) {             // CTA-uniform
        const int nr = T.nr - g0;
        uint32_t ye[kPyrRows];
        load_rows(yt + g0, ye);
        uint32_t q[kPyrRows][4];
#pragma unroll
        for (int r = 0; r < kPyrRows; ++r)
            gather4(tex, u, (float)(ye[r] & 0xFFFFu) + 1.0f, q[r][0], q[r][1], q[r][2], q[r][3]);
        uint8_t* d = dst + (int64_t)g0 * pitch;
        if (nr >= kPyrRows) {
#pragma unroll
            for (int r = 0; r < kPyrRows; ++r)
                d[r * pitch] = blend(q[r][3], q[r][2], q[r][0], q[r][1], ax, (int)(ye[r] >> 16));
        } else {
#pragma unroll
            for (int r = 0; r < kPyrRows; ++r)
                if (r < nr) d[r * pitch] = blend(q[r][3], q[r][2], q[r][0], q[r][1], ax, (int)(ye[r] >> 16));
        }
    }
}

}  // namespace

int launch_pyramid(const FrameInfo* d_frames, int n_frames, int max_tiles, const int (&max_class)[kPyrClasses],
                   bool safe, bool use_tex, uint8_t* levels, const LevelInfo* d_levels,
                   const uint32_t* d_tiles, const uint32_t* d_tabs, cudaStream_t s)
{
    if (n_frames <= 0 || max_tiles <= 0) return 0;
    if (use_tex) {                             // every tile by texture gathers (debug form)
        pyramid_tex_kernel<<<dim3(max_tiles, n_frames), kPyrCols, 0, s>>>(d_frames, levels, d_levels,
                                                                          d_tiles, d_tabs);
        return 1;
    }
    int launched = 0;
    // grid.x = the most tiles any frame has in the class (frames with fewer: surplus CTAs exit)
    if (max_class[kPyrGather] > 0) {
        const dim3 grid(max_class[kPyrGather], n_frames);
        if (safe)
            pyramid_gather4_kernel<<<grid, kPyrCols, 0, s>>>(d_frames, levels, d_levels, d_tiles, d_tabs);
        else
            pyramid_kernel<false><<<grid, kPyrCols, 0, s>>>(d_frames, levels, d_levels, d_tiles, d_tabs);
        ++launched;
    }
    if (max_class[kPyrQuad] > 0) {
        pyramid_quad_kernel<<<dim3(max_class[kPyrQuad], n_frames), kPyrCols, 0, s>>>(
            d_frames, levels, d_levels, d_tiles, d_tabs);
        ++launched;
    }
    return launched;
}

}  // namespace ccnn
