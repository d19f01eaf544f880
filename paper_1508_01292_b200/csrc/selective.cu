// selective.cu -- the selective unit: stage 2/3 on every stage-1 survivor (K3).
//
// PAPER.md §3.3: "the analyzed region is read from the original grayscale image
// together with certain neighborhood and scaled to the size of 51x55 pixels.  Then, the
// equalization of its histogram and mirror reflection with respect to the vertical axis
// are carried out" ... "The output of each CNN is a response map with a 5x5 size" ...
// K = number of responses exceeding T2; Eq. 2 (strict) with the early stop of
// P:99, or Eq. 3 (weak).  Readings O5-O8 fix the neighbourhood
// (51/35 x 55/39 about the window centre), the fixed-point bilinear sampling, the
// round-half-up equalisation, K pooled over both orientations and the raw box.
//
// B200 design: a persistent kernel (grid = SMs x 2) drains the survivor queue with a
// dynamic atomic counter -- the on-device form of the paper's asynchronous selective unit
// (P:125-131).  One 288-thread CTA per candidate:
//  * patch geometry in IEEE double with explicit _rn intrinsics (never contracted,
//    bit-identical to the oracle); integer sampling, histogram and equalisation;
//  * only the equalised patch E is stored; the mirrored orientation M(x,y) = E(50-x,y)
//    is read through mirrored addresses by layer 1 (no second image, no flipped weights);
//  * every layer's work is split over data (orientation x position [x map half]) so the
//    weights a warp uses are warp-uniform constant-bank kernel parameters; planes are
//    stored even/odd column de-interleaved so the stride-2 reads are conflict-free;
//  * CNN3 runs only when the rule needs it (P:99 early stop).
#include <type_traits>

#include "ccnn_internal.h"
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

// O2 sample coordinate: clamp to [0, n-1], i0 = floor(s), a = floor((s - i0)*2048 + 0.5)
__device__ __forceinline__ uint32_t bilin_coord(double s, int n)
{
    if (s < 0.0) s = 0.0;
    const double hi = (double)(n - 1);
    if (s > hi) s = hi;
    const double f = floor(s);
    const int a = (int)floor(__dadd_rn(__dmul_rn(__dsub_rn(s, f), 2048.0), 0.5));
    return (uint32_t)(int)f | ((uint32_t)a << 16);
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
constexpr size_t kP1Floats = 2 * 8 * kP1MS;    // pooled layer 1, one chunk of 8 maps: [orient][map][y][row]

// E(x, y) normalised (O3), for the FFMA layer 1 of CNN3
__device__ __forceinline__ float img_at(const SelSmem& sm, int y, int x)
{
    const __half h = reinterpret_cast<const __half*>(&sm.eh[y][0])[x];
    return fmaf(__half2float(h), 1.0f / 127.5f, -1.0f);
}

__device__ __forceinline__ void mma16816(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2,
                                         uint32_t a3, uint32_t b0, uint32_t b1)
{
    asm("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

// A-fragment pair of one input row for MMA rows m (conv column x = xb + 2m) and m + 8
// (x + 1), taps (kx0, kx0 + 1) with kx0 = 2 kb: E orientation -> pixels (x + kx0, +1) and
// (x + 1 + kx0, +1); mirrored M(x) = E(50 - x) -> the same pairs reversed.  Two word loads.
__device__ __forceinline__ void a_pair(const uint32_t* row, int o, int xb, int mg, int kb,
                                       uint32_t& am, uint32_t& am8)
{
    if (o == 0) {
        const int j = (xb >> 1) + mg + kb;
        const uint32_t w0 = row[j], w1 = row[j + 1];
        am = w0;
        am8 = __byte_perm(w0, w1, 0x5432);
    } else {
        const int j = 24 - (xb >> 1) - mg - kb;
        const uint32_t w0 = row[j], w1 = row[j + 1];
        am = __byte_perm(w0, w1, 0x3254);
        am8 = __byte_perm(w0, w0, 0x1032);
    }
}

// One selective CNN (architecture R: C4x4 1->A, P, C3x3 A->B, P, C7x8 B->C, C1x1 C->1,
// Eq. 1 after every conv) on both orientations: 51x55 -> 2 x 5x5 responses in sm.resp.
template <int A, int B, int C>
__device__ void run_net(const SelNetW<A, B, C>& W, SelSmem& sm, float* p1)
{
    const int tid = threadIdx.x;
    // layers 1-2 in chunks of AC input maps: P1 holds one chunk (both orientations), layer 2
    // accumulates over the chunks in registers -- half the P1 smem of CNN2, so 3 CTAs fit
    constexpr int AC = (A == 16) ? 8 : A;
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
    if constexpr (A == 16) {
    // ---- layer 1 on the tensor cores (mma.sync m16n8k16): tile = 16 conv-1 outputs of one
    //      conv row (MMA rows m / m+8 = columns xb+2m / xb+2m+1) x 16 taps of raw equalised
    //      pixels (exact in fp16), N = the chunk's 8 maps; weights / 127.5 * 2^s in fp16
    //      hi + lo (two MMAs), bias and 2^-s after the pooling max.  A tile pair (conv rows
    //      2py, 2py+1) holds whole pool cells per thread; 2 orient. x 26 rows x 3 column
    //      groups = 156 pairs over the 9 warps ----
        const int lane = tid & 31, warp = tid >> 5;
        const int c4 = lane & 3, mg = lane >> 2, kb = c4 & 1, ky0 = c4 >> 1;
        const uint32_t bh0 = W.l1frag[0][ch][lane][0], bh1 = W.l1frag[0][ch][lane][1];
        const uint32_t bl0 = W.l1frag[1][ch][lane][0], bl1 = W.l1frag[1][ch][lane][1];
        const float bias0 = W.b1h[8 * ch + 2 * c4], bias1 = W.b1h[8 * ch + 2 * c4 + 1];
        for (int pi = warp; pi < 156; pi += kSelThreads / 32) {
            const int o = pi / 78, rr = pi - o * 78, py = rr / 3, xb = 16 * (rr - 3 * py);
            const uint32_t* r0 = &sm.eh[2 * py + ky0][0];
            uint32_t a0, a1, a2, a3, e0, e1, e2, e3;
            a_pair(r0, o, xb, mg, kb, a0, a1);                 // conv row 2py: rows 2py+ky
            a_pair(r0 + 2 * kEW, o, xb, mg, kb, a2, a3);
            a_pair(r0 + kEW, o, xb, mg, kb, e0, e1);           // conv row 2py+1
            a_pair(r0 + 3 * kEW, o, xb, mg, kb, e2, e3);
            const int px = (xb >> 1) + mg;                     // pooled column
            const int col = (px & 1) ? kP1Odd + (px >> 1) : (px >> 1);
            float dA[4] = {0.f, 0.f, 0.f, 0.f}, dB[4] = {0.f, 0.f, 0.f, 0.f};
            mma16816(dA, a0, a1, a2, a3, bh0, bh1);
            mma16816(dB, e0, e1, e2, e3, bh0, bh1);
            mma16816(dA, a0, a1, a2, a3, bl0, bl1);
            mma16816(dB, e0, e1, e2, e3, bl0, bl1);
            const float m0 = fmaxf(fmaxf(dA[0], dA[2]), fmaxf(dB[0], dB[2]));
            const float m1 = fmaxf(fmaxf(dA[1], dA[3]), fmaxf(dB[1], dB[3]));
            float* const dst = p1 + (o * AC + 2 * c4) * kP1MS + py * kP1RS + col;
            dst[0] = act(fmaf(m0, W.l1_inv_scale, bias0));
            dst[kP1MS] = act(fmaf(m1, W.l1_inv_scale, bias1));
        }
    } else {
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
    const __grid_constant__ Cnn2W W2, const __grid_constant__ Cnn3W W3, const SelParams sp,
    const FrameInfo* __restrict__ frames, const LevelInfo* __restrict__ lvinfo,
    const S1Cand* __restrict__ cands, const uint32_t cand_cap, SelOut* __restrict__ out,
    float* __restrict__ dbg_resp, AccBox* __restrict__ acc, Ctrl* __restrict__ ctrl)
{
    extern __shared__ __align__(16) unsigned char sraw[];
    SelSmem& sm = *reinterpret_cast<SelSmem*>(sraw);
    float* const p1 = reinterpret_cast<float*>(sraw + ((sizeof(SelSmem) + 15) & ~size_t(15)));
    const int tid = threadIdx.x;
    const uint32_t n_cand = min(*(volatile uint32_t*)&ctrl->n_cand, cand_cap);

    for (;;) {
        if (tid == 0) sm.cand = (int)atomicAdd(&ctrl->sel_next, 1u);
        __syncthreads();
        const int ci = sm.cand;
        if ((uint32_t)ci >= n_cand) break;
        const S1Cand cd = cands[ci];
        const double sigma = lvinfo[cd.level].sigma;
        const FrameInfo F = frames[lvinfo[cd.level].frame];
        const uint8_t* frame = F.data;
        const int64_t pitch = F.pitch;
        const int Wd = F.w, Hd = F.h;

        // ---- O5 patch geometry, IEEE double, never contracted (bit-identical to the oracle)
        if (tid < kPatchW + kPatchH) {
            const double cx = __ddiv_rn(__dadd_rn((double)(4 * cd.ix), 13.5), sigma);
            const double cy = __ddiv_rn(__dadd_rn((double)(4 * cd.iy), 15.5), sigma);
            const double rw = __ddiv_rn(__ddiv_rn(1377.0, 35.0), sigma);   // 27*51/35
            const double rh = __ddiv_rn(__ddiv_rn(1705.0, 39.0), sigma);   // 31*55/39
            if (tid < kPatchW) {
                const double rx = __dsub_rn(cx, __ddiv_rn(rw, 2.0));
                const double t = __ddiv_rn(__dmul_rn(__dadd_rn((double)tid, 0.5), rw), 51.0);
                sm.colx[tid] = bilin_coord(__dsub_rn(__dadd_rn(rx, t), 0.5), Wd);
            } else {
                const int v = tid - kPatchW;
                const double ry = __dsub_rn(cy, __ddiv_rn(rh, 2.0));
                const double t = __ddiv_rn(__dmul_rn(__dadd_rn((double)v, 0.5), rh), 55.0);
                sm.rowy[v] = bilin_coord(__dsub_rn(__dadd_rn(ry, t), 0.5), Hd);
            }
        }
        if (tid < 256) sm.hist[tid] = 0;
        __syncthreads();
        // ---- O2 fixed-point bilinear sampling from the ORIGINAL frame + histogram; 4 pixels
        //      per thread per pass so their gathers are in flight together ----
        for (int k0 = tid; k0 < kPatchN; k0 += 4 * kSelThreads) {
            uint32_t px[4][4], axy[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int k = min(k0 + u * kSelThreads, kPatchN - 1);
                const int v = k / kPatchW, uu = k - v * kPatchW;
                const uint32_t xt = sm.colx[uu], yt = sm.rowy[v];
                const uint32_t x0 = xt & 0xFFFFu, y0 = yt & 0xFFFFu;
                const uint32_t x1 = min(x0 + 1u, (uint32_t)(Wd - 1)), y1 = min(y0 + 1u, (uint32_t)(Hd - 1));
                const uint8_t* r0 = frame + (int64_t)y0 * pitch;
                const uint8_t* r1 = frame + (int64_t)y1 * pitch;
                px[u][0] = __ldg(r0 + x0);
                px[u][1] = __ldg(r0 + x1);
                px[u][2] = __ldg(r1 + x0);
                px[u][3] = __ldg(r1 + x1);
                axy[u] = (xt >> 16) | (yt & 0xFFFF0000u);
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int k = k0 + u * kSelThreads;
                if (k >= kPatchN) break;
                const uint32_t ax = axy[u] & 0xFFFFu, ay = axy[u] >> 16;
                const uint32_t top = px[u][0] * (2048u - ax) + px[u][1] * ax;
                const uint32_t bot = px[u][2] * (2048u - ax) + px[u][3] * ax;
                const uint32_t val = (top * (2048u - ay) + bot * ay + (1u << 21)) >> 22;
                sm.patch[k] = (uint8_t)val;
                atomicAdd(&sm.hist[val], 1);
            }
        }
        __syncthreads();
        // ---- O6 histogram equalisation LUT (round half up), warp 0 ----
        if (tid < 32) {
            int h[8], run = 0;
#pragma unroll
            for (int k = 0; k < 8; ++k) { run += sm.hist[tid * 8 + k]; h[k] = run; }
            int incl = run;                               // inclusive scan of lane totals
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const int t = __shfl_up_sync(0xFFFFFFFFu, incl, d);
                if (tid >= d) incl += t;
            }
            const int excl = incl - run;
            // cdf_min = cdf at the smallest occupied value = count of that value
            int first = 256;
#pragma unroll
            for (int k = 7; k >= 0; --k) if (sm.hist[tid * 8 + k] > 0) first = tid * 8 + k;
#pragma unroll
            for (int d = 16; d >= 1; d >>= 1) first = min(first, __shfl_xor_sync(0xFFFFFFFFu, first, d));
            const int cmin = sm.hist[first];
            const int N = kPatchN;
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const int v = tid * 8 + k;
                const int cdf = excl + h[k];
                sm.lut[v] = (N == cmin) ? (uint8_t)v
                          : (uint8_t)((2 * 255 * (cdf - cmin) + (N - cmin)) / (2 * (N - cmin)));
            }
        }
        __syncthreads();
        // ---- E as fp16 pixel pairs (raw equalised values; O3 is applied by the layers) ----
        for (int k = tid; k < kPatchH * 26; k += kSelThreads) {
            const int v = k / 26, j = k - v * 26;
            const uint32_t p0 = sm.lut[sm.patch[v * kPatchW + 2 * j]];
            const uint32_t p1v = (2 * j + 1 < kPatchW) ? sm.lut[sm.patch[v * kPatchW + 2 * j + 1]] : 0u;
            const __half2 h = __floats2half2_rn((float)p0, (float)p1v);
            sm.eh[v][j] = *reinterpret_cast<const uint32_t*>(&h);
        }
        __syncthreads();

        // ---- CNN2 on both orientations, K2 ----
        run_net<16, 6, 2>(W2, sm, p1);
        float r2v = 0.f, r3v = 0.f;
        if (tid < 2 * kResp) r2v = sm.resp[tid / kResp][tid % kResp];
        const int K2 = __syncthreads_count(tid < 2 * kResp && r2v > sp.T2a);
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
        const bool stop = (sp.rule == 0) ? (K2 == 0) : (K2 >= sp.Tnn);   // P:99 / S:358
        int K3 = 0, delta, ran3 = 0;
        float best;
        if (stop) {
            delta = (sp.rule == 0) ? 0 : 1;
            best = block_max(r2v);
        } else {
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
            // O8 raw box: the window mapped back to original pixels, round half up
            SelOut so;
            so.K2 = K2; so.K3 = K3; so.delta = delta; so.cnn3_ran = ran3; so.score = best;
            so.bx = (int)floor(__dadd_rn(__ddiv_rn((double)(4 * cd.ix), sigma), 0.5));
            so.by = (int)floor(__dadd_rn(__ddiv_rn((double)(4 * cd.iy), sigma), 0.5));
            so.bw = (int)floor(__dadd_rn(__ddiv_rn(27.0, sigma), 0.5));
            so.bh = (int)floor(__dadd_rn(__ddiv_rn(31.0, sigma), 0.5));
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

void launch_selective(const Cnn2W& w2, const Cnn3W& w3, SelParams sp, const FrameInfo* d_frames,
                      const LevelInfo* d_levels, const S1Cand* cands, uint32_t cand_cap, SelOut* out,
                      float* dbg_resp, AccBox* acc, Ctrl* ctrl, int sm_count, cudaStream_t s)
{
    const size_t smem = selective_smem_bytes();
    cudaFuncSetAttribute(selective_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, selective_kernel, kSelThreads, smem);
    if (occ < 1) occ = 1;
    selective_kernel<<<sm_count * occ, kSelThreads, smem, s>>>(w2, w3, sp, d_frames, d_levels, cands,
                                                              cand_cap, out, dbg_resp, acc, ctrl);
}

}  // namespace ccnn
