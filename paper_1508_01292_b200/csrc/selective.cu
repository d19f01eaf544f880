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
// B200 design: a persistent kernel (grid = SMs x occupancy) drains the survivor queue
// with a dynamic atomic counter -- the on-device form of the paper's asynchronous
// selective unit.  One CTA per candidate: patch geometry in IEEE double
// (explicit _rn intrinsics: never contracted, bit-identical to the oracle), integer
// sampling/histogram/equalisation, then both orientations of CNN2 (and CNN3 when the
// rule needs it) in fp32 with weights as constant-bank kernel parameters.
#include <type_traits>

#include "ccnn_internal.h"

namespace ccnn {
namespace {

constexpr int kSelThreads = 256;
constexpr int kImgW = 52;                   // padded 51-wide patch rows

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
    float img[2][kPatchH][kImgW];           // E and mirrored M, normalised (O3)
    float p2[2][6][12][11];                 // pooled layer 2 (B <= 6 maps) [orient][map][y][x]
    float resp[2][kResp];
    float wmax[kSelThreads / 32];
    int cand;
};

// pooled layer 1 lives after SelSmem: [2][A][26][24]
template <int A>
constexpr int p1_floats() { return 2 * A * 26 * 24; }

// One selective CNN (architecture R: C4x4 1->A, P, C3x3 A->B, P, C7x8 B->C, C1x1 C->1,
// Eq. 1 after every conv) on both orientations: 51x55 -> 2 x 5x5 responses in sm.resp.
template <int A, int B, int C>
__device__ void run_net(const SelNetW<A, B, C>& W, SelSmem& sm, float* p1)
{
    const int tid = threadIdx.x;
    // ---- layer 1: conv4x4 1->A, pool, act -> p1[o][a][26][24]; item = pooled position ----
    for (int it = tid; it < 2 * 26 * 24; it += kSelThreads) {
        const int o = it / (26 * 24), rem = it % (26 * 24), py0 = rem / 24, px0 = rem % 24;
        float x[5][5];
#pragma unroll
        for (int r = 0; r < 5; ++r)
#pragma unroll
            for (int c = 0; c < 5; ++c) x[r][c] = sm.img[o][2 * py0 + r][2 * px0 + c];
#pragma unroll
        for (int a = 0; a < A; ++a) {
            float m = -INFINITY;
#pragma unroll
            for (int py = 0; py < 2; ++py)
#pragma unroll
                for (int px = 0; px < 2; ++px) {
                    float s = W.b1[a];
#pragma unroll
                    for (int ky = 0; ky < 4; ++ky)
#pragma unroll
                        for (int kx = 0; kx < 4; ++kx)
                            s = fmaf(W.w1[a][ky * 4 + kx], x[py + ky][px + kx], s);
                    m = fmaxf(m, s);
                }
            p1[((o * A + a) * 26 + py0) * 24 + px0] = act(m);   // pool then act (monotone)
        }
    }
    __syncthreads();
    // ---- layer 2: conv3x3 A->B, pool, act -> p2[o][b][12][11]; item = (map pair, position) ----
    constexpr int G = (B >= 2) ? 2 : 1, NG = B / G;
    static_assert(B % G == 0, "map groups");
    for (int it = tid; it < NG * 2 * 12 * 11; it += kSelThreads) {
        const int g = it / (2 * 12 * 11), rem = it % (2 * 12 * 11);
        const int o = rem / 132, pos = rem % 132, py0 = pos / 11, px0 = pos % 11;
        auto body = [&](auto Bc) {
            constexpr int B0 = decltype(Bc)::value;
            float s[G][4];
#pragma unroll
            for (int b = 0; b < G; ++b)
#pragma unroll
                for (int k = 0; k < 4; ++k) s[b][k] = W.b2[B0 + b];
#pragma unroll
            for (int a = 0; a < A; ++a) {
                const float* in = p1 + ((o * A + a) * 26 + 2 * py0) * 24 + 2 * px0;
                float v[4][4];
#pragma unroll
                for (int r = 0; r < 4; ++r)
#pragma unroll
                    for (int c = 0; c < 4; ++c) v[r][c] = in[r * 24 + c];
#pragma unroll
                for (int b = 0; b < G; ++b)
#pragma unroll
                    for (int py = 0; py < 2; ++py)
#pragma unroll
                        for (int px = 0; px < 2; ++px)
#pragma unroll
                            for (int ky = 0; ky < 3; ++ky)
#pragma unroll
                                for (int kx = 0; kx < 3; ++kx)
                                    s[b][py * 2 + px] = fmaf(W.w2[B0 + b][a][ky * 3 + kx],
                                                             v[py + ky][px + kx], s[b][py * 2 + px]);
            }
#pragma unroll
            for (int b = 0; b < G; ++b)
                sm.p2[o][B0 + b][py0][px0] =
                    act(fmaxf(fmaxf(s[b][0], s[b][1]), fmaxf(s[b][2], s[b][3])));
        };
        if constexpr (NG == 1) body(std::integral_constant<int, 0>{});
        else if constexpr (NG == 3) {
            if (g == 0) body(std::integral_constant<int, 0>{});
            else if (g == 1) body(std::integral_constant<int, 2>{});
            else body(std::integral_constant<int, 4>{});
        } else {
            static_assert(NG == 1 || NG == 3, "unsupported B");
        }
    }
    __syncthreads();
    // ---- layer 3 (C7x8 B->C, act) + layer 4 (C1x1 C->1, act); item = (orientation, cell) ----
    if (tid < 2 * kResp) {
        const int o = tid / kResp, cell = tid % kResp, y = cell / 5, x = cell % 5;
        float r = W.b4;
#pragma unroll 1
        for (int c = 0; c < C; ++c) {
            float s = W.b3[c];
#pragma unroll
            for (int b = 0; b < B; ++b)
#pragma unroll
                for (int ky = 0; ky < 8; ++ky)
#pragma unroll
                    for (int kx = 0; kx < 7; ++kx)
                        s = fmaf(W.w3[c][b][ky * 7 + kx], sm.p2[o][b][y + ky][x + kx], s);
            r = fmaf(W.w4[c], act(s), r);
        }
        sm.resp[o][cell] = act(r);
    }
    __syncthreads();
}

__global__ void __launch_bounds__(kSelThreads, 2) selective_kernel(
    const __grid_constant__ Cnn2W W2, const __grid_constant__ Cnn3W W3, const SelParams sp,
    const uint8_t* __restrict__ frames, const int64_t frame_stride, const int64_t pitch,
    const int Wd, const int Hd, const LevelInfo* __restrict__ lvinfo,
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
        const uint8_t* frame = frames + (int64_t)cd.frame * frame_stride;

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
        sm.hist[tid] = 0;                       // kSelThreads == 256 bins
        __syncthreads();
        // ---- O2 fixed-point bilinear sampling from the ORIGINAL frame + histogram ----
        for (int k = tid; k < kPatchN; k += kSelThreads) {
            const int v = k / kPatchW, u = k % kPatchW;
            const uint32_t xt = sm.colx[u], yt = sm.rowy[v];
            const uint32_t x0 = xt & 0xFFFFu, ax = xt >> 16, y0 = yt & 0xFFFFu, ay = yt >> 16;
            const uint32_t x1 = min(x0 + 1u, (uint32_t)(Wd - 1)), y1 = min(y0 + 1u, (uint32_t)(Hd - 1));
            const uint8_t* r0 = frame + (int64_t)y0 * pitch;
            const uint8_t* r1 = frame + (int64_t)y1 * pitch;
            const uint32_t top = (uint32_t)__ldg(r0 + x0) * (2048u - ax) + (uint32_t)__ldg(r0 + x1) * ax;
            const uint32_t bot = (uint32_t)__ldg(r1 + x0) * (2048u - ax) + (uint32_t)__ldg(r1 + x1) * ax;
            const uint32_t val = (top * (2048u - ay) + bot * ay + (1u << 21)) >> 22;
            sm.patch[k] = (uint8_t)val;
            atomicAdd(&sm.hist[val], 1);
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
        // ---- E and mirrored M, normalised to [-1, 1] (O3) ----
        for (int k = tid; k < kPatchN; k += kSelThreads) {
            const int v = k / kPatchW, u = k % kPatchW;
            const float e = fmaf((float)sm.lut[sm.patch[k]], 1.0f / 127.5f, -1.0f);
            sm.img[0][v][u] = e;
            sm.img[1][v][kPatchW - 1 - u] = e;
        }
        __syncthreads();

        // ---- CNN2 on both orientations, K2 ----
        run_net<16, 6, 2>(W2, sm, p1);
        float r2v = 0.f, r3v = 0.f;
        if (tid < 2 * kResp) r2v = sm.resp[tid / kResp][tid % kResp];
        const int K2 = __syncthreads_count(tid < 2 * kResp && r2v > sp.T2a);
        float best = -INFINITY;
        // block max of the responses of the last net evaluated (warp 0 + 1 hold them)
        auto block_max = [&](float v) {
            float* wm = sm.wmax;
            float m = (tid < 2 * kResp) ? v : -INFINITY;
#pragma unroll
            for (int d = 16; d >= 1; d >>= 1) m = fmaxf(m, __shfl_xor_sync(0xFFFFFFFFu, m, d));
            if ((tid & 31) == 0) wm[tid >> 5] = m;
            __syncthreads();
            float r = wm[0];
#pragma unroll
            for (int k = 1; k < kSelThreads / 32; ++k) r = fmaxf(r, wm[k]);
            __syncthreads();
            return r;
        };
        const bool stop = (sp.rule == 0) ? (K2 == 0) : (K2 >= sp.Tnn);   // P:99 / S:358
        int K3 = 0, delta, ran3 = 0;
        if (stop) {
            delta = (sp.rule == 0) ? 0 : 1;
            best = block_max(r2v);
        } else {
            // CNN3 reuses img; responses of CNN2 are kept in registers (r2v)
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
    return ((sizeof(SelSmem) + 15) & ~size_t(15)) + sizeof(float) * p1_floats<16>();
}

void launch_selective(const Cnn2W& w2, const Cnn3W& w3, SelParams sp, const uint8_t* frames,
                      int64_t frame_stride, int64_t pitch, int W, int H, const LevelInfo* d_levels,
                      const S1Cand* cands, uint32_t cand_cap, SelOut* out, float* dbg_resp,
                      AccBox* acc, Ctrl* ctrl, int sm_count, cudaStream_t s)
{
    const size_t smem = selective_smem_bytes();
    cudaFuncSetAttribute(selective_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, selective_kernel, kSelThreads, smem);
    if (occ < 1) occ = 1;
    selective_kernel<<<sm_count * occ, kSelThreads, smem, s>>>(w2, w3, sp, frames, frame_stride,
                                                              pitch, W, H, d_levels, cands, cand_cap,
                                                              out, dbg_resp, acc, ctrl);
}

}  // namespace ccnn
