// runtime.cu -- host runtime behind the C ABI (include/ccnn.h): context, validation,
// level planner, task table, device arena, launch sequence, readback, test hooks.
//
// Geometry (level table O1, pyramid sampling tables O2) is IEEE double evaluated in the
// same operation order as PAPER.md's reading in DESIGN.md; this TU is compiled with
// -ffp-contract=off so no multiply-add is fused and every value is bit-identical to
// the oracle's independent implementation.
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>
#include <algorithm>
#include <map>
#include <tuple>
#include <functional>
#include <queue>
#include <array>

#include "../../include/ccnn.h"
#include "ccnn_internal.h"
#include <cuda_fp16.h>

using namespace ccnn;

namespace {

struct DevBuf {
    void* p = nullptr;
    size_t bytes = 0;
    cudaError_t ensure(size_t want)
    {
        if (want <= bytes) return cudaSuccess;
        if (p) cudaFree(p);
        p = nullptr;
        bytes = 0;
        size_t grow = want + want / 4 + 4096;
        cudaError_t e = cudaMalloc(&p, grow);
        if (e == cudaSuccess) bytes = grow;
        return e;
    }
    void release() { if (p) cudaFree(p); p = nullptr; bytes = 0; }
    template <class T> T* as() const { return static_cast<T*>(p); }
};

struct PlanKey {                       // batch shape: every frame's size + search settings
    std::vector<std::pair<int, int>> dims;
    int min_face = -1;
    float scale_step = 0.f;
    bool operator==(const PlanKey& o) const
    {
        return min_face == o.min_face && scale_step == o.scale_step && dims == o.dims;
    }
};

bool finite_all(const float* w, int64_t n)
{
    for (int64_t k = 0; k < n; ++k) if (!std::isfinite(w[k])) return false;
    return true;
}

}  // namespace

struct ccnn_ctx {
    int device = 0;
    int sm_count = 148;
    int sel_grid = 0;                   // selective CNN2 grid (0 = sm_count; CCNN_SEL_GRID, experiments)
    int cnn3_grid = 0;                  // CNN3 + rule grid in SMs (0 = sm_count; CCNN_CNN3_SMS)
    cudaStream_t stream = nullptr;
    std::string err;
    int debug = 0;

    Cnn1W w1{};
    Cnn2W w2{};
    Cnn3W w3{};
    float T1 = 0.f;
    SelParams sp{};
    int min_cluster = 1;
    int max_w = 0, max_h = 0, max_batch = 0;
    int queue_cap = 4096;
    int seg_rows_param = 0;             // 0 = adaptive

    // plan (cached per batch shape)
    PlanKey key;
    std::vector<LevelInfo> levels;
    std::vector<S1Task> tasks;          // grouped by CTA (LPT schedule)
    std::vector<int32_t> cta_first;     // stage1_grid + 1 offsets into tasks
    int s1_grid = 0;
    bool s1_tc = true;                  // stage 1 on tcgen05 (stage1_tc.cu); CCNN_S1_LEGACY=1 -> stage1.cu
    bool patchwork = true;              // pack levels' tail pieces into shared bands;
                                        // CCNN_PATCHWORK=0: one band per tail (the ablation)
    DevBuf s1_bmats;                    // its B matrices
    DevBuf sel_bmats;                   // selective CNN2 (tcgen05) B matrices
    Cnn2Tc sel_consts{};                // ... and epilogue constants
    std::vector<uint32_t> tabs;
    int64_t arena_bytes = 0;            // all levels of all frames
    int64_t map_total = 0;              // dense stage-1 map floats (debug)
    int64_t windows_total = 0;
    double s1_mma_flops = 0.0;          // tensor-core FLOPs stage 1 issues for the planned batch
    int pyr_tiles = 0;                  // largest per-frame pyramid tile count
    int pyr_class_max[kPyrClasses] = {};   // ... per kernel class (gather, quad)
    std::vector<int32_t> frame_tiles_g;
    bool all_safe = true;               // every frame W, H >= 2 (pyramid fast path)
    std::vector<int32_t> frame_level0, frame_nlevels, frame_tiles, frame_tile_off;
    std::vector<uint32_t> ptiles;       // pyramid tile descriptors (pyramid.cu)

    // shared by consecutive batches (their kernels are ordered on the compute stream)
    DevBuf d_levels, d_tasks, d_cta_first, d_tabs, d_ptiles, dbg_resp, dbg_map;

    // per in-flight batch (ccnn_submit / ccnn_collect, NEXT #2 streaming ingest): three slots,
    // so the pyramid of batch k+2 can run in the background of batches k and k+1
    static constexpr int kSlots = 3;
    struct Slot {
        DevBuf frames;              // H2D destination (host input)
        DevBuf finfo;               // FrameInfo[n] of the batch
        DevBuf rgb, jobs;           // host RGB staging, GrayJob[] of the batch
        GrayJob* h_jobs = nullptr;  // pinned staging of jobs (max_batch entries)
        FrameInfo* h_finfo = nullptr;   // pinned staging of finfo (max_batch entries)
        DevBuf ctrl, out;           // control block, compacted boxes
        DevBuf arena;               // all levels of the batch (the pyramid of batch k+1 runs on
                                    // the pyramid stream while batch k's stage 1 reads its own)
        DevBuf resp2, epatch;       // CNN2 responses / equalised patches per survivor (selective_tc.cu)
        DevBuf cands, selout, acc, staging, counts;   // survivor queue .. NMS scratch: the
                                    // selective unit / NMS of batch k (tail stream) overlap
                                    // the stage 1 of batch k+1 (compute stream)
        Ctrl* h_ctrl = nullptr;     // pinned readback of ctrl
        std::vector<FrameInfo> fi_dev;  // what finfo holds on the device (skip identical uploads:
        const void* fi_dev_p = nullptr; // a small H2D queued behind the next batch's frame copy
                                        // on the copy engine would hold up this batch's pyramid)
        cudaEvent_t ev[9] = {};     // h2d0, h2d1, c0, pyramid, stage1, selective, end, stage-1 start,
                                    // selective start
        cudaEvent_t ev_user = nullptr;  // ctx stream at submit (orders the H2D of host frames)
        bool used = false;          // a batch has been enqueued on this slot before
        int n = 0, n_jobs = 0;
        uint32_t cand_cap = 0;
        int64_t windows = 0;
        double s1_mma_flops = 0.0;
        bool timed = false, empty = false;
        int pyr_launches = 0;
    } slot[kSlots];
    cudaStream_t copy_stream = nullptr, d2h_stream = nullptr;
    cudaStream_t pyr_stream = nullptr;  // pyramids (overlap the previous batch's stage 1..NMS)
    cudaEvent_t epoch = nullptr;        // CCNN_TIMELINE=1: per-batch event timestamps at collect
    int64_t batch_no = 0;
    cudaStream_t tail = nullptr;        // selective unit + NMS + readback of each batch
    cudaStream_t comp = nullptr;        // stage 1; ordered after the user's stream
                                        // (ccnn_set_stream) through the frames-ready event
    int next_slot = 0, inflight = 0;

    // texture objects over frames (pyramid tex2Dgather path), keyed by (data, w, h, pitch)
    std::map<std::tuple<uintptr_t, int, int, int64_t>, cudaTextureObject_t> tex_cache;
    int tex_align = 512, tex_pitch_align = 32;

    // last collected batch (test hooks, ccnn_last_boxes)
    int last_slot = 0;
    int last_n = 0, last_W = 0, last_H = 0;
    uint32_t last_cands = 0;
    uint32_t last_nout = 0;
    bool last_valid = false;
};

namespace {

int fail(ccnn_ctx* c, int code, const std::string& msg)
{
    if (c) c->err = msg;
    return code;
}

#define CU(call)                                                                          \
    do {                                                                                  \
        cudaError_t e_ = (call);                                                          \
        if (e_ != cudaSuccess)                                                            \
            return fail(ctx, CCNN_E_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
    } while (0)

// ---- architecture R check (include/ccnn.h CCNN_E_ARCH) ----
bool layers_equal(const ccnn_net& n, const int (*ref)[5], int nl)
{
    if (n.n_layers != nl || !n.layers) return false;
    for (int l = 0; l < nl; ++l) {
        const ccnn_layer& L = n.layers[l];
        if (L.kind != ref[l][0] || L.in_maps != ref[l][1] || L.out_maps != ref[l][2] ||
            L.kw != ref[l][3] || L.kh != ref[l][4])
            return false;
    }
    return true;
}

const int kR1[6][5] = {{0, 1, 6, 4, 4}, {1, 6, 6, 2, 2}, {0, 6, 6, 3, 3}, {1, 6, 6, 2, 2},
                       {0, 6, 2, 5, 6}, {0, 2, 1, 1, 1}};
const int kR2[6][5] = {{0, 1, 16, 4, 4}, {1, 16, 16, 2, 2}, {0, 16, 6, 3, 3}, {1, 6, 6, 2, 2},
                       {0, 6, 2, 7, 8}, {0, 2, 1, 1, 1}};
const int kR3[6][5] = {{0, 1, 2, 4, 4}, {1, 2, 2, 2, 2}, {0, 2, 2, 3, 3}, {1, 2, 2, 2, 2},
                       {0, 2, 25, 7, 8}, {0, 25, 1, 1, 1}};

int64_t conv_params(const int (*ref)[5], int nl)
{
    int64_t n = 0;
    for (int l = 0; l < nl; ++l)
        if (ref[l][0] == 0) n += (int64_t)ref[l][2] * (ref[l][1] * ref[l][3] * ref[l][4] + 1);
    return n;
}

// The weight blob is [kernels][bias] per conv layer (S:186 order); our structs hold the
// same values in the same order, so a straight copy per layer suffices.
inline float o_w1(int o, int k, const float* w) { return w[o * 16 + k]; }   // layer-1 [out][tap]

void unpack_cnn1(const float* w, Cnn1W& o)
{
    const float* p = w;
    std::memcpy(o.w1, p, sizeof(o.w1)); p += 96;
    std::memcpy(o.b1, p, sizeof(o.b1)); p += 6;
    std::memcpy(o.w2, p, sizeof(o.w2)); p += 324;
    std::memcpy(o.b2, p, sizeof(o.b2)); p += 6;
    std::memcpy(o.w3, p, sizeof(o.w3)); p += 360;
    std::memcpy(o.b3, p, sizeof(o.b3)); p += 2;
    std::memcpy(o.w4, p, sizeof(o.w4)); p += 2;
    o.b4 = *p;
    {                                                // tensor-core layer-1 fragments
        double mx = 0.0;
        for (int m = 0; m < 6; ++m)
            for (int k = 0; k < 16; ++k) mx = std::max(mx, std::fabs((double)o_w1(m, k, w)) / 127.5);
        // scale so that max |W'| lies in [8, 16): fp16 hi/lo parts stay normal
        const int e = mx > 0.0 ? (int)std::floor(std::log2(mx)) : 0;
        const double sc = std::ldexp(1.0, 3 - e);
        o.l1_inv_scale = (float)std::ldexp(1.0, e - 3);
        auto part = [&](int o_, int k, int lo) -> uint16_t {
            if (o_ >= 6) return 0;
            const float wp = (float)((double)o_w1(o_, k, w) / 127.5 * sc);
            const __half hi = __float2half_rn(wp);
            if (!lo) return __half_as_ushort(hi);
            return __half_as_ushort(__float2half_rn(wp - __half2float(hi)));
        };
        for (int lo = 0; lo < 2; ++lo)
            for (int lane = 0; lane < 32; ++lane) {
                const int n = lane / 4, k0 = (lane % 4) * 2;
                for (int r = 0; r < 2; ++r) {
                    const int k = k0 + 8 * r;
                    o.l1frag[lo][lane][r] = (uint32_t)part(n, k, lo) | ((uint32_t)part(n, k + 1, lo) << 16);
                }
            }
        for (int m = 0; m < 8; ++m) {
            double b = 0.0;
            if (m < 6) {
                b = (double)o.b1[m];
                for (int k = 0; k < 16; ++k) b -= (double)o_w1(m, k, w);
            }
            o.b1h[m] = (float)b;
        }
    }
    {                                                // tensor-core layer-2 scale (stage1_tc.cu)
        double mx = 0.0;
        for (int k = 0; k < 324; ++k) mx = std::max(mx, std::fabs((double)(&o.w2[0][0][0])[k]));
        const int e = mx > 0.0 ? (int)std::floor(std::log2(mx)) : 0;
        o.l2_inv_scale = (float)std::ldexp(1.0, e - 3);
        double m3 = 0.0;
        for (int k = 0; k < 360; ++k) m3 = std::max(m3, std::fabs((double)(&o.w3[0][0][0])[k]));
        const int e3 = m3 > 0.0 ? (int)std::floor(std::log2(m3)) : 0;
        o.l3_inv_scale = (float)std::ldexp(1.0, e3 - 3);
    }
    {                                                // stage1_tc.cu epilogues: x' = 2x/3
        const double k = 2.0 / 3.0;
        for (int m = 0; m < 6; ++m) o.tcx[m] = (float)(k * (double)o.b1h[m]);
        for (int m = 0; m < 6; ++m) o.tcx[6 + m] = (float)(k * (double)o.b2[m]);
        for (int m = 0; m < 2; ++m) o.tcx[12 + m] = (float)(k * (double)o.b3[m]);
        o.tcx[14] = (float)(k * (double)o.l1_inv_scale);
        o.tcx[15] = (float)(k * (double)o.l2_inv_scale);
        o.tcx[16] = (float)(k * (double)o.l3_inv_scale);
        for (int m = 0; m < 2; ++m) o.tcx[17 + m] = (float)(k * (double)o.w4[m]);
        o.tcx[19] = (float)(k * (double)o.b4);
    }
    for (int ci = 0; ci < 6; ++ci) {                 // vector-friendly copies (stage1.cu)
        for (int k = 0; k < 56; ++k) o.w2v[ci][k] = k < 54 ? o.w2[k / 9][ci][k % 9] : 0.f;
        for (int i = 0; i < 6; ++i)
            for (int m = 0; m < 2; ++m)
                for (int kx = 0; kx < 5; ++kx) o.w3v[ci][(i * 2 + m) * 5 + kx] = o.w3[m][ci][(5 - i) * 5 + kx];
    }
}
template <int A, int B, int C>
void unpack_sel(const float* p, SelNetW<A, B, C>& o)
{
    std::memcpy(o.w1, p, sizeof(o.w1)); p += A * 16;
    std::memcpy(o.b1, p, sizeof(o.b1)); p += A;
    std::memcpy(o.w2, p, sizeof(o.w2)); p += B * A * 9;
    std::memcpy(o.b2, p, sizeof(o.b2)); p += B;
    std::memcpy(o.w3, p, sizeof(o.w3)); p += C * B * 56;
    std::memcpy(o.b3, p, sizeof(o.b3)); p += C;
    std::memcpy(o.w4, p, sizeof(o.w4)); p += C;
    o.b4 = *p;
    double mx = 0.0;
    for (int a = 0; a < A; ++a)
        for (int k = 0; k < 16; ++k) mx = std::max(mx, std::fabs((double)o.w1[a][k]) / 127.5);
    const int e = mx > 0.0 ? (int)std::floor(std::log2(mx)) : 0;
    o.l1_inv_scale = (float)std::ldexp(1.0, e - 3);
    for (int a = 0; a < A; ++a) {
        double b = (double)o.b1[a];
        for (int k = 0; k < 16; ++k) b -= (double)o.w1[a][k];
        o.b1h[a] = (float)b;
    }
}

int64_t round_up(int64_t v, int64_t a) { return (v + a - 1) / a * a; }

// Texture object over one uint8 frame (pitch-2D, point sampling, clamp-to-edge, unnormalised
// coordinates), cached; 0 if the frame's address or pitch does not meet the texture
// alignment (the pyramid then takes its byte-gather form).
cudaTextureObject_t frame_texture(ccnn_ctx* c, const uint8_t* data, int w, int h, int64_t pitch)
{
    if ((uintptr_t)data % c->tex_align || pitch % c->tex_pitch_align) return 0;
    const auto key = std::make_tuple((uintptr_t)data, w, h, pitch);
    auto it = c->tex_cache.find(key);
    if (it != c->tex_cache.end()) return it->second;
    cudaResourceDesc rd{};
    rd.resType = cudaResourceTypePitch2D;
    rd.res.pitch2D.devPtr = const_cast<uint8_t*>(data);
    rd.res.pitch2D.desc = cudaCreateChannelDesc<unsigned char>();
    rd.res.pitch2D.width = (size_t)w;
    rd.res.pitch2D.height = (size_t)h;
    rd.res.pitch2D.pitchInBytes = (size_t)pitch;
    cudaTextureDesc td{};
    td.addressMode[0] = cudaAddressModeClamp;
    td.addressMode[1] = cudaAddressModeClamp;
    td.filterMode = cudaFilterModePoint;
    td.readMode = cudaReadModeElementType;
    td.normalizedCoords = 0;
    cudaTextureObject_t t = 0;
    if (cudaCreateTextureObject(&t, &rd, &td, nullptr) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    c->tex_cache.emplace(key, t);
    return t;
}

// destroy cached texture objects whose frame lies in [lo, lo + bytes) (all if bytes == 0);
// the caller guarantees no queued kernel still uses them
void drop_textures(ccnn_ctx* c, const void* lo, size_t bytes)
{
    for (auto it = c->tex_cache.begin(); it != c->tex_cache.end();) {
        const uintptr_t p = std::get<0>(it->first);
        if (bytes == 0 || (p >= (uintptr_t)lo && p < (uintptr_t)lo + bytes)) {
            cudaDestroyTextureObject(it->second);
            it = c->tex_cache.erase(it);
        } else {
            ++it;
        }
    }
}

// O2 sampling table entry: s = (d + 0.5)/sigma - 0.5, clamp [0, n-1], i0 = floor(s),
// i1 = min(i0 + 1, n - 1), a = floor((s - i0) * 2048 + 0.5); packed i0 | a << 16.
// For n >= 2 the clamped edge (i0 = n-1, a = 0) is re-encoded as (i0 = n-2, a = 2048):
// p[n-2]*0 + p[n-1]*2048 == p[n-1]*2048 exactly, so the kernel may always use i0 + 1.
uint32_t sample_entry(int d, double sigma, int n)
{
    double s = ((double)d + 0.5) / sigma - 0.5;
    if (s < 0.0) s = 0.0;
    if (s > (double)(n - 1)) s = (double)(n - 1);
    int f = (int)std::floor(s);
    int a = (int)std::floor((s - (double)f) * 2048.0 + 0.5);
    if (n >= 2 && f == n - 1) { f = n - 2; a = 2048; }
    return (uint32_t)f | ((uint32_t)a << 16);
}

// Level table O1 + stage-1 task table + sampling tables for one batch shape: every frame
// of the batch gets its own levels (frames may differ in size); the
// sampling tables are shared by the levels of equally-sized frames.
void build_plan(ccnn_ctx* c, const PlanKey& key)
{
    c->levels.clear();
    c->tasks.clear();
    c->tabs.clear();
    c->frame_level0.clear();
    c->frame_nlevels.clear();
    c->frame_tiles.clear();
    c->frame_tile_off.clear();
    c->ptiles.clear();
    c->frame_tiles_g.clear();
    c->pyr_tiles = 0;
    for (int& m : c->pyr_class_max) m = 0;
    c->all_safe = true;
    const double sf = (double)key.scale_step;
    int64_t off = 0, map_off = 0;
    c->windows_total = 0;
    std::map<std::pair<int, int>, std::vector<int32_t>> tab_cache;   // (W,H) -> tab_off per level
    std::map<std::pair<int, int>, std::pair<int32_t, int32_t>> tile_cache;   // -> (offset, count)
    std::map<std::pair<int, int>, std::array<int32_t, kPyrClasses>> class_cache;   // -> count per class
    for (int f = 0; f < (int)key.dims.size(); ++f) {
        const int W = key.dims[f].first, H = key.dims[f].second;
        auto it = tab_cache.find(key.dims[f]);
        const bool have_tabs = it != tab_cache.end();
        std::vector<int32_t> new_tabs;
        c->frame_level0.push_back((int32_t)c->levels.size());
        const int level0 = (int)c->levels.size();
        double s = (double)kWinW / (double)key.min_face;
        int k = 0;
        while (true) {
            const int lw = (int)std::floor((double)W * s);
            const int lh = (int)std::floor((double)H * s);
            if (lw < kWinW || lh < kWinH || k > kMaxLevels) break;   // > kMaxLevels: refused
            LevelInfo L{};
            L.sigma = s;
            L.lw = lw;
            L.lh = lh;
            L.pitch = (int)round_up(lw, 16);
            L.offset = off;
            L.map_off = map_off;
            L.nx = (lw - kWinW) / kStep + 1;
            L.ny = (lh - kWinH) / kStep + 1;
            L.frame = f;
            if (have_tabs) {
                L.tab_off = it->second[k];
            } else {
                L.tab_off = (int32_t)c->tabs.size();
                new_tabs.push_back(L.tab_off);
                // x entries for every pitch column (padding repeats the edge column), then
                // y entries for kPyrTileRows-rounded rows (padding repeats the last row): the
                // pyramid kernel reads them unclamped; 16-B aligned (pitch % 16 == 0)
                for (int x = 0; x < L.pitch; ++x) c->tabs.push_back(sample_entry(std::min(x, lw - 1), s, W));
                const int lh_pad = (int)round_up(lh, kPyrTileRows);
                for (int y = 0; y < lh_pad; ++y) c->tabs.push_back(sample_entry(std::min(y, lh - 1), s, H));
            }
            off += round_up((int64_t)L.pitch * lh, 256);
            map_off += (int64_t)L.nx * L.ny;
            c->windows_total += (int64_t)L.nx * L.ny;
            c->levels.push_back(L);
            s = s / sf;
            ++k;
        }
        c->frame_nlevels.push_back(k);
        // pyramid tile descriptors (level-in-frame | tile column << 8 | tile row << 16),
        // grouped by kernel class (gather | quad), largest levels first within a
        // class; shared by equally-sized frames
        if (!have_tabs) {
            tab_cache[key.dims[f]] = new_tabs;
            const int32_t first = (int32_t)c->ptiles.size();
            std::array<int32_t, kPyrClasses> cnt{};
            const bool safe = W >= 2 && H >= 2;
            for (int cls = 0; cls < kPyrClasses; ++cls)
                for (int l = 0; l < k && l < 256; ++l) {
                    const LevelInfo& L = c->levels[level0 + l];
                    const int lc = safe && L.sigma >= kPyrQuadSigma ? kPyrQuad : kPyrGather;
                    if (lc != cls) continue;
                    const int tx_n = (L.pitch + kPyrCols - 1) / kPyrCols;
                    const int ty_n = (L.lh + kPyrTileRows - 1) / kPyrTileRows;
                    for (int ty = 0; ty < ty_n; ++ty)
                        for (int tx = 0; tx < tx_n; ++tx)
                            c->ptiles.push_back((uint32_t)l | ((uint32_t)tx << 8) | ((uint32_t)ty << 16));
                    cnt[cls] += tx_n * ty_n;
                }
            tile_cache[key.dims[f]] = {first, (int32_t)c->ptiles.size() - first};
            class_cache[key.dims[f]] = cnt;
        }
        const auto tc = tile_cache[key.dims[f]];
        const auto cc = class_cache[key.dims[f]];
        c->frame_tile_off.push_back(tc.first);
        c->frame_tiles.push_back(tc.second);
        c->frame_tiles_g.push_back(cc[kPyrGather]);
        c->pyr_tiles = std::max(c->pyr_tiles, tc.second);
        for (int cls = 0; cls < kPyrClasses; ++cls) c->pyr_class_max[cls] = std::max(c->pyr_class_max[cls], cc[cls]);
        c->all_safe = c->all_safe && W >= 2 && H >= 2;
    }
    // slack so that the stage-1 loader's last (clamped) word read stays in bounds
    c->arena_bytes = round_up(off + 256, 256);
    c->map_total = map_off;
    const int TW = c->s1_tc ? stage1_tc_band_width() : stage1_band_width();
    auto task_cost = [&](int nrows) { return c->s1_tc ? stage1_tc_task_cost(nrows) : stage1_task_cost(nrows); };
    // segment height: the tallest segments (least vertical halo recompute) whose largest
    // task still fits in the average load of a CTA slot, so the dynamic longest-first list
    // schedule balances (measured at C4 with the tcgen05 kernel: full-height bands 0.418 ms
    // vs 0.452 at the former half-load rule's 128 rows; ccnn_params.segment_rows > 0 forces
    // a height)
    // bands: every full TW-wide band of a level is its own band; the tail pieces (the last,
    // narrower band of each level, or a whole narrow level) are packed side by side into
    // shared bands, first-fit by decreasing height (patchwork)
    struct Band { int npieces; S1Piece piece[kMaxPieces]; int height; int used; };
    std::vector<Band> bands;
    std::vector<S1Piece> tails;
    for (int l = 0; l < (int)c->levels.size(); ++l) {
        const LevelInfo& L = c->levels[l];
        int x0 = 0;
        for (; x0 + TW <= L.nx; x0 += TW) {
            Band b{};
            b.npieces = 1;
            b.piece[0] = S1Piece{(int16_t)l, (int16_t)x0, (int16_t)TW, 0};
            b.height = L.ny;
            b.used = TW;
            bands.push_back(b);
        }
        if (x0 < L.nx) tails.push_back(S1Piece{(int16_t)l, (int16_t)x0, (int16_t)(L.nx - x0), 0});
    }
    std::stable_sort(tails.begin(), tails.end(), [&](const S1Piece& a, const S1Piece& b) {
        return c->levels[a.level].ny > c->levels[b.level].ny;
    });
    const size_t first_tail_band = bands.size();
    for (const S1Piece& t : tails) {
        bool placed = false;
        for (size_t k = first_tail_band; c->patchwork && k < bands.size() && !placed; ++k) {
            Band& b = bands[k];
            if (b.npieces < kMaxPieces && b.used + kPieceGap + t.w <= TW) {
                S1Piece p = t;
                p.J = (int16_t)(b.used + kPieceGap);
                b.piece[b.npieces++] = p;
                b.used = p.J + p.w;
                placed = true;
            }
        }
        if (!placed) {
            Band b{};
            b.npieces = 1;
            b.piece[0] = t;
            b.height = c->levels[t.level].ny;   // tallest first: the band's height
            b.used = t.w;
            bands.push_back(b);
        }
    }
    auto make_tasks = [&](int seg, std::vector<S1Task>& one) {
        one.clear();
        for (const Band& b : bands) {
            const int nseg = std::max(1, (b.height + seg - 1) / seg);
            const int rows = (b.height + nseg - 1) / nseg;
            for (int y0 = 0; y0 < b.height; y0 += rows) {
                S1Task t{};
                t.y0 = (int16_t)y0;
                t.nrows = (int16_t)std::min(rows, b.height - y0);
                t.npieces = (int16_t)b.npieces;
                for (int p = 0; p < b.npieces; ++p) t.piece[p] = b.piece[p];
                one.push_back(t);
            }
        }
    };
    std::vector<S1Task> one;
    if (c->seg_rows_param > 0) {
        make_tasks(c->seg_rows_param, one);
    } else {
        for (int seg : {1 << 14, 256, 192, 128, 96, 64, 48, 32, 24, 16}) {
            make_tasks(seg, one);
            int64_t total = 0, biggest = 0;
            for (const S1Task& t : one) {
                total += task_cost(t.nrows);
                biggest = std::max<int64_t>(biggest, task_cost(t.nrows));
            }
            const int64_t slots = (int64_t)c->s1_grid * (c->s1_tc ? stage1_tc_pipes_per_cta() : 1);
            if (biggest * slots <= total) break;
        }
    }
    // tasks of all frames in one list, longest first (cost ~ super-steps, independent of the
    // band width); frame = the frame of the first piece (informational)
    std::vector<S1Task> all = one;
    for (S1Task& t : all) t.frame = c->levels[t.piece[0].level].frame;
    std::stable_sort(all.begin(), all.end(),
                     [](const S1Task& a, const S1Task& b) { return a.nrows > b.nrows; });
    // the kernel takes tasks in this order from an atomic counter (greedy list scheduling);
    // cta_first = {0, ..., 0, n_tasks}: grid size + total task count for the launch
    const int G = std::max(1, std::min<int>(c->s1_grid, (int)all.size()));
    c->tasks = all;
    c->s1_mma_flops = 0.0;
    if (c->s1_tc)
        for (const S1Task& t : all) c->s1_mma_flops += stage1_tc_task_mma_flops(t.nrows);
    c->cta_first.assign(G + 1, 0);
    c->cta_first[G] = (int32_t)all.size();
}

}  // namespace

extern "C" {

int ccnn_abi_version(void) { return CCNN_ABI_VERSION; }

const char* ccnn_last_error(const ccnn_ctx* ctx)
{
    if (!ctx) return "ccnn: NULL context (ccnn_create failed or was not called)";
    return ctx->err.c_str();
}

int ccnn_create(const ccnn_params* p, int cuda_device, ccnn_ctx** out)
{
    ccnn_ctx* ctx = nullptr;
    if (!p || !out) return CCNN_E_ARG;
    if (!layers_equal(p->net[0], kR1, 6) || !layers_equal(p->net[1], kR2, 6) ||
        !layers_equal(p->net[2], kR3, 6))
        return CCNN_E_ARCH;
    if (p->net[0].n_weights != conv_params(kR1, 6) || p->net[1].n_weights != conv_params(kR2, 6) ||
        p->net[2].n_weights != conv_params(kR3, 6))
        return CCNN_E_WEIGHTS;
    for (int k = 0; k < 3; ++k)
        if (!p->net[k].weights || !finite_all(p->net[k].weights, p->net[k].n_weights)) return CCNN_E_WEIGHTS;
    if (!std::isfinite(p->T1) || !std::isfinite(p->T2[0]) || !std::isfinite(p->T2[1])) return CCNN_E_WEIGHTS;
    if (p->Tnn < 1 || (p->rule != 0 && p->rule != 1) || p->max_w < kWinW || p->max_h < kWinH ||
        p->max_w > 16384 || p->max_h > 16384 || p->max_batch < 1 || p->max_batch > kNmsCap ||
        p->queue_capacity < 0 ||
        p->nms_min_cluster < 0 || p->segment_rows < 0)
        return CCNN_E_ARG;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || cuda_device < 0 || cuda_device >= ndev)
        return CCNN_E_CUDA;
    ctx = new ccnn_ctx();
    ctx->device = cuda_device;
    CU(cudaSetDevice(cuda_device));
    CU(cudaDeviceGetAttribute(&ctx->sm_count, cudaDevAttrMultiProcessorCount, cuda_device));
    if (const char* e = std::getenv("CCNN_SEL_GRID")) ctx->sel_grid = std::atoi(e);
    if (const char* e = std::getenv("CCNN_CNN3_SMS")) ctx->cnn3_grid = std::atoi(e);
    unpack_cnn1(p->net[0].weights, ctx->w1);
    unpack_sel(p->net[1].weights, ctx->w2);
    unpack_sel(p->net[2].weights, ctx->w3);
    ctx->T1 = p->T1;
    ctx->sp.T2a = p->T2[0];
    ctx->sp.T2b = p->T2[1];
    ctx->sp.Tnn = p->Tnn;
    ctx->sp.rule = p->rule;
    ctx->min_cluster = p->nms_min_cluster < 1 ? 1 : p->nms_min_cluster;
    ctx->max_w = p->max_w;
    ctx->max_h = p->max_h;
    ctx->max_batch = p->max_batch;
    ctx->queue_cap = p->queue_capacity > 0 ? p->queue_capacity : 4096;
    ctx->seg_rows_param = p->segment_rows;
    {
        const char* leg = std::getenv("CCNN_S1_LEGACY");
        ctx->s1_tc = !(leg && leg[0] == '1');
        const char* pw = std::getenv("CCNN_PATCHWORK");
        ctx->patchwork = !(pw && pw[0] == '0');
    }
    ctx->s1_grid = ctx->s1_tc ? stage1_tc_grid(ctx->sm_count) : stage1_grid(ctx->sm_count);
    if (const char* v = std::getenv("CCNN_VERBOSE"))
        if (v[0] == '1') std::fprintf(stderr, "ccnn: stage 1 %s, grid %d\n", ctx->s1_tc ? "tcgen05" : "legacy", ctx->s1_grid);
    if (ctx->s1_tc) {
        std::vector<uint16_t> bm(kStage1TcBmatHalves);
        stage1_tc_bmats(ctx->w1, bm.data());
        CU(ctx->s1_bmats.ensure(bm.size() * 2));
        CU(cudaMemcpy(ctx->s1_bmats.p, bm.data(), bm.size() * 2, cudaMemcpyHostToDevice));
    }
    {
        std::vector<uint16_t> bm(kSelTcBmatHalves);
        selective_tc_bmats(ctx->w2, bm.data(), &ctx->sel_consts);
        CU(ctx->sel_bmats.ensure(bm.size() * 2));
        CU(cudaMemcpy(ctx->sel_bmats.p, bm.data(), bm.size() * 2, cudaMemcpyHostToDevice));
    }
    CU(cudaGetLastError());
    for (auto& sl : ctx->slot) {
        CU(cudaMallocHost(&sl.h_ctrl, sizeof(Ctrl)));
        std::memset(sl.h_ctrl, 0, sizeof(Ctrl));
        CU(cudaMallocHost(&sl.h_finfo, sizeof(FrameInfo) * (size_t)p->max_batch));
        CU(cudaMallocHost(&sl.h_jobs, sizeof(GrayJob) * (size_t)p->max_batch));
        for (auto& e : sl.ev) CU(cudaEventCreate(&e));
        CU(cudaEventCreateWithFlags(&sl.ev_user, cudaEventDisableTiming));
        CU(sl.ctrl.ensure(sizeof(Ctrl)));
    }
    CU(cudaDeviceGetAttribute(&ctx->tex_align, cudaDevAttrTextureAlignment, cuda_device));
    CU(cudaDeviceGetAttribute(&ctx->tex_pitch_align, cudaDevAttrTexturePitchAlignment, cuda_device));
    ctx->tex_align = std::max(ctx->tex_align, 1);
    ctx->tex_pitch_align = std::max(ctx->tex_pitch_align, 1);
    CU(cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking));
    CU(cudaStreamCreateWithFlags(&ctx->d2h_stream, cudaStreamNonBlocking));
    {   // the compute stream outranks the pyramid stream: when both have CTAs waiting, the
        // block scheduler places stage 1 .. NMS first and the next batch's pyramid fills in
        int least = 0, greatest = 0;
        CU(cudaDeviceGetStreamPriorityRange(&least, &greatest));
        CU(cudaStreamCreateWithPriority(&ctx->pyr_stream, cudaStreamNonBlocking, least));
        CU(cudaStreamCreateWithPriority(&ctx->comp, cudaStreamNonBlocking, greatest));
        CU(cudaStreamCreateWithPriority(&ctx->tail, cudaStreamNonBlocking, greatest));
    }
    *out = ctx;
    return CCNN_OK;
}

int ccnn_set_stream(ccnn_ctx* ctx, void* cuda_stream)
{
    if (!ctx) return CCNN_E_ARG;
    ctx->stream = static_cast<cudaStream_t>(cuda_stream);
    return CCNN_OK;
}

int ccnn_set_debug(ccnn_ctx* ctx, int flags)
{
    if (!ctx) return CCNN_E_ARG;
    ctx->debug = flags;
    return CCNN_OK;
}

void ccnn_destroy(ccnn_ctx* ctx)
{
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    cudaDeviceSynchronize();
    drop_textures(ctx, nullptr, 0);
    for (DevBuf* b : {&ctx->d_levels, &ctx->d_tasks, &ctx->d_cta_first, &ctx->d_tabs, &ctx->d_ptiles,
                      &ctx->dbg_resp,
                      &ctx->dbg_map, &ctx->s1_bmats, &ctx->sel_bmats})
        b->release();
    for (auto& sl : ctx->slot) {
        sl.frames.release();
        sl.finfo.release();
        if (sl.h_finfo) cudaFreeHost(sl.h_finfo);
        sl.rgb.release();
        sl.jobs.release();
        if (sl.h_jobs) cudaFreeHost(sl.h_jobs);
        sl.ctrl.release();
        sl.out.release();
        sl.arena.release();
        for (DevBuf* b : {&sl.cands, &sl.selout, &sl.acc, &sl.staging, &sl.counts, &sl.resp2, &sl.epatch}) b->release();
        if (sl.h_ctrl) cudaFreeHost(sl.h_ctrl);
        for (auto& e : sl.ev) if (e) cudaEventDestroy(e);
        if (sl.ev_user) cudaEventDestroy(sl.ev_user);
    }
    if (ctx->copy_stream) cudaStreamDestroy(ctx->copy_stream);
    if (ctx->d2h_stream) cudaStreamDestroy(ctx->d2h_stream);
    if (ctx->pyr_stream) cudaStreamDestroy(ctx->pyr_stream);
    if (ctx->comp) cudaStreamDestroy(ctx->comp);
    if (ctx->tail) cudaStreamDestroy(ctx->tail);
    if (ctx->epoch) cudaEventDestroy(ctx->epoch);
    delete ctx;
}

int ccnn_submit_frames(ccnn_ctx* ctx, const ccnn_frame* frames, int n, int frames_on_device,
                       int min_face, float scale_step, int timed)
{
    if (!ctx) return CCNN_E_ARG;
    if (!frames) return fail(ctx, CCNN_E_ARG, "NULL frames");
    if (n <= 0 || n > ctx->max_batch) return fail(ctx, CCNN_E_ARG, "n out of [1, max_batch]");
    if (min_face < 1) return fail(ctx, CCNN_E_ARG, "min_face < 1");
    if (!(scale_step > 1.0f) || !std::isfinite(scale_step))
        return fail(ctx, CCNN_E_ARG, "scale_step must be > 1 (S:227)");
    PlanKey key;
    key.min_face = min_face;
    key.scale_step = scale_step;
    key.dims.reserve(n);
    for (int f = 0; f < n; ++f) {
        const ccnn_frame& F = frames[f];
        if (!F.data) return fail(ctx, CCNN_E_ARG, "NULL frame data");
        if (F.w < 1 || F.h < 1 || F.w > ctx->max_w || F.h > ctx->max_h)
            return fail(ctx, CCNN_E_ARG, "frame size out of [1, max_w] x [1, max_h]");
        const int ch = F.channels == 0 ? 1 : F.channels;
        if ((ch != 1 && ch != 3) || F.reserved != 0)
            return fail(ctx, CCNN_E_ARG, "channels must be 0, 1 or 3 and reserved 0");
        if (F.pitch < (int64_t)F.w * ch) return fail(ctx, CCNN_E_ARG, "pitch < width * channels");
        if ((double)kWinW / min_face * std::max(F.w, F.h) > 32000.0)
            return fail(ctx, CCNN_E_ARG, "level 0 too large (min_face too small for this frame)");
        key.dims.emplace_back(F.w, F.h);
    }
    if (ctx->inflight >= ccnn_ctx::kSlots) return fail(ctx, CCNN_E_STATE, "three batches in flight: ccnn_collect first");
    CU(cudaSetDevice(ctx->device));
    // device work: pyramid on pyr_stream, the rest on comp; both start after an event recorded
    // on the user's stream (device frames written there are complete), so batch k+1's pyramid
    // can overlap batch k's later stages
    cudaStream_t s = ctx->comp;

    const bool replan = !(key == ctx->key);
    if (replan) {
        CU(cudaStreamSynchronize(s));              // tables of an in-flight batch stay valid
        CU(cudaStreamSynchronize(ctx->pyr_stream));
        CU(cudaStreamSynchronize(ctx->tail));
        // the host plan changes now; the device tables only after the uploads below: until
        // ctx->key = key commits both, a failure (any CU() below) leaves the key invalid so
        // the next submit replans and re-uploads instead of pairing old tables with a new plan
        ctx->key = PlanKey{};
        build_plan(ctx, key);
    }
    const int L = (int)ctx->levels.size();
    for (int f = 0; f < n; ++f)
        if (ctx->frame_nlevels[f] > kMaxLevels) {
            ctx->key = PlanKey{};
            return fail(ctx, CCNN_E_ARG, "more than 256 pyramid levels (scale_step too close to 1)");
        }
    if (L > 32767) {
        ctx->key = PlanKey{};
        return fail(ctx, CCNN_E_ARG, "more than 32767 pyramid levels in one batch");
    }
    ccnn_ctx::Slot& sl = ctx->slot[ctx->next_slot];
    sl.n = n;
    sl.windows = ctx->windows_total;
    sl.s1_mma_flops = ctx->s1_mma_flops;
    sl.timed = timed != 0;
    sl.empty = (L == 0);                           // empty pyramid: not an error
    ctx->last_W = frames[0].w;
    ctx->last_H = frames[0].h;
    if (sl.empty) {
        ctx->key = key;
        sl.cand_cap = 0;
        sl.n_jobs = 0;
        CU(cudaEventRecord(sl.ev[6], s));
        ctx->next_slot = (ctx->next_slot + 1) % ccnn_ctx::kSlots;
        ctx->inflight++;
        return CCNN_OK;
    }

    const uint32_t cand_cap = (uint32_t)std::min<int64_t>((int64_t)ctx->queue_cap * n, 0x7FFFFFFF);
    sl.cand_cap = cand_cap;
    CU(sl.arena.ensure((size_t)ctx->arena_bytes));
    CU(ctx->d_levels.ensure(sizeof(LevelInfo) * L));
    CU(ctx->d_tasks.ensure(sizeof(S1Task) * ctx->tasks.size()));
    CU(ctx->d_cta_first.ensure(sizeof(int32_t) * ctx->cta_first.size()));
    CU(ctx->d_tabs.ensure(sizeof(uint32_t) * ctx->tabs.size()));
    CU(ctx->d_ptiles.ensure(sizeof(uint32_t) * std::max<size_t>(1, ctx->ptiles.size())));
    CU(sl.cands.ensure(sizeof(S1Cand) * cand_cap));
    CU(sl.selout.ensure(sizeof(SelOut) * cand_cap));
    CU(sl.resp2.ensure(sizeof(float) * 50 * (size_t)cand_cap));
    CU(sl.epatch.ensure((size_t)kEPatchBytes * cand_cap));
    CU(sl.acc.ensure(sizeof(AccBox) * cand_cap));
    CU(sl.staging.ensure(sizeof(OutBox) * kNmsCap * (size_t)n));
    CU(sl.counts.ensure(sizeof(int32_t) * n));
    CU(sl.out.ensure(sizeof(OutBox) * cand_cap));
    CU(sl.finfo.ensure(sizeof(FrameInfo) * n));
    const bool dbg1 = (ctx->debug & CCNN_DEBUG_STAGE1) != 0;
    if (dbg1) {
        CU(ctx->dbg_map.ensure(sizeof(float) * ctx->map_total));
        CU(ctx->dbg_resp.ensure(sizeof(float) * 100 * (size_t)cand_cap));
    }
    if (replan || ctx->key.min_face < 0) {
        CU(cudaMemcpyAsync(ctx->d_levels.p, ctx->levels.data(), sizeof(LevelInfo) * L,
                           cudaMemcpyHostToDevice, s));
        CU(cudaMemcpyAsync(ctx->d_tasks.p, ctx->tasks.data(), sizeof(S1Task) * ctx->tasks.size(),
                           cudaMemcpyHostToDevice, s));
        CU(cudaMemcpyAsync(ctx->d_tabs.p, ctx->tabs.data(), sizeof(uint32_t) * ctx->tabs.size(),
                           cudaMemcpyHostToDevice, s));
        if (!ctx->ptiles.empty())
            CU(cudaMemcpyAsync(ctx->d_ptiles.p, ctx->ptiles.data(), sizeof(uint32_t) * ctx->ptiles.size(),
                               cudaMemcpyHostToDevice, s));
        CU(cudaMemcpyAsync(ctx->d_cta_first.p, ctx->cta_first.data(),
                           sizeof(int32_t) * ctx->cta_first.size(), cudaMemcpyHostToDevice, s));
        CU(cudaStreamSynchronize(s));   // host vectors may change on the next replan
    }
    ctx->key = key;

    // ---- frames: device-resident, or H2D on the copy stream (host -> device boundary);
    //      the copy of batch k+1 overlaps the kernels of batch k ----
    FrameInfo* fi = sl.h_finfo;                    // pinned; reused only after this slot's collect
    GrayJob* jobs = sl.h_jobs;
    int n_jobs = 0;
    {
        // device copies: host gray frames keep the caller's pitch and a run of equally-sized
        // frames lying back to back in host memory stays back to back (one linear H2D for the
        // run: a pitched 2-D copy of short rows runs far below the PCIe rate); every RGB frame's
        // gray plane, and every frame when the texture pyramid is requested, gets a pitch and
        // frame offset that meet the texture alignment; host RGB frames are staged as they come
        const int64_t pa = std::max<int64_t>(16, ctx->tex_pitch_align);
        const int64_t fa = std::max<int64_t>(256, ctx->tex_align);
        const bool tex_layout = (ctx->debug & CCNN_DEBUG_PYR_TEX) != 0;
        auto chans = [&](int f) { return frames[f].channels == 0 ? 1 : frames[f].channels; };
        std::vector<int64_t> foff(n, -1), roff(n, -1), dpv(n, 0);
        int64_t total = 0, rtotal = 0;
        for (int f = 0; f < n; ++f) {
            if (frames_on_device && chans(f) == 1) continue;      // used in place
            const bool keep = !tex_layout && chans(f) == 1;      // host gray frame
            dpv[f] = keep ? frames[f].pitch : round_up(frames[f].w, pa);
            const bool follows = keep && f > 0 && foff[f - 1] >= 0 && chans(f - 1) == 1 &&
                                 dpv[f - 1] == dpv[f] && frames[f - 1].w == frames[f].w &&
                                 frames[f - 1].h == frames[f].h &&
                                 frames[f].data == frames[f - 1].data + dpv[f] * frames[f].h;
            if (!follows) total = round_up(total, fa);
            foff[f] = total;
            total += dpv[f] * (int64_t)frames[f].h;
            if (!frames_on_device && chans(f) == 3) {
                roff[f] = rtotal;
                rtotal += round_up(round_up(3LL * frames[f].w, 16) * frames[f].h, 256);
            }
        }
        total = round_up(total, fa);
        if (total) {
            const void* old_p = sl.frames.p;
            const size_t old_bytes = sl.frames.bytes;
            CU(sl.frames.ensure((size_t)total));
            if (sl.frames.p != old_p && old_p)         // cudaFree above waited for all work
                drop_textures(ctx, old_p, old_bytes);
        }
        if (rtotal) CU(sl.rgb.ensure((size_t)rtotal));
        uint8_t* gbuf = sl.frames.as<uint8_t>();
        for (int f = 0; f < n; ++f) {
            if (foff[f] < 0) {
                fi[f] = FrameInfo{frames[f].data, frames[f].pitch, frames[f].w, frames[f].h};
                continue;
            }
            const int64_t dp = dpv[f];
            fi[f] = FrameInfo{gbuf + foff[f], dp, frames[f].w, frames[f].h};
            if (chans(f) == 3) {
                const bool staged = !frames_on_device;
                jobs[n_jobs++] = GrayJob{staged ? sl.rgb.as<uint8_t>() + roff[f] : frames[f].data,
                                         staged ? round_up(3LL * frames[f].w, 16) : frames[f].pitch,
                                         gbuf + foff[f], dp, frames[f].w, frames[f].h};
            }
        }
        cudaStream_t cs = frames_on_device ? ctx->stream : ctx->copy_stream;
        if (!frames_on_device) {
            // the H2D starts after the work the caller enqueued on the ctx stream so far (e.g. a
            // D2H that fills these pinned host frames), as ccnn_set_stream promises
            CU(cudaEventRecord(sl.ev_user, ctx->stream));
            CU(cudaStreamWaitEvent(ctx->copy_stream, sl.ev_user, 0));
            // the previous batch of this slot (k - kSlots) read these buffers until its end event
            if (sl.used) CU(cudaStreamWaitEvent(ctx->copy_stream, sl.ev[6], 0));
        }
        CU(cudaEventRecord(sl.ev[0], cs));
        if (!frames_on_device) {
            int f = 0;
            while (f < n) {
                if (chans(f) == 3) {                   // host RGB -> staging
                    CU(cudaMemcpy2DAsync(sl.rgb.as<uint8_t>() + roff[f], round_up(3LL * frames[f].w, 16),
                                         frames[f].data, frames[f].pitch, 3 * (size_t)frames[f].w,
                                         frames[f].h, cudaMemcpyHostToDevice, cs));
                    ++f;
                    continue;
                }
                // one copy for every run of equally-sized gray frames laid out back to back (in
                // host memory and, by the layout above, in the slot buffer)
                int g = f + 1;
                const int64_t dp = dpv[f];
                while (g < n && chans(g) == 1 && frames[g].w == frames[f].w &&
                       frames[g].h == frames[f].h && frames[g].pitch == frames[f].pitch &&
                       frames[g].data == frames[f].data + (int64_t)(g - f) * frames[f].h * frames[f].pitch &&
                       foff[g] == foff[f] + (int64_t)(g - f) * dp * frames[f].h)
                    ++g;
                const int64_t rows = (int64_t)frames[f].h * (g - f);
                if (dp == frames[f].pitch)             // linear: up to the run's last pixel
                    CU(cudaMemcpyAsync(gbuf + foff[f], frames[f].data, (size_t)(dp * (rows - 1) + frames[f].w),
                                       cudaMemcpyHostToDevice, cs));
                else
                    CU(cudaMemcpy2DAsync(gbuf + foff[f], dp, frames[f].data, frames[f].pitch, frames[f].w,
                                         (size_t)rows, cudaMemcpyHostToDevice, cs));
                f = g;
            }
        }
        if (n_jobs) {
            CU(sl.jobs.ensure(sizeof(GrayJob) * n_jobs));
            CU(cudaMemcpyAsync(sl.jobs.p, jobs, sizeof(GrayJob) * n_jobs, cudaMemcpyHostToDevice, cs));
            launch_to_gray(sl.jobs.as<GrayJob>(), n_jobs, ctx->sm_count, cs);
            CU(cudaGetLastError());
        }
        CU(cudaEventRecord(sl.ev[1], cs));
        if (!frames_on_device) CU(cudaStreamWaitEvent(s, sl.ev[1], 0));
    }
    sl.n_jobs = n_jobs;
    if (ctx->tex_cache.size() > 4096) {                // bounded cache: rebuild
        CU(cudaStreamSynchronize(s));
        CU(cudaStreamSynchronize(ctx->pyr_stream));
        CU(cudaStreamSynchronize(ctx->tail));
        drop_textures(ctx, nullptr, 0);
    }
    // texture-gather pyramid only on request: measured slower than byte gathers on B200
    // (tld4 on 8-bit texels is TEX-throughput bound; K1)
    bool use_tex = (ctx->debug & CCNN_DEBUG_PYR_TEX) != 0;
    for (int f = 0; f < n; ++f) {
        fi[f].level0 = ctx->frame_level0[f];
        fi[f].nlevels = ctx->frame_nlevels[f];
        fi[f].tiles = ctx->frame_tiles[f];
        fi[f].tile_off = ctx->frame_tile_off[f];
        fi[f].tiles_g = ctx->frame_tiles_g[f];
        fi[f].tex = use_tex ? frame_texture(ctx, fi[f].data, fi[f].w, fi[f].h, fi[f].pitch) : 0;
        use_tex = use_tex && fi[f].tex != 0;
    }
    // pyramid on its own stream: after the frames are in place and after the previous batch
    // of this slot finished reading the slot's level arena (its stage 1); it overlaps the
    // previous batch's stage 1 .. NMS on the compute stream
    cudaStream_t ps = ctx->pyr_stream;
    CU(cudaStreamWaitEvent(ps, sl.ev[1], 0));
    if (sl.used) CU(cudaStreamWaitEvent(ps, sl.ev[4], 0));
    if (sl.fi_dev_p != sl.finfo.p || sl.fi_dev.size() != (size_t)n ||
        std::memcmp(sl.fi_dev.data(), fi, sizeof(FrameInfo) * n) != 0) {
        sl.fi_dev_p = nullptr;
        CU(cudaMemcpyAsync(sl.finfo.p, fi, sizeof(FrameInfo) * n, cudaMemcpyHostToDevice, ps));
        sl.fi_dev.assign(fi, fi + n);
        sl.fi_dev_p = sl.finfo.p;
    }
    const FrameInfo* dfi = sl.finfo.as<FrameInfo>();
    CU(cudaEventRecord(sl.ev[2], ps));
    if (ctx->epoch == nullptr && std::getenv("CCNN_TIMELINE")) {
        CU(cudaEventCreate(&ctx->epoch));
        CU(cudaEventRecord(ctx->epoch, ps));
    }
    // CCNN_EXP_SKIP_PYRAMID=1 (timing experiments only, results invalid unless every batch
    // repeats the slot's previous frames): no pyramid launch, stage 1 reads the slot's old levels
    static const bool exp_skip_pyr = std::getenv("CCNN_EXP_SKIP_PYRAMID") != nullptr;
    sl.pyr_launches = (exp_skip_pyr && sl.used) ? 0 :
        launch_pyramid(dfi, n, ctx->pyr_tiles, ctx->pyr_class_max, ctx->all_safe, use_tex,
                       sl.arena.as<uint8_t>(), ctx->d_levels.as<LevelInfo>(),
                       ctx->d_ptiles.as<uint32_t>(), ctx->d_tabs.as<uint32_t>(), ps);
    CU(cudaEventRecord(sl.ev[3], ps));
    // stage 1 on the compute stream once the slot's previous batch has finished with the
    // slot's queue / scratch (its tail) and this batch's pyramid is done
    Ctrl* dctrl = sl.ctrl.as<Ctrl>();
    if (sl.used) CU(cudaStreamWaitEvent(s, sl.ev[6], 0));
    CU(cudaMemsetAsync(dctrl, 0, sizeof(Ctrl), s));
    CU(cudaStreamWaitEvent(s, sl.ev[3], 0));
    CU(cudaEventRecord(sl.ev[7], s));
    if (ctx->s1_tc)
        launch_stage1_tc(ctx->w1, ctx->T1, ctx->s1_bmats.as<uint16_t>(), sl.arena.as<uint8_t>(),
                         ctx->d_levels.as<LevelInfo>(), ctx->d_tasks.as<S1Task>(), ctx->d_cta_first.as<int32_t>(),
                         (int)ctx->cta_first.size() - 1, sl.cands.as<S1Cand>(), cand_cap, dctrl,
                         dbg1 ? ctx->dbg_map.as<float>() : nullptr, s);
    else
        launch_stage1(ctx->w1, ctx->T1, sl.arena.as<uint8_t>(), ctx->d_levels.as<LevelInfo>(),
                      ctx->d_tasks.as<S1Task>(), ctx->d_cta_first.as<int32_t>(),
                      (int)ctx->cta_first.size() - 1, sl.cands.as<S1Cand>(), cand_cap, dctrl,
                      dbg1 ? ctx->dbg_map.as<float>() : nullptr, s);
    CU(cudaEventRecord(sl.ev[4], s));
    // selective unit + NMS + readback on the tail stream: they overlap the next batch's stage 1
    cudaStream_t ts = ctx->tail;
    CU(cudaStreamWaitEvent(ts, sl.ev[4], 0));
    CU(cudaEventRecord(sl.ev[8], ts));
    // CCNN_EXP_SKIP_TAIL=1 (timing experiments only, results invalid): no selective unit / NMS
    static const bool exp_skip_tail = std::getenv("CCNN_EXP_SKIP_TAIL") != nullptr;
    if (!exp_skip_tail) {
    launch_selective_cnn2_tc(ctx->sel_consts, ctx->sp, ctx->sel_bmats.as<uint16_t>(), dfi,
                             ctx->d_levels.as<LevelInfo>(), sl.cands.as<S1Cand>(), cand_cap,
                             sl.resp2.as<float>(), sl.epatch.as<uint8_t>(), dctrl,
                             ctx->sel_grid > 0 ? ctx->sel_grid : ctx->sm_count, ts);
    launch_selective(ctx->w3, ctx->sp, ctx->d_levels.as<LevelInfo>(), sl.cands.as<S1Cand>(), cand_cap,
                     sl.resp2.as<float>(), sl.epatch.as<uint8_t>(), sl.selout.as<SelOut>(),
                     dbg1 ? ctx->dbg_resp.as<float>() : nullptr, sl.acc.as<AccBox>(), dctrl,
                     ctx->cnn3_grid > 0 ? ctx->cnn3_grid : ctx->sm_count, ts);
    CU(cudaEventRecord(sl.ev[5], ts));
    launch_nms(sl.acc.as<AccBox>(), dctrl, n, ctx->min_cluster, sl.staging.as<OutBox>(),
               sl.counts.as<int32_t>(), sl.out.as<OutBox>(), ts);
    } else {
        CU(cudaEventRecord(sl.ev[5], ts));
    }
    CU(cudaGetLastError());
    CU(cudaMemcpyAsync(sl.h_ctrl, dctrl, sizeof(Ctrl), cudaMemcpyDeviceToHost, ts));
    CU(cudaEventRecord(sl.ev[6], ts));
    sl.used = true;
    ctx->next_slot = (ctx->next_slot + 1) % ccnn_ctx::kSlots;
    ctx->inflight++;
    return CCNN_OK;
}

int ccnn_submit(ccnn_ctx* ctx, const uint8_t* frames, int n, int w, int h, int64_t pitch,
                int frames_on_device, int min_face, float scale_step, int timed)
{
    if (!ctx) return CCNN_E_ARG;
    if (!frames) return fail(ctx, CCNN_E_ARG, "NULL frames");
    if (n <= 0 || n > ctx->max_batch) return fail(ctx, CCNN_E_ARG, "n out of [1, max_batch]");
    std::vector<ccnn_frame> fr(n);
    for (int f = 0; f < n; ++f) fr[f] = ccnn_frame{frames + (int64_t)f * h * pitch, w, h, pitch};
    return ccnn_submit_frames(ctx, fr.data(), n, frames_on_device, min_face, scale_step, timed);
}

int ccnn_collect(ccnn_ctx* ctx, ccnn_box* boxes, int64_t box_cap, int64_t* n_boxes, ccnn_stats* stats)
{
    if (!ctx) return CCNN_E_ARG;
    if (!n_boxes || (box_cap > 0 && !boxes)) return fail(ctx, CCNN_E_ARG, "NULL n_boxes / boxes");
    if (ctx->inflight == 0) return fail(ctx, CCNN_E_STATE, "no batch in flight");
    CU(cudaSetDevice(ctx->device));
    const int si = (ctx->next_slot - ctx->inflight + ccnn_ctx::kSlots) % ccnn_ctx::kSlots;   // oldest in-flight slot
    ccnn_ctx::Slot& sl = ctx->slot[si];
    ctx->inflight--;
    ctx->last_slot = si;
    ctx->last_valid = false;
    CU(cudaEventSynchronize(sl.ev[6]));
    if (stats) {
        std::memset(stats, 0, sizeof(*stats));
        stats->windows = sl.windows;
    }
    ctx->last_n = sl.n;
    if (sl.empty) {
        *n_boxes = 0;
        ctx->last_cands = 0;
        ctx->last_nout = 0;
        ctx->last_valid = true;
        return CCNN_OK;
    }
    const Ctrl& hc = *sl.h_ctrl;
    ctx->last_cands = hc.n_cand;
    if (hc.n_cand > sl.cand_cap)
        return fail(ctx, CCNN_E_QUEUE, "stage-1 survivor queue overflow: " + std::to_string(hc.n_cand) +
                                           " > capacity " + std::to_string(sl.cand_cap));
    if (hc.nms_overflow)
        return fail(ctx, CCNN_E_QUEUE, "more than 4096 accepted regions in one frame");
    ctx->last_valid = true;
    if (stats) {
        stats->stage1 = hc.n_cand;
        stats->stage2 = hc.n_stage2;
        stats->stage3 = hc.n_stage3;
        stats->nms = hc.n_out;
        stats->kernel_launches = 4 + sl.pyr_launches + (sl.n_jobs ? 1 : 0);
        stats->s1_mma_flops = sl.s1_mma_flops;
        const int from[5] = {0, 2, 7, 8, 5}, to[5] = {1, 3, 4, 5, 6};
        for (int k = 0; k < 5; ++k) {
            float t = 0.f;
            cudaEventElapsedTime(&t, sl.ev[from[k]], sl.ev[to[k]]);
            stats->ms[k] = t;
        }
    }
    if (ctx->epoch && sl.timed) {          // timeline diagnostics (ms since the first pyramid)
        const int ids[8] = {2, 3, 7, 4, 5, 6, 0, 1};
        float t[8] = {};
        for (int k = 0; k < 8; ++k) cudaEventElapsedTime(&t[k], ctx->epoch, sl.ev[ids[k]]);
        std::fprintf(stderr, "ccnn timeline batch %lld: pyr %.4f-%.4f s1 %.4f-%.4f sel-%.4f end %.4f h2d %.4f-%.4f\n",
                     (long long)ctx->batch_no, t[0], t[1], t[2], t[3], t[4], t[5], t[6], t[7]);
    }
    ++ctx->batch_no;
    *n_boxes = hc.n_out;
    ctx->last_nout = hc.n_out;
    if ((int64_t)hc.n_out > box_cap)
        return fail(ctx, CCNN_E_CAPACITY, "box_cap too small: need " + std::to_string(hc.n_out));
    if (hc.n_out) {
        static_assert(sizeof(OutBox) == sizeof(ccnn_box), "OutBox mirrors ccnn_box");
        CU(cudaMemcpyAsync(boxes, sl.out.p, sizeof(OutBox) * hc.n_out, cudaMemcpyDeviceToHost,
                           ctx->d2h_stream));
        CU(cudaStreamSynchronize(ctx->d2h_stream));
    }
    return CCNN_OK;
}

int ccnn_detect(ccnn_ctx* ctx, const uint8_t* frames, int n, int w, int h, int64_t pitch,
                int frames_on_device, int min_face, float scale_step, ccnn_box* boxes,
                int64_t box_cap, int64_t* n_boxes, ccnn_stats* stats)
{
    if (!ctx) return CCNN_E_ARG;
    if (!n_boxes || (box_cap > 0 && !boxes)) return fail(ctx, CCNN_E_ARG, "NULL n_boxes / boxes");
    if (ctx->inflight) return fail(ctx, CCNN_E_STATE, "ccnn_detect with batches in flight");
    const int rc = ccnn_submit(ctx, frames, n, w, h, pitch, frames_on_device, min_face, scale_step,
                               stats != nullptr);
    if (rc != CCNN_OK) return rc;
    return ccnn_collect(ctx, boxes, box_cap, n_boxes, stats);
}

int ccnn_detect_frames(ccnn_ctx* ctx, const ccnn_frame* frames, int n, int frames_on_device,
                       int min_face, float scale_step, ccnn_box* boxes, int64_t box_cap,
                       int64_t* n_boxes, ccnn_stats* stats)
{
    if (!ctx) return CCNN_E_ARG;
    if (!n_boxes || (box_cap > 0 && !boxes)) return fail(ctx, CCNN_E_ARG, "NULL n_boxes / boxes");
    if (ctx->inflight) return fail(ctx, CCNN_E_STATE, "ccnn_detect_frames with batches in flight");
    const int rc = ccnn_submit_frames(ctx, frames, n, frames_on_device, min_face, scale_step,
                                      stats != nullptr);
    if (rc != CCNN_OK) return rc;
    return ccnn_collect(ctx, boxes, box_cap, n_boxes, stats);
}

int ccnn_last_boxes(ccnn_ctx* ctx, ccnn_box* boxes, int64_t box_cap, int64_t* n_boxes)
{
    if (!ctx || !n_boxes || (box_cap > 0 && !boxes)) return CCNN_E_ARG;
    if (!ctx->last_valid) return fail(ctx, CCNN_E_STATE, "no completed detect");
    *n_boxes = ctx->last_nout;
    if ((int64_t)ctx->last_nout > box_cap)
        return fail(ctx, CCNN_E_CAPACITY, "box_cap too small: need " + std::to_string(ctx->last_nout));
    if (ctx->last_nout) {
        CU(cudaSetDevice(ctx->device));
        CU(cudaMemcpyAsync(boxes, ctx->slot[ctx->last_slot].out.p, sizeof(OutBox) * ctx->last_nout,
                           cudaMemcpyDeviceToHost, ctx->d2h_stream));
        CU(cudaStreamSynchronize(ctx->d2h_stream));
    }
    return CCNN_OK;
}

int ccnn_debug_levels(ccnn_ctx* ctx, int frame, double* sigma, int32_t* lw, int32_t* lh, int cap)
{
    if (!ctx) return CCNN_E_ARG;
    if (frame < 0 || frame >= (int)ctx->frame_nlevels.size())
        return fail(ctx, CCNN_E_ARG, "frame out of range");
    const int L = ctx->frame_nlevels[frame], l0 = ctx->frame_level0[frame];
    for (int l = 0; l < L && l < cap; ++l) {
        if (sigma) sigma[l] = ctx->levels[l0 + l].sigma;
        if (lw) lw[l] = ctx->levels[l0 + l].lw;
        if (lh) lh[l] = ctx->levels[l0 + l].lh;
    }
    return L;
}

// the level (frame, level) of the last batch, or nullptr
static const LevelInfo* debug_level_info(ccnn_ctx* ctx, int frame, int level)
{
    if (frame < 0 || frame >= ctx->last_n || frame >= (int)ctx->frame_nlevels.size()) return nullptr;
    if (level < 0 || level >= ctx->frame_nlevels[frame]) return nullptr;
    return &ctx->levels[ctx->frame_level0[frame] + level];
}

int ccnn_debug_level(ccnn_ctx* ctx, int frame, int level, uint8_t* out, int64_t cap)
{
    if (!ctx || !out) return CCNN_E_ARG;
    if (!ctx->last_valid) return fail(ctx, CCNN_E_STATE, "no completed detect");
    const LevelInfo* L = debug_level_info(ctx, frame, level);
    if (!L) return fail(ctx, CCNN_E_ARG, "frame/level out of range");
    if (cap < (int64_t)L->lw * L->lh) return fail(ctx, CCNN_E_CAPACITY, "cap < lw*lh");
    CU(cudaSetDevice(ctx->device));
    CU(cudaMemcpy2DAsync(out, L->lw, ctx->slot[ctx->last_slot].arena.as<uint8_t>() + L->offset, L->pitch, L->lw, L->lh,
                         cudaMemcpyDeviceToHost, ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
    return CCNN_OK;
}

int ccnn_debug_stage1_map(ccnn_ctx* ctx, int frame, int level, float* out, int64_t cap)
{
    if (!ctx || !out) return CCNN_E_ARG;
    if (!ctx->last_valid || !(ctx->debug & CCNN_DEBUG_STAGE1))
        return fail(ctx, CCNN_E_STATE, "needs CCNN_DEBUG_STAGE1 before ccnn_detect");
    const LevelInfo* L = debug_level_info(ctx, frame, level);
    if (!L) return fail(ctx, CCNN_E_ARG, "frame/level out of range");
    const int64_t cnt = (int64_t)L->nx * L->ny;
    if (cap < cnt) return fail(ctx, CCNN_E_CAPACITY, "cap < nx*ny");
    CU(cudaSetDevice(ctx->device));
    CU(cudaMemcpyAsync(out, ctx->dbg_map.as<float>() + L->map_off, sizeof(float) * cnt,
                       cudaMemcpyDeviceToHost, ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
    return CCNN_OK;
}

int ccnn_debug_counters(ccnn_ctx* ctx, uint32_t* out, int cap)
{
    if (!ctx || !out) return CCNN_E_ARG;
    const Ctrl* hc = ctx->slot[ctx->last_slot].h_ctrl;
    const int n = (int)(sizeof(hc->pad) / sizeof(uint32_t));
    for (int k = 0; k < n && k < cap; ++k) out[k] = hc->pad[k];
    return n;
}

int ccnn_debug_candidates(ccnn_ctx* ctx, ccnn_candidate* out, int64_t cap, int64_t* n)
{
    if (!ctx || !n) return CCNN_E_ARG;
    if (!ctx->last_valid) return fail(ctx, CCNN_E_STATE, "no completed detect");
    const int64_t cnt = ctx->last_cands;
    *n = cnt;
    if (cnt == 0 || !out) return CCNN_OK;            // count query
    if (cap < cnt) return fail(ctx, CCNN_E_CAPACITY, "cap < candidate count");
    CU(cudaSetDevice(ctx->device));
    std::vector<S1Cand> c(cnt);
    std::vector<SelOut> so(cnt);
    std::vector<float> resp;
    const ccnn_ctx::Slot& ls = ctx->slot[ctx->last_slot];
    CU(cudaMemcpyAsync(c.data(), ls.cands.p, sizeof(S1Cand) * cnt, cudaMemcpyDeviceToHost, ctx->stream));
    CU(cudaMemcpyAsync(so.data(), ls.selout.p, sizeof(SelOut) * cnt, cudaMemcpyDeviceToHost, ctx->stream));
    const bool have_resp = (ctx->debug & CCNN_DEBUG_STAGE1) && ctx->dbg_resp.p;
    if (have_resp) {
        resp.resize((size_t)cnt * 100);
        CU(cudaMemcpyAsync(resp.data(), ctx->dbg_resp.p, sizeof(float) * 100 * cnt,
                           cudaMemcpyDeviceToHost, ctx->stream));
    }
    CU(cudaStreamSynchronize(ctx->stream));
    for (int64_t k = 0; k < cnt; ++k) {
        ccnn_candidate& o = out[k];
        std::memset(&o, 0, sizeof(o));
        o.frame = c[k].frame;
        o.level = c[k].level - ctx->frame_level0[c[k].frame];   // global -> per-frame id
        o.ix = c[k].ix;
        o.iy = c[k].iy;
        o.s1 = c[k].s1;
        o.K2 = so[k].K2;
        o.K3 = so[k].K3;
        o.delta = so[k].delta;
        o.cnn3_ran = so[k].cnn3_ran;
        o.score = so[k].score;
        o.bx = so[k].bx;
        o.by = so[k].by;
        o.bw = so[k].bw;
        o.bh = so[k].bh;
        if (have_resp) {
            std::memcpy(o.r2, &resp[k * 100], sizeof(o.r2));
            std::memcpy(o.r3, &resp[k * 100 + 50], sizeof(o.r3));
        }
    }
    return CCNN_OK;
}

int ccnn_debug_group(ccnn_ctx* ctx, const ccnn_box* raw, int64_t n, int n_frames, ccnn_box* out,
                     int64_t cap, int64_t* n_out)
{
    if (!ctx) return CCNN_E_ARG;
    if (!n_out || (n > 0 && !raw) || (cap > 0 && !out) || n < 0 || n > 0x7FFFFFFF)
        return fail(ctx, CCNN_E_ARG, "bad arguments");
    if (n_frames < 1 || n_frames > ctx->max_batch) return fail(ctx, CCNN_E_ARG, "n_frames out of [1, max_batch]");
    if (ctx->inflight) return fail(ctx, CCNN_E_STATE, "ccnn_debug_group with batches in flight");
    std::vector<AccBox> acc((size_t)std::max<int64_t>(n, 1));
    for (int64_t k = 0; k < n; ++k) {
        const ccnn_box& b = raw[k];
        // the NMS kernel holds coordinates as int16 (frames are at most 16384 px)
        if (b.frame < 0 || b.frame >= n_frames || b.x < 0 || b.y < 0 || b.w < 1 || b.h < 1 ||
            (int64_t)b.x + b.w > 32767 || (int64_t)b.y + b.h > 32767 || !std::isfinite(b.score))
            return fail(ctx, CCNN_E_ARG, "raw box out of range");
        acc[k] = AccBox{b.frame, b.x, b.y, b.w, b.h, b.score};
    }
    CU(cudaSetDevice(ctx->device));
    DevBuf d_acc, d_ctrl, d_staging, d_counts, d_out;
    struct Guard {
        DevBuf* b[5];
        ~Guard() { for (DevBuf* x : b) x->release(); }
    } guard{{&d_acc, &d_ctrl, &d_staging, &d_counts, &d_out}};
    CU(d_acc.ensure(sizeof(AccBox) * acc.size()));
    CU(d_ctrl.ensure(sizeof(Ctrl)));
    CU(d_staging.ensure(sizeof(OutBox) * kNmsCap * (size_t)n_frames));
    CU(d_counts.ensure(sizeof(int32_t) * n_frames));
    CU(d_out.ensure(sizeof(OutBox) * acc.size()));
    Ctrl hc{};
    hc.n_acc = (uint32_t)n;
    cudaStream_t s = ctx->comp;
    CU(cudaMemcpyAsync(d_acc.p, acc.data(), sizeof(AccBox) * n, cudaMemcpyHostToDevice, s));
    CU(cudaMemcpyAsync(d_ctrl.p, &hc, sizeof(Ctrl), cudaMemcpyHostToDevice, s));
    launch_nms(d_acc.as<AccBox>(), d_ctrl.as<Ctrl>(), n_frames, ctx->min_cluster, d_staging.as<OutBox>(),
               d_counts.as<int32_t>(), d_out.as<OutBox>(), s);
    CU(cudaGetLastError());
    CU(cudaMemcpyAsync(&hc, d_ctrl.p, sizeof(Ctrl), cudaMemcpyDeviceToHost, s));
    CU(cudaStreamSynchronize(s));
    if (hc.nms_overflow) return fail(ctx, CCNN_E_QUEUE, "more than 4096 raw boxes in one frame");
    *n_out = hc.n_out;
    if ((int64_t)hc.n_out > cap) return fail(ctx, CCNN_E_CAPACITY, "cap < grouped box count");
    if (hc.n_out) {
        CU(cudaMemcpy(out, d_out.p, sizeof(OutBox) * hc.n_out, cudaMemcpyDeviceToHost));
    }
    return CCNN_OK;
}

}  // extern "C"
