// nms.cu -- grouping / NMS of accepted regions on device (K4).
//
// PAPER.md §3.3: "The last stage of the pipeline detector is Non-Maximum
// Suppression (NMS) algorithm, which aggregates the found regions to form the resulting
// areas of faces localization."  No parameters are given; reading O9 (SPEC S:332,
// S:357): transitive grouping of the raw boxes whose IoU >= 0.3 (exact integer test
// 10*inter >= 3*union), components smaller than nms_min_cluster dropped, per component
// the coordinate mean rounded half up ((2*sum + n) div 2n), the max score, neighbours =
// size; output sorted by (frame, score desc, y, x, w, h).  Integer sums make the result
// independent of the (nondeterministic) order in which accepted boxes arrive.
//
// One CTA per frame, everything in shared memory: the frame's boxes are bitonic-sorted by
// x so each box only tests the contiguous run of later boxes that start inside its width
// (all-pairs was O(n^2) and instruction-bound on cluttered frames), a warp per box; lock-free union-find
// (hook the larger root under the smaller, path splitting), shared-memory atomics for the
// per-component sums, rank sort in shared memory.  The last CTA to finish (ticket) compacts all frames'
// results into one array.
#include "ccnn_internal.h"

namespace ccnn {
namespace {

constexpr int kNmsThreads = 1024;          // (512: C5 NMS 0.112 ms, 1024: 0.096 ms per 16 frames)

struct NmsSmem {
    short4 box[kNmsCap];         // x, y, w, h of this frame's raw boxes (sorted by x)
    float score[kNmsCap];
    uint32_t key[kNmsCap];       // sort keys: x << 16 | arrival slot (later: group sizes)
    int parent[kNmsCap];
    int sx[kNmsCap], sy[kNmsCap], sw[kNmsCap], sh[kNmsCap], cnt[kNmsCap];
    int best[kNmsCap];           // order-preserving int image of the max score
    int n, m, is_last;
};

__device__ __forceinline__ int f2ord(float f)
{
    const int i = __float_as_int(f);
    return i >= 0 ? i : i ^ 0x7FFFFFFF;
}
__device__ __forceinline__ float ord2f(int i) { return __int_as_float(i >= 0 ? i : i ^ 0x7FFFFFFF); }

__device__ __forceinline__ bool iou_edge(short4 a, short4 b)
{
    const long long ix = (long long)min(a.x + a.z, b.x + b.z) - max(a.x, b.x);
    const long long iy = (long long)min(a.y + a.w, b.y + b.w) - max(a.y, b.y);
    if (ix <= 0 || iy <= 0) return false;
    const long long inter = ix * iy;
    const long long uni = (long long)a.z * a.w + (long long)b.z * b.w - inter;
    return 10 * inter >= 3 * uni;
}

// Invariant: parent[x] <= x (roots are only hooked under smaller roots), so following
// parents strictly decreases the index; path halving (parent[k] = grandparent) keeps the
// invariant, so concurrent halving writes are benign.  Without it, dense clutter graphs
// built parent chains hundreds long (C5: 3.4 ms per 16 frames).
__device__ __forceinline__ int find_root(int* parent, int k)
{
    volatile int* vp = parent;
    int p = vp[k];
    while (p != k) {                 // path splitting: every visited node skips to its grandparent
        const int gp = vp[p];
        if (gp != p) atomicMin(&parent[k], gp);   // monotone (parent[x] <= x): benign, atomic
        k = p;
        p = gp;
    }
    return k;
}

__device__ __forceinline__ void unite(int* parent, int a, int b)
{
    for (;;) {
        a = find_root(parent, a);
        b = find_root(parent, b);
        if (a == b) return;
        if (a < b) { const int t = a; a = b; b = t; }       // hook larger root under smaller
        if (atomicCAS(&parent[a], a, b) == a) return;
    }
}

// total order: score desc, y, x, w, h, then slot (ties only between identical boxes)
__device__ __forceinline__ bool before(const OutBox& a, int ia, const OutBox& b, int ib)
{
    if (a.score != b.score) return a.score > b.score;
    if (a.y != b.y) return a.y < b.y;
    if (a.x != b.x) return a.x < b.x;
    if (a.w != b.w) return a.w < b.w;
    if (a.h != b.h) return a.h < b.h;
    return ia < ib;
}

__global__ void __launch_bounds__(kNmsThreads) nms_kernel(
    const AccBox* __restrict__ acc, Ctrl* __restrict__ ctrl, const int n_frames,
    const int min_cluster, OutBox* __restrict__ staging, int32_t* __restrict__ frame_counts,
    OutBox* __restrict__ out)
{
    extern __shared__ __align__(16) unsigned char sraw[];
    NmsSmem& sm = *reinterpret_cast<NmsSmem*>(sraw);
    const int tid = threadIdx.x;
    const int f = blockIdx.x;
    const int n_acc = (int)*(volatile uint32_t*)&ctrl->n_acc;
    if (tid == 0) { sm.n = 0; sm.m = 0; }
    __syncthreads();
    for (int k = tid; k < n_acc; k += kNmsThreads) {
        const AccBox b = acc[k];
        if (b.frame != f) continue;
        const int s = atomicAdd(&sm.n, 1);
        if (s < kNmsCap) {
            sm.box[s] = make_short4((short)b.x, (short)b.y, (short)b.w, (short)b.h);
            sm.score[s] = b.score;
        }
    }
    __syncthreads();
    const int n = sm.n;
    // staging per frame: kNmsCap slots for its sorted groups
    OutBox* const st = staging + (int64_t)f * kNmsCap;
    if (n > kNmsCap) {
        if (tid == 0) { atomicExch(&ctrl->nms_overflow, 1u); frame_counts[f] = 0; }
    } else {
        for (int i = tid; i < n; i += kNmsThreads) {
            sm.parent[i] = i;
            sm.sx[i] = sm.sy[i] = sm.sw[i] = sm.sh[i] = sm.cnt[i] = 0;
            sm.best[i] = f2ord(-INFINITY);
        }
        __syncthreads();
        // bitonic sort of (x, slot) keys, padded to a power of two with +inf keys
        int np2 = 1;
        while (np2 < n) np2 <<= 1;
        for (int i = tid; i < np2; i += kNmsThreads)
            sm.key[i] = i < n ? ((uint32_t)(uint16_t)sm.box[i].x << 16) | (uint32_t)i : 0xFFFFFFFFu;
        __syncthreads();
        for (int k = 2; k <= np2; k <<= 1)
            for (int j = k >> 1; j > 0; j >>= 1) {
                for (int i = tid; i < np2; i += kNmsThreads) {
                    const int ixj = i ^ j;
                    if (ixj > i) {
                        const uint32_t a = sm.key[i], b = sm.key[ixj];
                        if (((i & k) == 0) == (a > b)) { sm.key[i] = b; sm.key[ixj] = a; }
                    }
                }
                __syncthreads();
            }
        // permute boxes into x order (parent[] as scratch for the scores)
        short4 bx[kNmsCap / kNmsThreads];
        float sc[kNmsCap / kNmsThreads];
#pragma unroll
        for (int q = 0; q < kNmsCap / kNmsThreads; ++q) {
            const int i = tid + q * kNmsThreads;
            if (i < n) { const int src = sm.key[i] & 0xFFFFu; bx[q] = sm.box[src]; sc[q] = sm.score[src]; }
        }
        __syncthreads();
#pragma unroll
        for (int q = 0; q < kNmsCap / kNmsThreads; ++q) {
            const int i = tid + q * kNmsThreads;
            if (i < n) { sm.box[i] = bx[q]; sm.score[i] = sc[q]; }
        }
        __syncthreads();
        // edges of the IoU >= 0.3 graph -> union-find; b > a with x_b >= x_a can only
        // overlap a while x_b < x_a + w_a.  A warp per box a, its lanes test 32 consecutive
        // b at a time (the runs differ a lot in length on cluttered frames: one thread per a
        // left the CTA waiting for its longest run)
        {
            const int lane = tid & 31;
            for (int a = tid >> 5; a < n; a += kNmsThreads / 32) {
                const short4 ba = sm.box[a];
                const int xend = ba.x + ba.z;
                for (int b0 = a + 1; b0 < n; b0 += 32) {
                    const int b = b0 + lane;
                    bool in = false;
                    if (b < n) {
                        const short4 bb = sm.box[b];
                        in = bb.x < xend;
                        if (in && iou_edge(ba, bb)) unite(sm.parent, a, b);
                    }
                    if (__ballot_sync(0xFFFFFFFFu, in) != 0xFFFFFFFFu) break;   // x-sorted: run ended
                }
            }
        }
        __syncthreads();
        for (int i = tid; i < n; i += kNmsThreads) {
            const int r = find_root(sm.parent, i);
            const short4 b = sm.box[i];
            atomicAdd(&sm.sx[r], (int)b.x);
            atomicAdd(&sm.sy[r], (int)b.y);
            atomicAdd(&sm.sw[r], (int)b.z);
            atomicAdd(&sm.sh[r], (int)b.w);
            atomicAdd(&sm.cnt[r], 1);
            atomicMax(&sm.best[r], f2ord(sm.score[i]));
        }
        __syncthreads();
        // the groups, compacted into the (no longer needed) box / score / key arrays: means
        // fit in 16 bits (every coordinate does); key = the group's size
        for (int i = tid; i < n; i += kNmsThreads) {
            if (sm.parent[i] != i || sm.cnt[i] < min_cluster) continue;
            const int c = sm.cnt[i];
            const int g = atomicAdd(&sm.m, 1);
            sm.box[g] = make_short4((short)((2 * sm.sx[i] + c) / (2 * c)), (short)((2 * sm.sy[i] + c) / (2 * c)),
                                    (short)((2 * sm.sw[i] + c) / (2 * c)), (short)((2 * sm.sh[i] + c) / (2 * c)));
            sm.score[g] = ord2f(sm.best[i]);
            sm.key[g] = (uint32_t)c;
        }
        __syncthreads();
        const int m = sm.m;
        for (int i = tid; i < m; i += kNmsThreads) {             // rank sort (shared memory)
            OutBox a;
            a.frame = f;
            a.x = sm.box[i].x; a.y = sm.box[i].y; a.w = sm.box[i].z; a.h = sm.box[i].w;
            a.score = sm.score[i];
            a.neighbors = (int)sm.key[i];
            int r = 0;
            for (int j = 0; j < m; ++j) {
                const short4 bj = sm.box[j];
                OutBox b;
                b.x = bj.x; b.y = bj.y; b.w = bj.z; b.h = bj.w;
                b.score = sm.score[j];
                r += before(b, j, a, i);
            }
            st[r] = a;
        }
        if (tid == 0) frame_counts[f] = m;
    }
    // ---- the last CTA to finish compacts every frame's sorted result ----
    __threadfence();
    __syncthreads();
    if (tid == 0) sm.is_last = (atomicAdd(&ctrl->nms_done, 1u) == (uint32_t)(n_frames - 1));
    __syncthreads();
    if (!sm.is_last) return;
    __threadfence();
    // frame offsets: block-wide exclusive scan of the frame counts, kNmsThreads frames per pass
    // (all loads issued together -- a serial walk over the frames was a chain of dependent
    // global loads, ~1 us each), into sm.sx[] (the frames' first output index) -- then every
    // output box is copied by its own thread (binary search for its frame)
    const int lane = tid & 31, wid = tid >> 5;
    int base = 0;
    for (int g0 = 0; g0 < n_frames; g0 += kNmsThreads) {
        const int g = g0 + tid;
        const int c = g < n_frames ? *(volatile int32_t*)&frame_counts[g] : 0;
        int x = c;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const int t = __shfl_up_sync(0xFFFFFFFFu, x, d);
            if (lane >= d) x += t;
        }
        if (lane == 31) sm.sy[wid] = x;                       // warp totals
        __syncthreads();
        if (wid == 0) {
            int w = lane < kNmsThreads / 32 ? sm.sy[lane] : 0;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const int t = __shfl_up_sync(0xFFFFFFFFu, w, d);
                if (lane >= d) w += t;
            }
            if (lane < kNmsThreads / 32) sm.sw[lane] = w;      // inclusive warp prefix
        }
        __syncthreads();
        const int incl = x + (wid > 0 ? sm.sw[wid - 1] : 0);
        if (g < n_frames) sm.sx[g] = base + incl - c;          // n_frames <= kNmsCap (ccnn_create)
        base += sm.sw[kNmsThreads / 32 - 1];
        __syncthreads();
    }
    const int total = base;
    for (int i = tid; i < total; i += kNmsThreads) {
        int lo = 0, hi = n_frames - 1;                        // last frame with offset <= i
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (sm.sx[mid] <= i) lo = mid; else hi = mid - 1;
        }
        out[i] = staging[(int64_t)lo * kNmsCap + (i - sm.sx[lo])];
    }
    if (tid == 0) ctrl->n_out = (uint32_t)total;
}

}  // namespace

void launch_nms(const AccBox* acc, Ctrl* ctrl, int n_frames, int min_cluster, OutBox* staging,
                int32_t* frame_counts, OutBox* out, cudaStream_t s)
{
    const size_t smem = sizeof(NmsSmem);
    cudaFuncSetAttribute(nms_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    nms_kernel<<<n_frames, kNmsThreads, smem, s>>>(acc, ctrl, n_frames, min_cluster, staging,
                                                   frame_counts, out);
}

}  // namespace ccnn
