/*
 * ccnn.h -- C ABI of the B200-native compact CNN cascade face detector hot path
 * (Kalinovskii & Spitsyn, "Compact Convolutional Neural Network Cascade for Face
 * Detection", arXiv 1508.01292).  Library: paper_1508_01292_b200/libccnn.so.
 *
 * Citations: P:n = PAPER.md line n (section / equation named), S:n = SPEC.md line n,
 * Rk / Ok = readings listed in DESIGN.md.
 *
 * What ccnn_detect computes (Fig. 3), per frame:
 *   1. an image pyramid: sigma_0 = 27/min_face, sigma_{k+1} = sigma_k/scale_step, every
 *      level bilinearly resampled from the original frame (O1-O2);
 *   2. stage 1: CNN1 densely scans every level; each response cell is one 27x31
 *      window at a 4-px step; windows whose response EXCEEDS T1 survive (O4);
 *   3. the selective unit for each survivor: the window with its neighbourhood is read
 *      from the ORIGINAL frame, scaled to 51x55, histogram-equalised and mirrored
 *      (O5-O6); CNN2 and CNN3 give 5x5 response maps on both orientations;
 *      K = number of responses exceeding T2; Eq. 2 (strict, with the
 *      early stop of P:99) or Eq. 3 (weak) decides (O7);
 *   4. NMS: accepted windows mapped back to original pixels are grouped (IoU >= 0.3,
 *      transitive) into the resulting face areas (O8-O9).
 * All CNN arithmetic is fp32 on the GPU ("single precision"); all geometry is
 * integer or IEEE double without contraction, bit-identical to the oracle.
 *
 * Conventions
 *   - every int-returning function returns CCNN_OK (0) or a negative CCNN_E_* code and
 *     records a message readable with ccnn_last_error(ctx);
 *   - a ccnn_ctx belongs to one CUDA device and is NOT thread-safe (one ctx per thread /
 *     stream); all device work is ordered after the ctx stream (ccnn_set_stream);
 *   - the ctx copies everything it is given at create time; the caller owns `frames`,
 *     `boxes` and `stats` buffers.
 */
#ifndef CCNN_H
#define CCNN_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CCNN_ABI_VERSION 5

/* status codes */
#define CCNN_OK          0
#define CCNN_E_ARG      -1  /* bad argument: n<=0, w/h out of range, min_face<1, scale_step<=1, NULL pointer */
#define CCNN_E_ARCH     -2  /* architecture is not R (27x31->1x1 stride 4; 51x55->5x5; final 1 map) */
#define CCNN_E_WEIGHTS  -3  /* weight count mismatch or non-finite weight/threshold */
#define CCNN_E_CAPACITY -4  /* box_cap too small; *n_boxes holds the required count (retry) */
#define CCNN_E_QUEUE    -5  /* survivor queue / per-frame box capacity exceeded (raise queue_capacity) */
#define CCNN_E_CUDA     -6  /* a CUDA runtime call failed */
#define CCNN_E_STATE    -7  /* debug hook called without the data it reads */

/* One layer.  kind 0 = valid conv, stride 1, bias, followed by the Eq. 1
 * activation; kind 1 = 2x2 max-pool, stride 2, floor (reading R2). */
typedef struct {
    int32_t kind;
    int32_t in_maps, out_maps;
    int32_t kw, kh;            /* kernel width x height (pool: 2, 2) */
} ccnn_layer;

/* One network: layers in forward order; weights = for each conv layer its kernels
 * [out][in][kh][kw] followed by bias[out] (S:186 order), float32, n_weights values. */
typedef struct {
    int32_t n_layers;
    const ccnn_layer* layers;
    const float* weights;
    int64_t n_weights;
} ccnn_net;

typedef struct {
    ccnn_net net[3];           /* CNN1, CNN2, CNN3 (Fig. 1 -- reconstructed R, R1) */
    float T1;                  /* stage-1 threshold, survivor iff response > T1       */
    float T2[2];               /* response thresholds for CNN2 / CNN3; equal values
                                  reproduce the paper's single T2                            */
    int32_t Tnn;               /* discrete threshold T_nn == T_m of Eq. 2, >=1 */
    int32_t rule;              /* 0 = Eq. 2 strict, 1 = Eq. 3 weak             */
    int32_t nms_min_cluster;   /* drop groups smaller than this (O9; default 1)               */
    int32_t max_w, max_h;      /* largest frame accepted by ccnn_detect                        */
    int32_t max_batch;         /* largest n accepted by ccnn_detect (1 .. 4096)                */
    int32_t queue_capacity;    /* stage-1 survivor records per frame (S:430 default 4096)     */
    int32_t segment_rows;      /* stage-1 task height in window rows (0 = adaptive)            */
} ccnn_params;

/* A resulting face area in original-image pixels. */
typedef struct {
    int32_t frame;             /* index within the ccnn_detect batch */
    int32_t x, y, w, h;
    float   score;             /* max selective response of the group (O7, O9) */
    int32_t neighbors;         /* number of raw detections merged */
} ccnn_box;

/* Table-1-shaped counts of the last ccnn_detect, plus timings. */
typedef struct {
    int64_t windows;           /* sliding-window positions over all levels and frames */
    int64_t stage1;            /* stage-1 survivors (response > T1) */
    int64_t stage2;            /* survivors with K2 > 0 */
    int64_t stage3;            /* accepted by the decision rule (delta = 1) */
    int64_t nms;               /* resulting boxes */
    float   ms[5];             /* device ms: [0] H2D, [1] pyramid, [2] stage 1,
                                  [3] selective, [4] NMS + output (CUDA events) */
    int64_t kernel_launches;   /* kernels this call launched */
    double  s1_mma_flops;      /* tensor-core work the stage-1 kernel issued for this call
                                  (2 x M x N x K of every tcgen05.mma: hi+lo splits and the
                                  implicit GEMMs' zero taps included); 0 for the legacy kernel */
} ccnn_stats;

typedef struct ccnn_ctx ccnn_ctx;   /* opaque; owns all device state of one detector */

/* Create a detector on `cuda_device`.  Validates the architecture (CCNN_E_ARCH),
 * weights and thresholds (CCNN_E_WEIGHTS) and sizes (CCNN_E_ARG); copies the weights.
 * *out is set only on success. */
int ccnn_create(const ccnn_params* p, int cuda_device, ccnn_ctx** out);

/* Order all later device work of ctx after `cuda_stream` (a cudaStream_t, e.g.
 * torch.cuda.current_stream().cuda_stream; NULL = the legacy default stream): every
 * ccnn_detect / ccnn_submit records an event on this stream (after the work the caller
 * enqueued there, e.g. writing device frames) and the ctx's internal streams (pyramid,
 * stage 1, selective unit + NMS) start after it.  Completion is reported to the host by
 * ccnn_detect / ccnn_collect returning. */
int ccnn_set_stream(ccnn_ctx* ctx, void* cuda_stream);

/* Detect faces in n frames of w x h uint8 grayscale, row pitch `pitch` bytes,
 * frame f at frames + f*h*pitch.  frames_on_device != 0: `frames` is a device pointer
 * on the ctx device; else a host pointer (pinned memory recommended) copied H2D
 * inside the call.  min_face >= 1 (minSize), scale_step > 1 (scaleFactor).
 * On success writes the boxes sorted by (frame, score desc, y, x, w, h) into
 * boxes[0 .. *n_boxes) (host memory) and returns CCNN_OK; when box_cap < required,
 * returns CCNN_E_CAPACITY with *n_boxes = required.  A frame smaller than the window
 * at every scale yields no boxes (not an error).  Synchronous on return.
 * stats may be NULL. */
int ccnn_detect(ccnn_ctx* ctx, const uint8_t* frames, int n, int w, int h, int64_t pitch,
                int frames_on_device, int min_face, float scale_step,
                ccnn_box* boxes, int64_t box_cap, int64_t* n_boxes, ccnn_stats* stats);

/* One frame of a variable-size batch (stills of mixed sizes, e.g.
 * the FDDB benchmark images).  data: w x h pixels, row pitch `pitch` bytes;
 * host or device memory per the call's frames_on_device.  channels: 0 or 1 = 8-bit
 * grayscale (pitch >= w); 3 = interleaved 8-bit R,G,B (pitch >= 3w), converted on
 * the GPU to Rec.601 luma (299 R + 587 G + 114 B + 500) div 1000 (reading I1, SPEC
 * S:216-223) before the pyramid; any other value is CCNN_E_ARG.  reserved must be 0. */
typedef struct {
    const uint8_t* data;
    int32_t w, h;
    int64_t pitch;
    int32_t channels;
    int32_t reserved;
} ccnn_frame;

/* ccnn_detect over n frames of individual sizes: each frame gets its own level table
 * (O1), all levels of all frames share one pyramid / stage-1 / selective / NMS launch.
 * Every frame must satisfy 1 <= w <= max_w, 1 <= h <= max_h; box.frame indexes `frames`.
 * Errors and ownership exactly as ccnn_detect.  ccnn_detect(frames, n, w, h, pitch) is
 * this call with frames[f] = {frames + f*h*pitch, w, h, pitch}. */
int ccnn_detect_frames(ccnn_ctx* ctx, const ccnn_frame* frames, int n, int frames_on_device,
                       int min_face, float scale_step,
                       ccnn_box* boxes, int64_t box_cap, int64_t* n_boxes, ccnn_stats* stats);

/* Streaming form of ccnn_detect (a video stream).
 * ccnn_submit enqueues one batch (same arguments as ccnn_detect) and returns at once: host
 * frames are copied H2D on an internal copy stream into one of three per-ctx frame buffers,
 * so the copy of batch k+1 overlaps the kernels of batch k; each batch's pyramid runs on a
 * low-priority internal stream in the background of the earlier batches' stage 1 .. NMS
 * (high-priority internal stream); both start after an event recorded on the ctx stream at
 * submit time.  Host frames must stay valid (and should be pinned) until the batch is
 * collected; device frames until then too.  At most three batches may be in flight
 * (CCNN_E_STATE otherwise); timed != 0 records the per-stage events reported by
 * ccnn_collect's stats.
 * ccnn_collect waits for the OLDEST in-flight batch and returns its boxes exactly like
 * ccnn_detect (including CCNN_E_CAPACITY + ccnn_last_boxes).  ccnn_detect = submit +
 * collect and is refused while batches are in flight.  Do not change the stream while
 * batches are in flight. */
int ccnn_submit(ccnn_ctx* ctx, const uint8_t* frames, int n, int w, int h, int64_t pitch,
                int frames_on_device, int min_face, float scale_step, int timed);
int ccnn_collect(ccnn_ctx* ctx, ccnn_box* boxes, int64_t box_cap, int64_t* n_boxes,
                 ccnn_stats* stats);
/* Streaming form of ccnn_detect_frames (the ccnn_frame array itself may be reused at
 * once; the pixel data it points to must stay valid until the batch is collected). */
int ccnn_submit_frames(ccnn_ctx* ctx, const ccnn_frame* frames, int n, int frames_on_device,
                       int min_face, float scale_step, int timed);

/* Copy the boxes of the last ccnn_detect / ccnn_collect on ctx (also valid after it
 * returned CCNN_E_CAPACITY, so a caller can fetch the result without detecting again).
 * Valid until the next ccnn_submit / ccnn_detect on ctx: with two batches still in flight
 * that submit reuses the collected batch's output buffer.
 * *n_boxes = the number of boxes; CCNN_E_CAPACITY if box_cap < *n_boxes. */
int ccnn_last_boxes(ccnn_ctx* ctx, ccnn_box* boxes, int64_t box_cap, int64_t* n_boxes);

void ccnn_destroy(ccnn_ctx* ctx);

/* Message of the last failing call on ctx ("" if none; static text if ctx is NULL). */
const char* ccnn_last_error(const ccnn_ctx* ctx);

/* CCNN_ABI_VERSION of the loaded library. */
int ccnn_abi_version(void);

/* ------------------------------------------------------------------------------------
 * Test hooks (not for users).  Enable with ccnn_set_debug BEFORE ccnn_detect; they read
 * device state the last ccnn_detect left behind.
 * ---------------------------------------------------------------------------------- */
#define CCNN_DEBUG_LEVELS   1  /* keep the pyramid levels (already resident)        */
#define CCNN_DEBUG_STAGE1   2  /* also write every stage-1 response to a dense map */
#define CCNN_DEBUG_PYR_TEX  4  /* pyramid by texture gathers (tld4), not byte gathers */
int ccnn_set_debug(ccnn_ctx* ctx, int flags);

/* Level table of frame `frame` of the last submitted batch: up to cap levels, returns
 * that frame's level count (>= 0), or a negative status. */
int ccnn_debug_levels(ccnn_ctx* ctx, int frame, double* sigma, int32_t* lw, int32_t* lh, int cap);

/* Copy level `level` of frame `frame` (lw*lh bytes, row pitch lw) to host `out`. */
int ccnn_debug_level(ccnn_ctx* ctx, int frame, int level, uint8_t* out, int64_t cap);

/* Copy the dense stage-1 response map (ny x nx fp32) of (frame, level);
 * needs CCNN_DEBUG_STAGE1. */
int ccnn_debug_stage1_map(ccnn_ctx* ctx, int frame, int level, float* out, int64_t cap);

/* One stage-1 survivor with its selective-unit outcome (a5 + a6-a8 of DESIGN.md). */
typedef struct {
    int32_t frame, level, ix, iy;  /* window column j / row i on `level` */
    float   s1;                    /* stage-1 response */
    int32_t K2, K3, delta, cnn3_ran;
    float   score;
    float   r2[50], r3[50];        /* [orientation E, M][5x5] responses; r3 zero if not run */
    int32_t bx, by, bw, bh;        /* raw box (O8) */
} ccnn_candidate;

/* Device profiling counters of the last detect (kernel-build dependent; zeros unless
 * built with -DS1_PROFILE): up to cap words into out, returns the count. */
int ccnn_debug_counters(ccnn_ctx* ctx, uint32_t* out, int cap);

/* Copy the survivors of the last detect (unordered), *n = total count; out == NULL only
 * queries the count. */
int ccnn_debug_candidates(ccnn_ctx* ctx, ccnn_candidate* out, int64_t cap, int64_t* n);

/* Run the on-device grouping / NMS (step 4; reading O9) alone on n caller-given raw
 * boxes (host array; frame in [0, n_frames), x, y >= 0, w, h >= 1, x + w and y + h <= 32767,
 * finite score; `neighbors` ignored) of n_frames <= max_batch frames, with the ctx's
 * nms_min_cluster.  Writes the groups to out[0 .. *n_out) in the ccnn_detect output order
 * (frame, score desc, y, x, w, h).  CCNN_E_QUEUE if a frame has more than 4096 raw boxes,
 * CCNN_E_CAPACITY if cap < *n_out, CCNN_E_STATE while batches are in flight.  Synchronous;
 * uses temporary device buffers. */
int ccnn_debug_group(ccnn_ctx* ctx, const ccnn_box* raw, int64_t n, int n_frames, ccnn_box* out,
                     int64_t cap, int64_t* n_out);

#ifdef __cplusplus
}
#endif
#endif /* CCNN_H */
