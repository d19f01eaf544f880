/*
 * ccnn_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, obviously-correct CPU oracle of the compact CNN cascade hot path
 * (Kalinovskii & Spitsyn, arXiv 1508.01292).  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load it.  It shares no
 * code, header, table or constant with the CUDA path (paper_1508_01292_b200/).
 *
 * Citations: P:n = PAPER.md line n, S:n = SPEC.md line n, Rk / Ok = DESIGN.md
 * readings.  All floating point is IEEE double (compiled -ffp-contract=off);
 * weights are the float32 inputs promoted to double.
 */
#ifndef CCNN_ORACLE_H
#define CCNN_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* one layer: kind 0 = valid conv (stride 1) + bias + Eq.1 activation, kind 1 = 2x2/2 max-pool */
typedef struct { int kind, in_maps, out_maps, kw, kh; } or_layer;
/* weights: per conv layer kernels [out][in][kh][kw] then bias[out] (S:186 order) */
typedef struct { int n_layers; const or_layer* layers; const float* weights; } or_net;

typedef struct { int32_t frame, x, y, w, h; double score; int32_t neighbors; } or_box;

typedef struct {                 /* one stage-1 survivor and its selective-unit result */
    int32_t frame, level, ix, iy; /* window column j, row i on level `level` */
    double s1;                    /* stage-1 score */
    int32_t K2, K3, delta, cnn3_ran;
    double score;                 /* max response of the last net evaluated (O7) */
    double r2[50], r3[50];        /* CNN2 / CNN3 responses: [orientation][5x5], E then M */
    int32_t bx, by, bw, bh;       /* raw box in original-image pixels (O8) */
} or_cand;

typedef struct {
    float T1;        /* stage-1 threshold, strict > */
    float T2[2];     /* CNN2 / CNN3 response thresholds */
    int32_t Tnn;     /* Eq.2 discrete threshold */
    int32_t rule;    /* 0 = Eq.2 strict, 1 = Eq.3 weak */
    int32_t nms_min_cluster; /* O9, default 1 */
} or_params;

typedef struct { int64_t windows, stage1, stage2, stage3, nms; } or_stats;

/* ---- nnkernel ---- */
double or_activation(double x);
int  or_conv2d_valid(const double* in, int in_maps, int w, int h, const float* kern,
                     const float* bias, int out_maps, int kw, int kh, double* out);
void or_activate_maps(double* m, long n);
void or_pool2(const double* in, int maps, int w, int h, double* out);
long or_param_count(const or_net* net);
int  or_forward_shape(const or_net* net, int w, int h, int* ow, int* oh, int* omaps);
int  or_forward(const or_net* net, const double* in, int w, int h, double* out,
                int* ow, int* oh, int* omaps);
int  or_receptive_field(const or_net* net, int* rw, int* rh);
int  or_output_stride(const or_net* net);

/* ---- pyramid ---- */
int  or_level_table(int W, int H, int min_face, float scale_step, int win_w, int win_h,
                    int max_levels, double* sigma, int* lw, int* lh);
void or_resample(const uint8_t* src, int W, int H, long pitch, double sigma,
                 int lw, int lh, uint8_t* dst);
double or_normalise(uint8_t v);

/* ---- stage 1 ---- */
double or_stage1_window(const or_net* cnn1, const uint8_t* level, int lw, int lh, int i, int j);
int  or_stage1_dense(const or_net* cnn1, const uint8_t* level, int lw, int lh, double* map);
int  or_window_grid(int lw, int lh, int* nx, int* ny);

/* ---- selective unit ---- */
void or_extract_patch(const uint8_t* frame, int W, int H, long pitch, double sigma,
                      int i, int j, uint8_t* patch);
void or_equalize(const uint8_t* in, int n, uint8_t* out);
void or_mirror(const uint8_t* in, int w, int h, uint8_t* out);
int  or_decision(int K2, int K3, int Tnn, int rule);
void or_classify(const or_net* cnn2, const or_net* cnn3, const uint8_t* patch,
                 const or_params* p, or_cand* c);
void or_raw_box(double sigma, int i, int j, int32_t* x, int32_t* y, int32_t* w, int32_t* h);

/* ---- NMS / grouping ---- */
int  or_iou_edge(const or_box* a, const or_box* b);
int  or_group(const or_box* in, int n, int min_cluster, or_box* out);

/* ---- full pipeline for a batch of frames (Fig. 3) ----
 * dense != 0 uses or_stage1_dense (the paper's dense scan) instead of the per-window
 * definition; the two are pinned equal by tests.  n_threads <= 0 means all cores.
 * cands/boxes are malloc'ed; free with or_free.  Returns 0, or <0 on error. */
int  or_detect(const or_net nets[3], const uint8_t* frames, int n, int W, int H, long pitch,
               int min_face, float scale_step, const or_params* p, int dense, int n_threads,
               or_cand** cands, int64_t* n_cands, or_box** boxes, int64_t* n_boxes,
               or_stats* stats);
void or_free(void* p);

#ifdef __cplusplus
}
#endif
#endif
