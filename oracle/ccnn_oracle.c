/*
 * ccnn_oracle.c -- TEST INFRASTRUCTURE ONLY (see ccnn_oracle.h).
 *
 * A plain CPU implementation of what the compact CNN cascade computes, written to
 * be checked against PAPER.md by eye.  Every function cites the passage it follows.
 * Readings of silent / garbled passages are DESIGN.md R1-R3 and O1-O10.
 *
 * Precision: IEEE double everywhere (build with -ffp-contract=off); decisions that
 * turn a score into an integer (survivor, K counts) are taken in single precision,
 * the paper's precision ("The calculations are carried out using single
 * precision"): the double score is rounded to float and compared with the float
 * threshold.
 *
 * Pins: tests/test_oracle_*.py (run with -m "not gpu").
 */
#include "ccnn_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>
#include <unistd.h>

/* ------------------------------------------------------------------------- */
/* nnkernel                                                                   */
/* ------------------------------------------------------------------------- */

/* Eq. 1 (§3.1): f(x) = 1.7159 * tanh(2x/3) with
 * tanh(y) ~= sgn(y) * (1 - 1 / (1 + |y| + y^2 + 1.41645 * y^4)).  Literal form. */
double or_activation(double x)
{
    double y = 2.0 * x / 3.0;
    double ay = fabs(y);
    double sgn = (y > 0.0) ? 1.0 : ((y < 0.0) ? -1.0 : 0.0);
    double t = sgn * (1.0 - 1.0 / (1.0 + ay + y * y + 1.41645 * (y * y * y * y)));
    return 1.7159 * t;
}

/* Valid 2-D convolution, stride 1 ("Convolution stride is 1 pixel"):
 * out[o][y][x] = bias[o] + sum_i sum_ky sum_kx kern[o][i][ky][kx] * in[i][y+ky][x+kx]
 * (cross-correlation, no kernel flip).  No activation here. */
int or_conv2d_valid(const double* in, int in_maps, int w, int h, const float* kern,
                    const float* bias, int out_maps, int kw, int kh, double* out)
{
    int ow = w - kw + 1, oh = h - kh + 1;
    if (ow < 1 || oh < 1) return -1;
    for (int o = 0; o < out_maps; ++o)
        for (int y = 0; y < oh; ++y)
            for (int x = 0; x < ow; ++x) {
                double s = (double)bias[o];
                for (int i = 0; i < in_maps; ++i)
                    for (int ky = 0; ky < kh; ++ky)
                        for (int kx = 0; kx < kw; ++kx)
                            s += (double)kern[((o * in_maps + i) * kh + ky) * kw + kx] *
                                 in[((long)i * h + (y + ky)) * w + (x + kx)];
                out[((long)o * oh + y) * ow + x] = s;
            }
    return 0;
}

/* Eq. 1 applied element-wise. */
void or_activate_maps(double* m, long n)
{
    for (long k = 0; k < n; ++k) m[k] = or_activation(m[k]);
}

/* 2x2 max-pool, stride 2 ("pooling stride is 2 pixels"); reduction max and
 * floor on odd sizes are readings R2. */
void or_pool2(const double* in, int maps, int w, int h, double* out)
{
    int ow = w / 2, oh = h / 2;
    for (int m = 0; m < maps; ++m)
        for (int y = 0; y < oh; ++y)
            for (int x = 0; x < ow; ++x) {
                const double* p = in + ((long)m * h + 2 * y) * w + 2 * x;
                double v = p[0];
                if (p[1] > v) v = p[1];
                if (p[w] > v) v = p[w];
                if (p[w + 1] > v) v = p[w + 1];
                out[((long)m * oh + y) * ow + x] = v;
            }
}

/* Parameter count ("797, 1,819 and 2,923 parameters"). */
long or_param_count(const or_net* net)
{
    long n = 0;
    for (int l = 0; l < net->n_layers; ++l) {
        const or_layer* L = &net->layers[l];
        if (L->kind == 0) n += (long)L->out_maps * ((long)L->in_maps * L->kw * L->kh + 1);
    }
    return n;
}

/* Forward shape chaining. */
int or_forward_shape(const or_net* net, int w, int h, int* ow, int* oh, int* omaps)
{
    int maps = 1;
    for (int l = 0; l < net->n_layers; ++l) {
        const or_layer* L = &net->layers[l];
        if (L->in_maps != maps) return -1;
        if (L->kind == 0) { w = w - L->kw + 1; h = h - L->kh + 1; maps = L->out_maps; }
        else              { w = w / 2; h = h / 2; }
        if (w < 1 || h < 1) return -1;
    }
    *ow = w; *oh = h; *omaps = maps;
    return 0;
}

/* Forward pass: the layers in order, conv -> Eq.1 activation, pool.
 * The activation follows every conv including the last (reading R3). */
int or_forward(const or_net* net, const double* in, int w, int h, double* out,
               int* ow, int* oh, int* omaps)
{
    int fw, fh, fm;
    if (or_forward_shape(net, w, h, &fw, &fh, &fm) != 0) return -1;
    long cap = 0;
    {   /* largest intermediate */
        int cw = w, ch = h, cm = 1;
        cap = (long)cw * ch;
        for (int l = 0; l < net->n_layers; ++l) {
            const or_layer* L = &net->layers[l];
            if (L->kind == 0) { cw -= L->kw - 1; ch -= L->kh - 1; cm = L->out_maps; }
            else              { cw /= 2; ch /= 2; }
            if ((long)cw * ch * cm > cap) cap = (long)cw * ch * cm;
        }
    }
    double* a = (double*)malloc(sizeof(double) * cap);
    double* b = (double*)malloc(sizeof(double) * cap);
    if (!a || !b) { free(a); free(b); return -2; }
    memcpy(a, in, sizeof(double) * (size_t)w * h);
    int cw = w, ch = h, cm = 1;
    const float* wp = net->weights;
    for (int l = 0; l < net->n_layers; ++l) {
        const or_layer* L = &net->layers[l];
        if (L->kind == 0) {
            const float* kern = wp;
            const float* bias = wp + (long)L->out_maps * L->in_maps * L->kh * L->kw;
            or_conv2d_valid(a, cm, cw, ch, kern, bias, L->out_maps, L->kw, L->kh, b);
            wp = bias + L->out_maps;
            cw -= L->kw - 1; ch -= L->kh - 1; cm = L->out_maps;
            or_activate_maps(b, (long)cw * ch * cm);
        } else {
            or_pool2(a, cm, cw, ch, b);
            cw /= 2; ch /= 2;
        }
        double* t = a; a = b; b = t;
    }
    memcpy(out, a, sizeof(double) * (size_t)cw * ch * cm);
    free(a); free(b);
    *ow = cw; *oh = ch; *omaps = cm;
    return 0;
}

/* Receptive field by inverse dimension chaining: the input size that
 * yields a 1x1 output.  conv: r -> r + k - 1; floor pool: r -> 2r. */
int or_receptive_field(const or_net* net, int* rw, int* rh)
{
    int w = 1, h = 1;
    for (int l = net->n_layers - 1; l >= 0; --l) {
        const or_layer* L = &net->layers[l];
        if (L->kind == 0) { w += L->kw - 1; h += L->kh - 1; }
        else              { w *= 2; h *= 2; }
    }
    *rw = w; *rh = h;
    return 0;
}

/* Output stride = product of pool strides ("4 pixel step"). */
int or_output_stride(const or_net* net)
{
    int s = 1;
    for (int l = 0; l < net->n_layers; ++l) if (net->layers[l].kind == 1) s *= 2;
    return s;
}

/* ------------------------------------------------------------------------- */
/* pyramid                                                                    */
/* ------------------------------------------------------------------------- */

/* Level table, O1 (P:87, P:156 minSize/scaleFactor):
 * sigma_0 = win_w / min_face (upscaling allowed), sigma_{k+1} = sigma_k / scale_step
 * (iterated IEEE division), level k = (floor(W*sigma_k), floor(H*sigma_k)); stop
 * before the first level the whole window does not fit.  scale_step arrives as
 * float (ABI) and is promoted exactly. */
int or_level_table(int W, int H, int min_face, float scale_step, int win_w, int win_h,
                   int max_levels, double* sigma, int* lw, int* lh)
{
    if (min_face < 1 || !(scale_step > 1.0f)) return -1;
    double sf = (double)scale_step;
    double s = (double)win_w / (double)min_face;
    int n = 0;
    while (n < max_levels) {
        int w = (int)floor((double)W * s);
        int h = (int)floor((double)H * s);
        if (w < win_w || h < win_h) break;
        sigma[n] = s; lw[n] = w; lh[n] = h;
        ++n;
        s = s / sf;
    }
    return n;
}

/* Fixed-point bilinear sample coordinate, O2 (reading): pixel centre mapping
 * s = (d + 0.5)/sigma - 0.5 (or a caller-given s), clamp to [0, n-1],
 * i0 = floor(s), i1 = min(i0+1, n-1), a = floor((s - i0) * 2048 + 0.5) in [0, 2048]. */
static void bilin_coord(double s, int n, int* i0, int* i1, int* a)
{
    if (s < 0.0) s = 0.0;
    if (s > (double)(n - 1)) s = (double)(n - 1);
    int f = (int)floor(s);
    *i0 = f;
    *i1 = (f + 1 < n) ? f + 1 : n - 1;
    *a = (int)floor((s - (double)f) * 2048.0 + 0.5);
}

/* Integer blend of four pixels with 11-bit weights, round half up (O2). */
static uint8_t bilin_blend(int p00, int p01, int p10, int p11, int ax, int ay)
{
    long top = (long)p00 * (2048 - ax) + (long)p01 * ax;
    long bot = (long)p10 * (2048 - ax) + (long)p11 * ax;
    long v = (top * (2048 - ay) + bot * ay + (1L << 21)) >> 22;
    return (uint8_t)v;
}

/* Frame ingest of an interleaved 8-bit R,G,B raster (reading I1; the paper assumes
 * grayscale input, "original grayscale image"; SPEC S:216-223 to_grayscale):
 * Rec.601 luma 0.299 R + 0.587 G + 0.114 B rounded to nearest, ties up -- in exact
 * integers (299 R + 587 G + 114 B + 500) div 1000.  dst is w x h, row pitch w. */
void or_to_gray(const uint8_t* rgb, int w, int h, long pitch, uint8_t* dst)
{
    for (int y = 0; y < h; ++y)
        for (int x = 0; x < w; ++x) {
            const uint8_t* p = rgb + (long)y * pitch + 3L * x;
            dst[(long)y * w + x] = (uint8_t)((299L * p[0] + 587L * p[1] + 114L * p[2] + 500L) / 1000L);
        }
}

/* Pyramid level by bilinear resampling of the ORIGINAL frame, O2 (P:121 GPU pyramid;
 * S:228 "bilinear resampling").  dst is lw x lh, row pitch lw. */
void or_resample(const uint8_t* src, int W, int H, long pitch, double sigma,
                 int lw, int lh, uint8_t* dst)
{
    for (int y = 0; y < lh; ++y) {
        int y0, y1, ay;
        bilin_coord(((double)y + 0.5) / sigma - 0.5, H, &y0, &y1, &ay);
        for (int x = 0; x < lw; ++x) {
            int x0, x1, ax;
            bilin_coord(((double)x + 0.5) / sigma - 0.5, W, &x0, &x1, &ax);
            dst[(long)y * lw + x] = bilin_blend(src[y0 * pitch + x0], src[y0 * pitch + x1],
                                                src[y1 * pitch + x0], src[y1 * pitch + x1],
                                                ax, ay);
        }
    }
}

/* Pixel normalisation to [-1, 1], O3 (paper silent, "raw data"). */
double or_normalise(uint8_t v) { return ((double)v - 127.5) / 127.5; }

/* ------------------------------------------------------------------------- */
/* stage 1                                                                    */
/* ------------------------------------------------------------------------- */

/* Window grid on a level (27x31 window, 4-px step). */
int or_window_grid(int lw, int lh, int* nx, int* ny)
{
    if (lw < 27 || lh < 31) { *nx = 0; *ny = 0; return 0; }
    *nx = (lw - 27) / 4 + 1;
    *ny = (lh - 31) / 4 + 1;
    return 0;
}

/* The definition, O4: the stage-1 score of window (i, j) is CNN1 run on
 * the 27x31 crop at pixel offset (4j, 4i) of the level. */
double or_stage1_window(const or_net* cnn1, const uint8_t* level, int lw, int lh, int i, int j)
{
    (void)lh;
    double crop[27 * 31];
    for (int y = 0; y < 31; ++y)
        for (int x = 0; x < 27; ++x)
            crop[y * 27 + x] = or_normalise(level[(long)(4 * i + y) * lw + (4 * j + x)]);
    double out[1];
    int ow, oh, om;
    if (or_forward(cnn1, crop, 27, 31, out, &ow, &oh, &om) != 0 || ow != 1 || oh != 1 || om != 1)
        return NAN;
    return out[0];
}

/* The paper's dense scan ("The first CNN densely scans ... each image of the
 * pyramid"): CNN1 run once over the whole level; cell (i, j) of the response map is
 * window (4j, 4i).  map is ny x nx.  Pinned equal to or_stage1_window by tests. */
int or_stage1_dense(const or_net* cnn1, const uint8_t* level, int lw, int lh, double* map)
{
    int nx, ny, ow, oh, om;
    or_window_grid(lw, lh, &nx, &ny);
    if (nx == 0) return 0;
    double* in = (double*)malloc(sizeof(double) * (size_t)lw * lh);
    double* out = (double*)malloc(sizeof(double) * (size_t)lw * lh);
    if (!in || !out) { free(in); free(out); return -2; }
    for (long k = 0; k < (long)lw * lh; ++k) in[k] = or_normalise(level[k]);
    int rc = or_forward(cnn1, in, lw, lh, out, &ow, &oh, &om);
    if (rc == 0 && (ow != nx || oh != ny || om != 1)) rc = -3;
    if (rc == 0) memcpy(map, out, sizeof(double) * (size_t)nx * ny);
    free(in); free(out);
    return rc;
}

/* ------------------------------------------------------------------------- */
/* selective unit                                                             */
/* ------------------------------------------------------------------------- */

/* Patch extraction, O5 ("read from the original grayscale image together with
 * certain neighborhood and scaled to the size of 51x55").
 * Window centre in original pixels, expanded about it by 51/35 x 55/39 (reading),
 * sampled 51x55 with the O2 fixed-point bilinear rule, edge replication by clamping.
 * patch is 55 rows x 51 columns. */
void or_extract_patch(const uint8_t* frame, int W, int H, long pitch, double sigma,
                      int i, int j, uint8_t* patch)
{
    double cx = ((double)(4 * j) + 13.5) / sigma;
    double cy = ((double)(4 * i) + 15.5) / sigma;
    double rw = (1377.0 / 35.0) / sigma;   /* 27 * 51 / 35 */
    double rh = (1705.0 / 39.0) / sigma;   /* 31 * 55 / 39 */
    double rx = cx - rw / 2.0;
    double ry = cy - rh / 2.0;
    for (int v = 0; v < 55; ++v) {
        int y0, y1, ay;
        double sy = (ry + (((double)v + 0.5) * rh) / 55.0) - 0.5;
        bilin_coord(sy, H, &y0, &y1, &ay);
        for (int u = 0; u < 51; ++u) {
            int x0, x1, ax;
            double sx = (rx + (((double)u + 0.5) * rw) / 51.0) - 0.5;
            bilin_coord(sx, W, &x0, &x1, &ax);
            patch[v * 51 + u] = bilin_blend(frame[y0 * pitch + x0], frame[y0 * pitch + x1],
                                            frame[y1 * pitch + x0], frame[y1 * pitch + x1],
                                            ax, ay);
        }
    }
}

/* Histogram equalisation, O6 ("equalization of its histogram"):
 * out(v) = round_half_up(255 * (cdf(v) - cdf_min) / (N - cdf_min)); a single-valued
 * image is returned unchanged. */
void or_equalize(const uint8_t* in, int n, uint8_t* out)
{
    long hist[256] = {0}, cdf[256];
    for (int k = 0; k < n; ++k) hist[in[k]]++;
    long run = 0, cmin = -1;
    for (int v = 0; v < 256; ++v) {
        run += hist[v];
        cdf[v] = run;
        if (cmin < 0 && hist[v] > 0) cmin = cdf[v];
    }
    if ((long)n == cmin) { memcpy(out, in, (size_t)n); return; }
    long den = 2 * ((long)n - cmin);
    for (int k = 0; k < n; ++k)
        out[k] = (uint8_t)((2 * 255 * (cdf[in[k]] - cmin) + ((long)n - cmin)) / den);
}

/* Mirror reflection about the vertical axis: out(x, y) = in(w-1-x, y). */
void or_mirror(const uint8_t* in, int w, int h, uint8_t* out)
{
    for (int y = 0; y < h; ++y)
        for (int x = 0; x < w; ++x) out[y * w + x] = in[y * w + (w - 1 - x)];
}

/* Decision rule: Eq. 2 (strict) or Eq. 3 (weak); T_m == T_nn (reading,
 * garbled OCR). */
int or_decision(int K2, int K3, int Tnn, int rule)
{
    if (rule == 0) return ((K2 >= Tnn && K3 > 0) || (K2 > 0 && K3 >= Tnn)) ? 1 : 0;
    return (K2 >= Tnn || K3 >= Tnn) ? 1 : 0;
}

/* CNN on a 51x55 uint8 plane -> 25 responses ("response map with a 5x5 size"). */
static void net_on_patch(const or_net* net, const uint8_t* plane, double* r25)
{
    double in[51 * 55];
    for (int k = 0; k < 51 * 55; ++k) in[k] = or_normalise(plane[k]);
    int ow, oh, om;
    if (or_forward(net, in, 51, 55, r25, &ow, &oh, &om) != 0 || ow != 5 || oh != 5 || om != 1)
        for (int k = 0; k < 25; ++k) r25[k] = NAN;
}

/* Selective unit, O6-O7: equalise, mirror, CNN2 on both orientations,
 * K2 = #{r > T2}, stop if CNN2 cannot satisfy the rule, CNN3 likewise,
 * Eq. 2 / Eq. 3.  Score = max response of the last net evaluated. */
void or_classify(const or_net* cnn2, const or_net* cnn3, const uint8_t* patch,
                 const or_params* p, or_cand* c)
{
    uint8_t E[51 * 55], M[51 * 55];
    or_equalize(patch, 51 * 55, E);
    or_mirror(E, 51, 55, M);
    net_on_patch(cnn2, E, c->r2);
    net_on_patch(cnn2, M, c->r2 + 25);
    int K2 = 0;
    double best2 = -INFINITY;
    for (int k = 0; k < 50; ++k) {
        if ((float)c->r2[k] > p->T2[0]) ++K2;
        if (c->r2[k] > best2) best2 = c->r2[k];
    }
    c->K2 = K2; c->K3 = 0; c->cnn3_ran = 0;
    for (int k = 0; k < 50; ++k) c->r3[k] = 0.0;
    int stop = (p->rule == 0) ? (K2 == 0) : (K2 >= p->Tnn);
    if (stop) {
        c->delta = (p->rule == 0) ? 0 : 1;
        c->score = best2;
        return;
    }
    net_on_patch(cnn3, E, c->r3);
    net_on_patch(cnn3, M, c->r3 + 25);
    int K3 = 0;
    double best3 = -INFINITY;
    for (int k = 0; k < 50; ++k) {
        if ((float)c->r3[k] > p->T2[1]) ++K3;
        if (c->r3[k] > best3) best3 = c->r3[k];
    }
    c->K3 = K3; c->cnn3_ran = 1;
    c->delta = or_decision(K2, K3, p->Tnn, p->rule);
    c->score = best3;
}

/* Raw box, O8 (P:101 silent): the stage-1 window mapped back to original pixels,
 * round half up. */
void or_raw_box(double sigma, int i, int j, int32_t* x, int32_t* y, int32_t* w, int32_t* h)
{
    *x = (int32_t)floor((double)(4 * j) / sigma + 0.5);
    *y = (int32_t)floor((double)(4 * i) / sigma + 0.5);
    *w = (int32_t)floor(27.0 / sigma + 0.5);
    *h = (int32_t)floor(31.0 / sigma + 0.5);
}

/* ------------------------------------------------------------------------- */
/* NMS / grouping, O9                               */
/* ------------------------------------------------------------------------- */

/* Edge iff IoU >= 0.3, exactly: 10 * inter >= 3 * union (integers). */
int or_iou_edge(const or_box* a, const or_box* b)
{
    int64_t ix = (int64_t)((a->x + a->w < b->x + b->w) ? a->x + a->w : b->x + b->w) -
                 ((a->x > b->x) ? a->x : b->x);
    int64_t iy = (int64_t)((a->y + a->h < b->y + b->h) ? a->y + a->h : b->y + b->h) -
                 ((a->y > b->y) ? a->y : b->y);
    if (ix <= 0 || iy <= 0) return 0;
    int64_t inter = ix * iy;
    int64_t uni = (int64_t)a->w * a->h + (int64_t)b->w * b->h - inter;
    return 10 * inter >= 3 * uni;
}

static int find_root(int* parent, int k)
{
    while (parent[k] != k) k = parent[k];
    return k;
}

static int box_order(const void* pa, const void* pb)
{
    const or_box* a = (const or_box*)pa;
    const or_box* b = (const or_box*)pb;
    if (a->score != b->score) return (a->score > b->score) ? -1 : 1;
    if (a->y != b->y) return (a->y < b->y) ? -1 : 1;
    if (a->x != b->x) return (a->x < b->x) ? -1 : 1;
    if (a->w != b->w) return (a->w < b->w) ? -1 : 1;
    if (a->h != b->h) return (a->h < b->h) ? -1 : 1;
    return 0;
}

/* Transitive grouping of one frame's raw boxes: connected components of the IoU>=0.3
 * graph; components smaller than min_cluster dropped; per component the coordinate
 * mean rounded half up ((2*sum + n) div (2n)), the max score, neighbors = size;
 * sorted by (score desc, y, x, w, h).  Returns the number of boxes written. */
int or_group(const or_box* in, int n, int min_cluster, or_box* out)
{
    if (n <= 0) return 0;
    int* parent = (int*)malloc(sizeof(int) * n);
    for (int k = 0; k < n; ++k) parent[k] = k;
    for (int a = 0; a < n; ++a)
        for (int b = a + 1; b < n; ++b)
            if (or_iou_edge(&in[a], &in[b])) {
                int ra = find_root(parent, a), rb = find_root(parent, b);
                if (ra != rb) parent[(ra > rb) ? ra : rb] = (ra > rb) ? rb : ra;
            }
    int m = 0;
    for (int r = 0; r < n; ++r) {
        if (find_root(parent, r) != r) continue;
        int64_t sx = 0, sy = 0, sw = 0, sh = 0, cnt = 0;
        double best = -INFINITY;
        for (int k = 0; k < n; ++k)
            if (find_root(parent, k) == r) {
                sx += in[k].x; sy += in[k].y; sw += in[k].w; sh += in[k].h; ++cnt;
                if (in[k].score > best) best = in[k].score;
            }
        if (cnt < min_cluster) continue;
        or_box o;
        o.frame = in[r].frame;
        o.x = (int32_t)((2 * sx + cnt) / (2 * cnt));
        o.y = (int32_t)((2 * sy + cnt) / (2 * cnt));
        o.w = (int32_t)((2 * sw + cnt) / (2 * cnt));
        o.h = (int32_t)((2 * sh + cnt) / (2 * cnt));
        o.score = best;
        o.neighbors = (int32_t)cnt;
        out[m++] = o;
    }
    free(parent);
    qsort(out, (size_t)m, sizeof(or_box), box_order);
    return m;
}

/* ------------------------------------------------------------------------- */
/* full pipeline (Fig. 3; SPEC detect S:338-346)                   */
/* ------------------------------------------------------------------------- */

typedef struct {
    void (*fn)(void* ctx, long k);
    void* ctx;
    long n;
    long next;
} par_job;

static void* par_worker(void* arg)
{
    par_job* J = (par_job*)arg;
    for (;;) {
        long k = __atomic_fetch_add(&J->next, 1, __ATOMIC_RELAXED);
        if (k >= J->n) break;
        J->fn(J->ctx, k);
    }
    return NULL;
}

static int n_cores(void)
{
    long c = sysconf(_SC_NPROCESSORS_ONLN);
    return c < 1 ? 1 : (int)c;
}

/* independent work items k = 0..n-1 on n_threads threads (order-free: each writes its own slot) */
static void par_for(long n, int n_threads, void (*fn)(void*, long), void* ctx)
{
    par_job J = {fn, ctx, n, 0};
    if (n_threads <= 1 || n <= 1) { par_worker(&J); return; }
    if (n_threads > 256) n_threads = 256;
    pthread_t th[256];
    for (int t = 0; t < n_threads; ++t) pthread_create(&th[t], NULL, par_worker, &J);
    for (int t = 0; t < n_threads; ++t) pthread_join(th[t], NULL);
}

typedef struct {
    const or_net* cnn1;
    uint8_t** lev; const int* lw; const int* lh; const int* nx; const int* ny;
    const long* row_first;   /* first task index of each level (rows) */
    int n_levels;
    double** map;            /* per level ny x nx */
    int dense;
} s1_ctx;

static void s1_task(void* vctx, long k)
{
    s1_ctx* C = (s1_ctx*)vctx;
    if (C->dense) {           /* one task per level */
        or_stage1_dense(C->cnn1, C->lev[k], C->lw[k], C->lh[k], C->map[k]);
        return;
    }
    int l = 0;
    while (l + 1 < C->n_levels && C->row_first[l + 1] <= k) ++l;
    int i = (int)(k - C->row_first[l]);
    for (int j = 0; j < C->nx[l]; ++j)
        C->map[l][(long)i * C->nx[l] + j] =
            or_stage1_window(C->cnn1, C->lev[l], C->lw[l], C->lh[l], i, j);
}

typedef struct {
    const or_net* nets; const uint8_t* frame; int W, H; long pitch;
    const double* sigma; const or_params* p; or_cand* cands;
} sel_ctx;

static void sel_task(void* vctx, long k)
{
    sel_ctx* C = (sel_ctx*)vctx;
    or_cand* c = &C->cands[k];
    uint8_t patch[51 * 55];
    double s = C->sigma[c->level];
    or_extract_patch(C->frame, C->W, C->H, C->pitch, s, c->iy, c->ix, patch);
    or_classify(&C->nets[1], &C->nets[2], patch, C->p, c);
    or_raw_box(s, c->iy, c->ix, &c->bx, &c->by, &c->bw, &c->bh);
}

int or_detect(const or_net nets[3], const uint8_t* frames, int n, int W, int H, long pitch,
              int min_face, float scale_step, const or_params* p, int dense, int n_threads,
              or_cand** cands_out, int64_t* n_cands_out, or_box** boxes_out,
              int64_t* n_boxes_out, or_stats* stats)
{
    enum { MAXL = 512 };
    double sigma[MAXL];
    int lw[MAXL], lh[MAXL], nx[MAXL], ny[MAXL];
    if (n_threads <= 0) n_threads = n_cores();
    int L = or_level_table(W, H, min_face, scale_step, 27, 31, MAXL, sigma, lw, lh);
    if (L < 0) return -1;
    long row_first[MAXL + 1];
    long rows = 0, windows_per_frame = 0;
    for (int l = 0; l < L; ++l) {
        or_window_grid(lw[l], lh[l], &nx[l], &ny[l]);
        row_first[l] = rows;
        rows += ny[l];
        windows_per_frame += (long)nx[l] * ny[l];
    }
    row_first[L] = rows;

    uint8_t* lev[MAXL];
    double* map[MAXL];
    for (int l = 0; l < L; ++l) {
        lev[l] = (uint8_t*)malloc((size_t)lw[l] * lh[l]);
        map[l] = (double*)malloc(sizeof(double) * (size_t)nx[l] * ny[l]);
    }
    long cap_c = 1024, nc = 0;
    or_cand* cands = (or_cand*)malloc(sizeof(or_cand) * cap_c);
    long cap_b = 1024, nb = 0;
    or_box* boxes = (or_box*)malloc(sizeof(or_box) * cap_b);
    or_stats st = {0, 0, 0, 0, 0};

    for (int f = 0; f < n; ++f) {
        const uint8_t* frame = frames + (long)f * H * pitch;
        for (int l = 0; l < L; ++l) or_resample(frame, W, H, pitch, sigma[l], lw[l], lh[l], lev[l]);
        s1_ctx S = {&nets[0], lev, lw, lh, nx, ny, row_first, L, map, dense};
        par_for(dense ? L : rows, n_threads, s1_task, &S);
        /* survivors: (float) score > T1, in (level, i, j) order */
        long first = nc;
        for (int l = 0; l < L; ++l)
            for (int i = 0; i < ny[l]; ++i)
                for (int j = 0; j < nx[l]; ++j) {
                    double s1 = map[l][(long)i * nx[l] + j];
                    if (!((float)s1 > p->T1)) continue;
                    if (nc == cap_c) { cap_c *= 2; cands = (or_cand*)realloc(cands, sizeof(or_cand) * cap_c); }
                    or_cand* c = &cands[nc++];
                    memset(c, 0, sizeof(*c));
                    c->frame = f; c->level = l; c->ix = j; c->iy = i; c->s1 = s1;
                }
        sel_ctx C = {nets, frame, W, H, pitch, sigma, p, cands + first};
        par_for(nc - first, n_threads, sel_task, &C);
        /* raw boxes of accepted regions -> grouping */
        long nraw = 0;
        or_box* raw = (or_box*)malloc(sizeof(or_box) * (size_t)(nc - first + 1));
        for (long k = first; k < nc; ++k) {
            or_cand* c = &cands[k];
            st.stage1++;
            if (c->K2 > 0) st.stage2++;
            if (!c->delta) continue;
            st.stage3++;
            or_box b = {f, c->bx, c->by, c->bw, c->bh, c->score, 1};
            raw[nraw++] = b;
        }
        or_box* grouped = (or_box*)malloc(sizeof(or_box) * (size_t)(nraw + 1));
        int ng = or_group(raw, (int)nraw, p->nms_min_cluster, grouped);
        if (nb + ng > cap_b) {
            while (nb + ng > cap_b) cap_b *= 2;
            boxes = (or_box*)realloc(boxes, sizeof(or_box) * cap_b);
        }
        memcpy(boxes + nb, grouped, sizeof(or_box) * (size_t)ng);
        nb += ng;
        st.nms += ng;
        st.windows += windows_per_frame;
        free(raw); free(grouped);
    }
    for (int l = 0; l < L; ++l) { free(lev[l]); free(map[l]); }
    if (stats) *stats = st;
    if (cands_out) { *cands_out = cands; } else free(cands);
    if (n_cands_out) *n_cands_out = nc;
    if (boxes_out) { *boxes_out = boxes; } else free(boxes);
    if (n_boxes_out) *n_boxes_out = nb;
    return 0;
}

void or_free(void* p) { free(p); }
