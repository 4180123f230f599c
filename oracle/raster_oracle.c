/*
 * CPU ORACLE — test infrastructure only.
 *
 * Plain-C float64 restatement of the reference rasterizer inner loops
 * (splinesplat `_kernels.py`).  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library; the
 * product path (paper_2503_14171_b200/) never links or calls it.
 *
 * Parity pin: tests/test_oracle_golden.py compares this code (through
 * oracle/oracle.py) against golden vectors produced by the reference itself
 * (tests/golden/make_golden.py).  Build: oracle/Makefile
 * (gcc -O2 -ffp-contract=off, so every multiply/add rounds separately like the
 * numba-compiled reference; exp() is glibc's, as numba's np.exp lowers to it).
 *
 * Semantics followed:
 *   forward  : _kernels.py:32-129  (per-pixel front-to-back blend, cull
 *              1/255, clamp 0.999, early termination 1 - A < 1e-4)
 *   backward : _kernels.py:132-365 (replay culls up to count, back-to-front
 *              sweep with algebraic A-state inversion, per-splat adjoints)
 *   tiling   : raster_forward.py:126-149 / raster_backward.py:95-124
 *              (16x16 tiles, per-tile candidate lists in rank order, fixed
 *              tile-order reduction of per-tile partial gradients)
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORACLE_TILE 16

static const double kClamp = 0.999;        /* core.py:23 ALPHA_CLAMP */
static const double kCull = 1.0 / 255.0;   /* core.py:24 ALPHA_CULL */
static const double kTerm = 1e-4;          /* core.py:25 EARLY_TERMINATION */

/* _kernels.py:29 LOG_CULL = log(ALPHA_CULL) — passed in by the caller so the
 * bit pattern is numpy's, not a recomputation. */
typedef struct {
    const double *means;   /* (N,2) render-resolution, rank order */
    const double *conics;  /* (N,3) a,b,c */
    const double *sigmas;  /* (N,)  */
    const double *colors;  /* (N,3) */
    const int64_t *bboxes; /* (N,4) x0,x1,y0,y1 half-open */
    const double *bg;      /* (3,)  */
    double log_cull;
} Pack;

/* One footprint evaluation: returns 0 when culled, else fills alpha and its
 * spatial derivatives (zero when clamped) — _kernels.py:61-87. */
static int footprint(const Pack *p, int64_t g, int px, int py, double cx, double cy,
                     double *al, double *ax, double *ay, double *axy, int *clamped)
{
    const int64_t *bb = p->bboxes + 4 * g;
    if (px < bb[0] || px >= bb[1]) return 0;
    if (py < bb[2] || py >= bb[3]) return 0;
    double dx = cx - p->means[2 * g];
    double dy = cy - p->means[2 * g + 1];
    double ca = p->conics[3 * g], cb = p->conics[3 * g + 1], cc = p->conics[3 * g + 2];
    double expo = -(ca * dx * dx + 2.0 * cb * dx * dy + cc * dy * dy);
    if (expo < p->log_cull) return 0;
    double a_raw = p->sigmas[g] * exp(expo);
    if (a_raw < kCull) return 0;
    if (a_raw > kClamp) {
        *al = kClamp; *ax = 0.0; *ay = 0.0; *axy = 0.0; *clamped = 1;
    } else {
        double gx = -(2.0 * ca * dx + 2.0 * cb * dy);
        double gy = -(2.0 * cb * dx + 2.0 * cc * dy);
        *al = a_raw;
        *ax = a_raw * gx;
        *ay = a_raw * gy;
        *axy = a_raw * (gx * gy - 2.0 * cb);
        *clamped = 0;
    }
    return 1;
}

/* Blend one pixel over a rank-ordered candidate list (_kernels.py:40-124). */
static void forward_pixel(const Pack *p, const int64_t *cand, int64_t ncand, int px, int py,
                          int W, double *color, double *ddx, double *ddy, double *ddxy,
                          double *alpha, double *adx, double *ady, double *adxy, int32_t *count)
{
    double cx = px + 0.5, cy = py + 0.5;
    double b[3] = {0, 0, 0}, bx[3] = {0, 0, 0}, by[3] = {0, 0, 0}, bxy[3] = {0, 0, 0};
    double acc = 0.0, accx = 0.0, accy = 0.0, accxy = 0.0;
    int32_t n = 0;
    for (int64_t ci = 0; ci < ncand; ++ci) {
        int64_t g = cand[ci];
        double al, ax, ay, axy;
        int clamped;
        if (!footprint(p, g, px, py, cx, cy, &al, &ax, &ay, &axy, &clamped)) continue;
        double t = 1.0 - acc;
        const double *col = p->colors + 3 * g;
        double term_xy = t * axy - accy * ax - accxy * al - accx * ay;
        for (int c = 0; c < 3; ++c) bx[c] += col[c] * (t * ax - accx * al);
        for (int c = 0; c < 3; ++c) by[c] += col[c] * (t * ay - accy * al);
        for (int c = 0; c < 3; ++c) bxy[c] += col[c] * term_xy;
        for (int c = 0; c < 3; ++c) b[c] += col[c] * (t * al);
        double nx = accx * (1.0 - al) + t * ax;
        double ny = accy * (1.0 - al) + t * ay;
        double nxy = accxy * (1.0 - al) + t * axy - accx * ay - accy * ax;
        acc = acc + al * t;
        accx = nx; accy = ny; accxy = nxy;
        n += 1;
        if (1.0 - acc < kTerm) break;
    }
    int64_t o = (int64_t)py * W + px;
    double tf = 1.0 - acc;
    for (int c = 0; c < 3; ++c) {
        color[3 * o + c] = b[c] + tf * p->bg[c];
        ddx[3 * o + c] = bx[c] - accx * p->bg[c];
        ddy[3 * o + c] = by[c] - accy * p->bg[c];
        ddxy[3 * o + c] = bxy[c] - accxy * p->bg[c];
    }
    alpha[o] = acc; adx[o] = accx; ady[o] = accy; adxy[o] = accxy;
    count[o] = n;
}

/* Render every 16x16 tile from CSR candidate lists (raster_forward.py:152-187). */
void oracle_forward(int W, int H, const int64_t *tile_off, const int64_t *tile_cand,
                    const double *means, const double *conics, const double *sigmas,
                    const double *colors, const int64_t *bboxes, const double *bg,
                    double log_cull,
                    double *color, double *ddx, double *ddy, double *ddxy,
                    double *alpha, double *adx, double *ady, double *adxy, int32_t *count,
                    int nthreads)
{
    Pack p = {means, conics, sigmas, colors, bboxes, bg, log_cull};
    int ntx = (W + ORACLE_TILE - 1) / ORACLE_TILE;
    int nty = (H + ORACLE_TILE - 1) / ORACLE_TILE;
    int ntiles = ntx * nty;
    (void)nthreads;
#pragma omp parallel for schedule(dynamic, 1) num_threads(nthreads > 0 ? nthreads : 1)
    for (int t = 0; t < ntiles; ++t) {
        int tx0 = (t % ntx) * ORACLE_TILE, ty0 = (t / ntx) * ORACLE_TILE;
        int tx1 = tx0 + ORACLE_TILE < W ? tx0 + ORACLE_TILE : W;
        int ty1 = ty0 + ORACLE_TILE < H ? ty0 + ORACLE_TILE : H;
        const int64_t *cand = tile_cand + tile_off[t];
        int64_t ncand = tile_off[t + 1] - tile_off[t];
        for (int py = ty0; py < ty1; ++py)
            for (int px = tx0; px < tx1; ++px)
                forward_pixel(&p, cand, ncand, px, py, W, color, ddx, ddy, ddxy,
                              alpha, adx, ady, adxy, count);
    }
}

/* Untiled path: one region, one candidate list (raster_forward.py:172-175). */
void oracle_forward_region(int W, int px0, int px1, int py0, int py1,
                           const int64_t *cand, int64_t ncand,
                           const double *means, const double *conics, const double *sigmas,
                           const double *colors, const int64_t *bboxes, const double *bg,
                           double log_cull,
                           double *color, double *ddx, double *ddy, double *ddxy,
                           double *alpha, double *adx, double *ady, double *adxy, int32_t *count)
{
    Pack p = {means, conics, sigmas, colors, bboxes, bg, log_cull};
    for (int py = py0; py < py1; ++py)
        for (int px = px0; px < px1; ++px)
            forward_pixel(&p, cand, ncand, px, py, W, color, ddx, ddy, ddxy,
                          alpha, adx, ady, adxy, count);
}

/* Per-contributor record of the backward replay (_kernels.py:144-149). */
typedef struct { int64_t pos; double al, ax, ay, axy; int clamped; } Contrib;

/* Backward for one tile; partial gradients go to part[pos*9 + k] where pos is
 * the candidate's position in the tile list, k = d_color(3), d_sigma(1),
 * d_mean(2), d_conic(3).  Mirrors _kernels.py:150-365. */
static void backward_tile(const Pack *p, const int64_t *cand, int64_t ncand,
                          int tx0, int tx1, int ty0, int ty1, int W,
                          const double *alpha_img, const double *adx_img, const double *ady_img,
                          const double *adxy_img, const int32_t *count_img,
                          const double *w, const double *wx, const double *wy, const double *wxy,
                          double *part, Contrib *stk)
{
    for (int py = ty0; py < ty1; ++py) {
        double cy = py + 0.5;
        for (int px = tx0; px < tx1; ++px) {
            double cx = px + 0.5;
            int64_t o = (int64_t)py * W + px;
            int32_t m = count_img[o];
            if (m == 0) continue;
            const double *W0 = w + 3 * o, *WX = wx + 3 * o, *WY = wy + 3 * o, *WXY = wxy + 3 * o;
            int allzero = 1;
            for (int c = 0; c < 3; ++c)
                if (W0[c] != 0.0 || WX[c] != 0.0 || WY[c] != 0.0 || WXY[c] != 0.0) allzero = 0;
            if (allzero) continue;
            int64_t n = 0;
            for (int64_t ci = 0; ci < ncand && n < m; ++ci) {
                Contrib *s = stk + n;
                if (!footprint(p, cand[ci], px, py, cx, cy, &s->al, &s->ax, &s->ay, &s->axy,
                               &s->clamped))
                    continue;
                s->pos = ci;
                ++n;
            }
            double av = alpha_img[o], avx = adx_img[o], avy = ady_img[o], avxy = adxy_img[o];
            double bh[3], bhx[3] = {0, 0, 0}, bhy[3] = {0, 0, 0}, bhxy[3] = {0, 0, 0};
            for (int c = 0; c < 3; ++c) bh[c] = p->bg[c];
            for (int64_t k = n - 1; k >= 0; --k) {
                const Contrib *s = stk + k;
                int64_t g = cand[s->pos];
                double *pg = part + 9 * s->pos;
                const double *col = p->colors + 3 * g;
                double al = s->al, ax = s->ax, ay = s->ay, axy = s->axy;
                double om = 1.0 - al;
                double a_prev = (av - al) / om;
                double t = 1.0 - a_prev;
                double ax_prev = (avx - t * ax) / om;
                double ay_prev = (avy - t * ay) / om;
                double axy_prev = (avxy - t * axy + ax_prev * ay + ay_prev * ax) / om;
                double abar = 0.0, abar_x = 0.0, abar_y = 0.0, abar_xy = 0.0;
                for (int c = 0; c < 3; ++c) {
                    double diff = col[c] - bh[c];
                    double u0 = t * diff;
                    double u1 = -ax_prev * diff - t * bhx[c];
                    double u2 = -ay_prev * diff - t * bhy[c];
                    double u3 = -axy_prev * diff + ax_prev * bhy[c] + ay_prev * bhx[c] - t * bhxy[c];
                    pg[c] += (W0[c] * (t * al)
                              + WX[c] * (t * ax - ax_prev * al)
                              + WY[c] * (t * ay - ay_prev * al)
                              + WXY[c] * (t * axy - axy_prev * al - ay_prev * ax - ax_prev * ay));
                    abar += W0[c] * u0 + WX[c] * u1 + WY[c] * u2 + WXY[c] * u3;
                    abar_x += WX[c] * u0 + WXY[c] * u2;
                    abar_y += WY[c] * u0 + WXY[c] * u1;
                    abar_xy += WXY[c] * u0;
                }
                if (!s->clamped) {
                    double dx = cx - p->means[2 * g];
                    double dy = cy - p->means[2 * g + 1];
                    double ca = p->conics[3 * g], cb = p->conics[3 * g + 1], cc = p->conics[3 * g + 2];
                    double gx = -(2.0 * ca * dx + 2.0 * cb * dy);
                    double gy = -(2.0 * cb * dx + 2.0 * cc * dy);
                    double gxy = -2.0 * cb;
                    double hxy = gx * gy + gxy;
                    pg[3] += (abar * al + abar_x * ax + abar_y * ay + abar_xy * axy) / p->sigmas[g];
                    pg[4] += al * (abar * (-gx) + abar_x * (-gx * gx + 2.0 * ca)
                                   + abar_y * (-gx * gy + 2.0 * cb)
                                   + abar_xy * (-gx * hxy + 2.0 * ca * gy + 2.0 * cb * gx));
                    pg[5] += al * (abar * (-gy) + abar_x * (-gy * gx + 2.0 * cb)
                                   + abar_y * (-gy * gy + 2.0 * cc)
                                   + abar_xy * (-gy * hxy + 2.0 * cb * gy + 2.0 * cc * gx));
                    pg[6] += al * (abar * (-dx * dx) + abar_x * (-dx * dx * gx - 2.0 * dx)
                                   + abar_y * (-dx * dx * gy)
                                   + abar_xy * (-dx * dx * hxy - 2.0 * dx * gy));
                    pg[7] += al * (abar * (-2.0 * dx * dy) + abar_x * (-2.0 * dx * dy * gx - 2.0 * dy)
                                   + abar_y * (-2.0 * dx * dy * gy - 2.0 * dx)
                                   + abar_xy * (-2.0 * dx * dy * hxy - 2.0 * dy * gy - 2.0 * gx * dx
                                                - 2.0));
                    pg[8] += al * (abar * (-dy * dy) + abar_x * (-dy * dy * gx)
                                   + abar_y * (-dy * dy * gy - 2.0 * dy)
                                   + abar_xy * (-dy * dy * hxy - 2.0 * dy * gx));
                }
                double nbx[3], nby[3], nbxy[3];
                for (int c = 0; c < 3; ++c) {
                    nbx[c] = om * bhx[c] + ax * (col[c] - bh[c]);
                    nby[c] = om * bhy[c] + ay * (col[c] - bh[c]);
                    nbxy[c] = (om * bhxy[c] + axy * (col[c] - bh[c]) - ay * bhx[c] - ax * bhy[c]);
                }
                for (int c = 0; c < 3; ++c) {
                    bh[c] = om * bh[c] + al * col[c];
                    bhx[c] = nbx[c]; bhy[c] = nby[c]; bhxy[c] = nbxy[c];
                }
                av = a_prev; avx = ax_prev; avy = ay_prev; avxy = axy_prev;
            }
        }
    }
}

/* Full backward over all tiles; render-space gradients in rank order
 * (raster_backward.py:87-124). out9 is (N,9): d_color(3) d_sigma d_mean(2) d_conic(3). */
void oracle_backward(int W, int H, const int64_t *tile_off, const int64_t *tile_cand,
                     const double *means, const double *conics, const double *sigmas,
                     const double *colors, const int64_t *bboxes, const double *bg,
                     double log_cull,
                     const double *alpha_img, const double *adx_img, const double *ady_img,
                     const double *adxy_img, const int32_t *count_img,
                     const double *w, const double *wx, const double *wy, const double *wxy,
                     double *out9, int64_t n_splats, int nthreads)
{
    Pack p = {means, conics, sigmas, colors, bboxes, bg, log_cull};
    int ntx = (W + ORACLE_TILE - 1) / ORACLE_TILE;
    int nty = (H + ORACLE_TILE - 1) / ORACLE_TILE;
    int ntiles = ntx * nty;
    int64_t total = tile_off[ntiles];
    double *part = (double *)calloc((size_t)(total > 0 ? total : 1) * 9, sizeof(double));
    (void)nthreads;
#pragma omp parallel num_threads(nthreads > 0 ? nthreads : 1)
    {
        int64_t maxc = 1;
        for (int t = 0; t < ntiles; ++t)
            if (tile_off[t + 1] - tile_off[t] > maxc) maxc = tile_off[t + 1] - tile_off[t];
        Contrib *stk = (Contrib *)malloc((size_t)maxc * sizeof(Contrib));
#pragma omp for schedule(dynamic, 1)
        for (int t = 0; t < ntiles; ++t) {
            int tx0 = (t % ntx) * ORACLE_TILE, ty0 = (t / ntx) * ORACLE_TILE;
            int tx1 = tx0 + ORACLE_TILE < W ? tx0 + ORACLE_TILE : W;
            int ty1 = ty0 + ORACLE_TILE < H ? ty0 + ORACLE_TILE : H;
            backward_tile(&p, tile_cand + tile_off[t], tile_off[t + 1] - tile_off[t],
                          tx0, tx1, ty0, ty1, W, alpha_img, adx_img, ady_img, adxy_img,
                          count_img, w, wx, wy, wxy, part + 9 * tile_off[t], stk);
        }
        free(stk);
    }
    memset(out9, 0, (size_t)n_splats * 9 * sizeof(double));
    /* fixed tile order, then list order — same summation order as adding the
     * reference's per-tile N-sized buffers one after another */
    for (int64_t j = 0; j < total; ++j) {
        int64_t g = tile_cand[j];
        for (int k = 0; k < 9; ++k) out9[9 * g + k] += part[9 * j + k];
    }
    free(part);
}
