/*
 * oracle_ops.c -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, fp64 direct (nested-loop) operators for the LR-CNN oracle.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load this library.  It shares no code, header or constant with the CUDA
 * path in paper_2401_11471_b200/.
 *
 * Layout: NCHW tensors, OIHW weights, all double.  Padding is given per side
 * (top, bottom, left, right) so that the row-centric CPU executor can apply
 * the paper's "semi-closed padding" (Sec. III-B "Conclusion and
 * Solution"): an interior band cut gets zero padding rows, only the original
 * outer edges carry p.
 *
 * Accumulation order inside every MUL-SUM is channel, then kernel row, then
 * kernel column, then the bias.
 *
 * Ops:
 *   conv2d_fwd        Eq. (1) z^l = Conv(z^{l-1}, theta_l)
 *   conv2d_bwd_data   delta^{l-1} = Get_error(delta^l, theta^l)   (Alg. 1 l.17)
 *   conv2d_bwd_weight g^l = Gradient(delta^l, z^{l-1}), Eq. (2)
 *   maxpool_fwd/bwd   "replacing some values with a single max"
 *                     ties -> lowest flat index; padded cells never win.
 */
#include <stddef.h>
#include <math.h>

#define IDX4(a, b, c, d, B1, C1, D1) ((((size_t)(a) * (B1) + (b)) * (C1) + (c)) * (D1) + (d))

/* Output extent, standard law floor((H + pads - k)/s) + 1. */
int oracle_out_dim(int h, int pad_a, int pad_b, int k, int s)
{
    int span = h + pad_a + pad_b - k;
    if (span < 0 || s < 1) return -1;
    return span / s + 1;
}

/* y[b,co,oy,ox] = sum_ci sum_ky sum_kx w[co,ci,ky,kx] * x[b,ci,oy*s-pt+ky,ox*s-pl+kx] + bias[co]
 * (out-of-range input cells are the zero padding). */
void oracle_conv2d_fwd(int B, int Ci, int H, int W, const double *x,
                       int Co, int k, int s, int pt, int pb, int pl, int pr,
                       const double *w, const double *bias, double *y)
{
    int Ho = oracle_out_dim(H, pt, pb, k, s), Wo = oracle_out_dim(W, pl, pr, k, s);
    #pragma omp parallel for collapse(2) schedule(static)
    for (int b = 0; b < B; ++b)
        for (int co = 0; co < Co; ++co) {
            double *yo = y + IDX4(b, co, 0, 0, Co, Ho, Wo);
            for (size_t i = 0; i < (size_t)Ho * Wo; ++i) yo[i] = 0.0;
            for (int ci = 0; ci < Ci; ++ci)
                for (int ky = 0; ky < k; ++ky)
                    for (int kx = 0; kx < k; ++kx) {
                        double wv = w[IDX4(co, ci, ky, kx, Ci, k, k)];
                        const double *xi = x + IDX4(b, ci, 0, 0, Ci, H, W);
                        for (int oy = 0; oy < Ho; ++oy) {
                            int iy = oy * s - pt + ky;
                            if (iy < 0 || iy >= H) continue;
                            for (int ox = 0; ox < Wo; ++ox) {
                                int ix = ox * s - pl + kx;
                                if (ix < 0 || ix >= W) continue;
                                yo[(size_t)oy * Wo + ox] += wv * xi[(size_t)iy * W + ix];
                            }
                        }
                    }
            if (bias)
                for (size_t i = 0; i < (size_t)Ho * Wo; ++i) yo[i] += bias[co];
        }
}

/* dx = adjoint of conv2d_fwd applied to dy:  dx[b,ci,iy,ix] = sum over (co,ky,kx,oy,ox)
 * with iy = oy*s-pt+ky, ix = ox*s-pl+kx of w[co,ci,ky,kx]*dy[b,co,oy,ox]. */
void oracle_conv2d_bwd_data(int B, int Ci, int H, int W,
                            int Co, int k, int s, int pt, int pb, int pl, int pr,
                            const double *w, const double *dy, double *dx)
{
    int Ho = oracle_out_dim(H, pt, pb, k, s), Wo = oracle_out_dim(W, pl, pr, k, s);
    #pragma omp parallel for collapse(2) schedule(static)
    for (int b = 0; b < B; ++b)
        for (int ci = 0; ci < Ci; ++ci) {
            double *xo = dx + IDX4(b, ci, 0, 0, Ci, H, W);
            for (size_t i = 0; i < (size_t)H * W; ++i) xo[i] = 0.0;
            for (int co = 0; co < Co; ++co)
                for (int ky = 0; ky < k; ++ky)
                    for (int kx = 0; kx < k; ++kx) {
                        double wv = w[IDX4(co, ci, ky, kx, Ci, k, k)];
                        const double *d = dy + IDX4(b, co, 0, 0, Co, Ho, Wo);
                        for (int oy = 0; oy < Ho; ++oy) {
                            int iy = oy * s - pt + ky;
                            if (iy < 0 || iy >= H) continue;
                            for (int ox = 0; ox < Wo; ++ox) {
                                int ix = ox * s - pl + kx;
                                if (ix < 0 || ix >= W) continue;
                                xo[(size_t)iy * W + ix] += wv * d[(size_t)oy * Wo + ox];
                            }
                        }
                    }
        }
}

/* dw[co,ci,ky,kx] = sum_{b,oy,ox} dy[b,co,oy,ox] * x[b,ci,oy*s-pt+ky,ox*s-pl+kx];
 * db[co] = sum_{b,oy,ox} dy[b,co,oy,ox]  (db may be NULL).  Overwrites dw/db. */
void oracle_conv2d_bwd_weight(int B, int Ci, int H, int W, const double *x,
                              int Co, int k, int s, int pt, int pb, int pl, int pr,
                              const double *dy, double *dw, double *db)
{
    int Ho = oracle_out_dim(H, pt, pb, k, s), Wo = oracle_out_dim(W, pl, pr, k, s);
    #pragma omp parallel for collapse(2) schedule(static)
    for (int co = 0; co < Co; ++co)
        for (int ci = 0; ci < Ci; ++ci)
            for (int ky = 0; ky < k; ++ky)
                for (int kx = 0; kx < k; ++kx) {
                    double acc = 0.0;
                    for (int b = 0; b < B; ++b) {
                        const double *d = dy + IDX4(b, co, 0, 0, Co, Ho, Wo);
                        const double *xi = x + IDX4(b, ci, 0, 0, Ci, H, W);
                        for (int oy = 0; oy < Ho; ++oy) {
                            int iy = oy * s - pt + ky;
                            if (iy < 0 || iy >= H) continue;
                            for (int ox = 0; ox < Wo; ++ox) {
                                int ix = ox * s - pl + kx;
                                if (ix < 0 || ix >= W) continue;
                                acc += d[(size_t)oy * Wo + ox] * xi[(size_t)iy * W + ix];
                            }
                        }
                    }
                    dw[IDX4(co, ci, ky, kx, Ci, k, k)] = acc;
                }
    if (db) {
        for (int co = 0; co < Co; ++co) {
            double acc = 0.0;
            for (int b = 0; b < B; ++b) {
                const double *d = dy + IDX4(b, co, 0, 0, Co, Ho, Wo);
                for (size_t i = 0; i < (size_t)Ho * Wo; ++i) acc += d[i];
            }
            db[co] = acc;
        }
    }
}

/* Max pooling; padded cells are excluded from the window (they never win).
 * argmax holds the flat (iy*W+ix) index inside the (b,c) plane, ties -> lowest index
 * (first in raster order, strict '>' comparison).  A window with no valid cell
 * yields 0 and argmax -1 (cannot happen for the configurations used). */
void oracle_maxpool_fwd(int B, int C, int H, int W, const double *x,
                        int k, int s, int pt, int pb, int pl, int pr,
                        double *y, long *argmax)
{
    int Ho = oracle_out_dim(H, pt, pb, k, s), Wo = oracle_out_dim(W, pl, pr, k, s);
    #pragma omp parallel for collapse(2) schedule(static)
    for (int b = 0; b < B; ++b)
        for (int c = 0; c < C; ++c) {
            const double *xi = x + IDX4(b, c, 0, 0, C, H, W);
            for (int oy = 0; oy < Ho; ++oy)
                for (int ox = 0; ox < Wo; ++ox) {
                    double best = -INFINITY;
                    long bi = -1;
                    for (int ky = 0; ky < k; ++ky) {
                        int iy = oy * s - pt + ky;
                        if (iy < 0 || iy >= H) continue;
                        for (int kx = 0; kx < k; ++kx) {
                            int ix = ox * s - pl + kx;
                            if (ix < 0 || ix >= W) continue;
                            double v = xi[(size_t)iy * W + ix];
                            if (bi < 0 || v > best) { best = v; bi = (long)iy * W + ix; }
                        }
                    }
                    size_t o = IDX4(b, c, oy, ox, C, Ho, Wo);
                    y[o] = bi < 0 ? 0.0 : best;
                    argmax[o] = bi;
                }
        }
}

/* dx[b,c,argmax] += dy[b,c,oy,ox]  (dx overwritten first). */
void oracle_maxpool_bwd(int B, int C, int H, int W, int Ho, int Wo,
                        const long *argmax, const double *dy, double *dx)
{
    #pragma omp parallel for collapse(2) schedule(static)
    for (int b = 0; b < B; ++b)
        for (int c = 0; c < C; ++c) {
            double *xo = dx + IDX4(b, c, 0, 0, C, H, W);
            for (size_t i = 0; i < (size_t)H * W; ++i) xo[i] = 0.0;
            for (int oy = 0; oy < Ho; ++oy)
                for (int ox = 0; ox < Wo; ++ox) {
                    size_t o = IDX4(b, c, oy, ox, C, Ho, Wo);
                    if (argmax[o] >= 0) xo[argmax[o]] += dy[o];
                }
        }
}
