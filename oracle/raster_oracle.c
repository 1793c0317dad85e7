/* Oracle raster loops — TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).
 *
 * Plain-C restatement of the three numba kernels of the reference tiled
 * rasterizer, splatforge/_raster_kernels.py:
 *   oracle_project  <- project_kernel  (_raster_kernels.py:20-105)
 *   oracle_bin      <- bin_tiles       (_raster_kernels.py:108-143)
 *   oracle_forward  <- forward_kernel  (_raster_kernels.py:146-201)
 * Built with -ffp-contract=off: numba evaluates these IEEE float64 expressions
 * left to right without FMA contraction, and so does this file. The tile
 * window [ty_lo, ty_hi) of oracle_bin/oracle_forward restricts the work to a
 * band of tile rows (whole image = [0, nty)); it exists only so bench.py can
 * time a bounded sample of a frame whose full CSR would not fit in memory.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ALPHA_CUTOFF (1.0 / 255.0)
#define TRANS_CUTOFF (1.0 / 255.0)

static inline double dmax(double a, double b) { return a > b ? a : b; }
static inline int64_t imax(int64_t a, int64_t b) { return a > b ? a : b; }
static inline int64_t imin(int64_t a, int64_t b) { return a < b ? a : b; }

void oracle_project(const double *centers, const double *quats, const double *scales, int64_t n,
                    const double *rot, const double *tr, double fx, double fy, double cx,
                    double cy, int64_t width, int64_t height, double z_near, double dilation,
                    double *sx, double *sy, double *depth, double *cov_a, double *cov_b,
                    double *cov_c, double *radius, uint8_t *keep) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) {
        const double *p = centers + 3 * i;
        sx[i] = sy[i] = depth[i] = cov_a[i] = cov_b[i] = cov_c[i] = radius[i] = 0.0;
        keep[i] = 0;
        double px = rot[0] * p[0] + rot[1] * p[1] + rot[2] * p[2] + tr[0];
        double py = rot[3] * p[0] + rot[4] * p[1] + rot[5] * p[2] + tr[1];
        double pz = rot[6] * p[0] + rot[7] * p[1] + rot[8] * p[2] + tr[2];
        if (pz <= z_near) continue;
        const double *q = quats + 4 * i;
        double w = q[0], x = q[1], y = q[2], z = q[3];
        double qn = sqrt(w * w + x * x + y * y + z * z);
        w /= qn; x /= qn; y /= qn; z /= qn;
        double r[9] = {
            1.0 - 2.0 * (y * y + z * z), 2.0 * (x * y - w * z), 2.0 * (x * z + w * y),
            2.0 * (x * y + w * z), 1.0 - 2.0 * (x * x + z * z), 2.0 * (y * z - w * x),
            2.0 * (x * z - w * y), 2.0 * (y * z + w * x), 1.0 - 2.0 * (x * x + y * y)};
        /* U = R_splat T^T (row i of R against row j of the camera rotation) */
        double u[9];
        for (int a = 0; a < 3; ++a)
            for (int b = 0; b < 3; ++b)
                u[3 * a + b] = r[3 * a] * rot[3 * b] + r[3 * a + 1] * rot[3 * b + 1] +
                               r[3 * a + 2] * rot[3 * b + 2];
        const double *sc = scales + 3 * i;
        double d0 = sc[0] * sc[0], d1 = sc[1] * sc[1], d2 = sc[2] * sc[2];
#define SIG(j, k) (d0 * u[j] * u[k] + d1 * u[3 + j] * u[3 + k] + d2 * u[6 + j] * u[6 + k])
        double s00 = SIG(0, 0), s01 = SIG(0, 1), s02 = SIG(0, 2);
        double s11 = SIG(1, 1), s12 = SIG(1, 2), s22 = SIG(2, 2);
#undef SIG
        double jx = fx / pz, jy = fy / pz;
        double jxz = -fx * px / (pz * pz), jyz = -fy * py / (pz * pz);
        double a = jx * jx * s00 + 2.0 * jx * jxz * s02 + jxz * jxz * s22 + dilation;
        double b = jx * jy * s01 + jx * jyz * s02 + jxz * jy * s12 + jxz * jyz * s22;
        double c = jy * jy * s11 + 2.0 * jy * jyz * s12 + jyz * jyz * s22 + dilation;
        double mid = 0.5 * (a + c);
        double gap = sqrt(dmax(0.25 * (a - c) * (a - c) + b * b, 0.0));
        double rad = 3.0 * sqrt(dmax(mid + gap, 0.0));
        double csx = jx * px + cx, csy = jy * py + cy;
        if (csx + rad < 0.0 || csx - rad > (double)width - 1.0) continue;
        if (csy + rad < 0.0 || csy - rad > (double)height - 1.0) continue;
        sx[i] = csx; sy[i] = csy; depth[i] = pz;
        cov_a[i] = a; cov_b[i] = b; cov_c[i] = c; radius[i] = rad; keep[i] = 1;
    }
}

static void tile_range(double sx, double sy, double r, double ft, int64_t ntx, int64_t nty,
                       int64_t *x0, int64_t *x1, int64_t *y0, int64_t *y1) {
    *x0 = imax((int64_t)floor((sx - r) / ft), 0);
    *x1 = imin((int64_t)floor((sx + r) / ft), ntx - 1);
    *y0 = imax((int64_t)floor((sy - r) / ft), 0);
    *y1 = imin((int64_t)floor((sy + r) / ft), nty - 1);
}

/* Pass 1: counts per tile (offsets must hold ntx*nty+1 entries); returns E. */
int64_t oracle_bin_count(const double *sx, const double *sy, const double *radius, int64_t n,
                         int64_t tile, int64_t ntx, int64_t nty, int64_t ty_lo, int64_t ty_hi,
                         int64_t tx_lo, int64_t tx_hi, int64_t *offsets) {
    memset(offsets, 0, sizeof(int64_t) * (ntx * nty + 1));
    double ft = (double)tile;
    for (int64_t i = 0; i < n; ++i) {
        int64_t x0, x1, y0, y1;
        tile_range(sx[i], sy[i], radius[i], ft, ntx, nty, &x0, &x1, &y0, &y1);
        y0 = imax(y0, ty_lo);
        y1 = imin(y1, ty_hi - 1);
        x0 = imax(x0, tx_lo);   /* crop window (tests): tiles outside stay empty */
        x1 = imin(x1, tx_hi - 1);
        for (int64_t ty = y0; ty <= y1; ++ty)
            for (int64_t tx = x0; tx <= x1; ++tx) offsets[ty * ntx + tx + 1] += 1;
    }
    for (int64_t t = 0; t < ntx * nty; ++t) offsets[t + 1] += offsets[t];
    return offsets[ntx * nty];
}

/* Pass 2: scatter splat ranks in iteration (= depth) order. */
void oracle_bin_fill(const double *sx, const double *sy, const double *radius, int64_t n,
                     int64_t tile, int64_t ntx, int64_t nty, int64_t ty_lo, int64_t ty_hi,
                     int64_t tx_lo, int64_t tx_hi, const int64_t *offsets, int64_t *ids) {
    int64_t *cursor = (int64_t *)malloc(sizeof(int64_t) * (ntx * nty));
    memcpy(cursor, offsets, sizeof(int64_t) * (ntx * nty));
    double ft = (double)tile;
    for (int64_t i = 0; i < n; ++i) {
        int64_t x0, x1, y0, y1;
        tile_range(sx[i], sy[i], radius[i], ft, ntx, nty, &x0, &x1, &y0, &y1);
        y0 = imax(y0, ty_lo);
        y1 = imin(y1, ty_hi - 1);
        x0 = imax(x0, tx_lo);   /* crop window (tests): tiles outside stay empty */
        x1 = imin(x1, tx_hi - 1);
        for (int64_t ty = y0; ty <= y1; ++ty)
            for (int64_t tx = x0; tx <= x1; ++tx) ids[cursor[ty * ntx + tx]++] = i;
    }
    free(cursor);
}

void oracle_forward(int64_t width, int64_t height, int64_t tile, int64_t ntx, int64_t nty,
                    int64_t ty_lo, int64_t ty_hi, const int64_t *offsets, const int64_t *ids,
                    const double *sx, const double *sy, const double *radius,
                    const double *inv_a, const double *inv_b, const double *inv_c,
                    const double *opac, const double *attr, double alpha_max, int terminate,
                    double *out, double *trans) {
    int64_t t_lo = ty_lo * ntx, t_hi = ty_hi * ntx;
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t t = t_lo; t < t_hi; ++t) {
        int64_t tx = t % ntx, ty = t / ntx;
        int64_t x_end = imin((tx + 1) * tile, width), y_end = imin((ty + 1) * tile, height);
        for (int64_t e = offsets[t]; e < offsets[t + 1]; ++e) {
            int64_t s = ids[e];
            double rad = radius[s] + 1.0, rr = rad * rad;
            double mx = sx[s], my = sy[s];
            double ia = inv_a[s], ib = inv_b[s], ic = inv_c[s], op = opac[s];
            double a0 = attr[3 * s], a1 = attr[3 * s + 1], a2 = attr[3 * s + 2];
            int64_t px0 = imax(tx * tile, (int64_t)ceil(mx - rad));
            int64_t px1 = imin(x_end - 1, (int64_t)floor(mx + rad));
            int64_t py0 = imax(ty * tile, (int64_t)ceil(my - rad));
            int64_t py1 = imin(y_end - 1, (int64_t)floor(my + rad));
            for (int64_t py = py0; py <= py1; ++py) {
                double dy = (double)py - my;
                for (int64_t px = px0; px <= px1; ++px) {
                    int64_t pix = py * width + px;
                    double tr = trans[pix];
                    if (terminate && tr < TRANS_CUTOFF) continue;
                    double dx = (double)px - mx;
                    if (dx * dx + dy * dy > rr) continue;
                    double q = ia * dx * dx + 2.0 * ib * dx * dy + ic * dy * dy;
                    double alpha = op * exp(-0.5 * q);
                    if (alpha > alpha_max) alpha = alpha_max;
                    if (alpha < ALPHA_CUTOFF) continue;
                    double w = tr * alpha;
                    out[3 * pix] += w * a0;
                    out[3 * pix + 1] += w * a1;
                    out[3 * pix + 2] += w * a2;
                    trans[pix] = tr * (1.0 - alpha);
                }
            }
        }
    }
}

/* backward_kernel (_raster_kernels.py:204-310): per-pixel forward replay of
 * the tile list (no box/circle test, break after the blend that takes T below
 * the cutoff), then a reverse sweep reconstructing T_k and the suffix sums;
 * gradients accumulate into per-CSR-entry slots. mode 0 rgb (background
 * composited), 1 normal (upstream through the renormalisation), 2 depth. */
void oracle_backward(int64_t width, int64_t height, int64_t tile, int64_t ntx, int64_t nty,
                     const int64_t *offsets, const int64_t *ids, const double *sx,
                     const double *sy, const double *inv_a, const double *inv_b,
                     const double *inv_c, const double *opac, const double *attr,
                     double alpha_max, int terminate, int mode, const double *background,
                     const double *upstream, double *g_mu, double *g_q, double *g_opac,
                     double *g_attr) {
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t t = 0; t < ntx * nty; ++t) {
        int64_t tx = t % ntx, ty = t / ntx;
        int64_t x_end = imin((tx + 1) * tile, width), y_end = imin((ty + 1) * tile, height);
        int64_t start = offsets[t], end = offsets[t + 1];
        for (int64_t py = ty * tile; py < y_end; ++py)
            for (int64_t px = tx * tile; px < x_end; ++px) {
                double tr = 1.0, n0 = 0.0, n1 = 0.0, n2 = 0.0;
                int64_t e_last = start - 1;
                for (int64_t e = start; e < end; ++e) {
                    int64_t s = ids[e];
                    double dx = (double)px - sx[s], dy = (double)py - sy[s];
                    double q = inv_a[s] * dx * dx + 2.0 * inv_b[s] * dx * dy + inv_c[s] * dy * dy;
                    double alpha = opac[s] * exp(-0.5 * q);
                    if (alpha > alpha_max) alpha = alpha_max;
                    if (alpha < ALPHA_CUTOFF) continue;
                    double w = tr * alpha;
                    n0 += w * attr[3 * s];
                    n1 += w * attr[3 * s + 1];
                    n2 += w * attr[3 * s + 2];
                    tr *= 1.0 - alpha;
                    e_last = e;
                    if (terminate && tr < TRANS_CUTOFF) break;
                }
                double t_fin = tr;
                const double *up = upstream + 3 * (py * width + px);
                double u0 = up[0], u1 = up[1], u2 = up[2];
                if (mode == 1) {
                    double nn = sqrt(n0 * n0 + n1 * n1 + n2 * n2);
                    if (nn > 1e-12) {
                        double dot = (n0 * u0 + n1 * u1 + n2 * u2) / (nn * nn * nn);
                        u0 = u0 / nn - n0 * dot;
                        u1 = u1 / nn - n1 * dot;
                        u2 = u2 / nn - n2 * dot;
                    }
                }
                double d_tfin = 0.0;
                if (mode == 0) d_tfin = u0 * background[0] + u1 * background[1] + u2 * background[2];
                if (u0 == 0.0 && u1 == 0.0 && u2 == 0.0) continue;
                double s0 = 0.0, s1 = 0.0, s2 = 0.0, t_next = t_fin;
                for (int64_t e = e_last; e > start - 1; --e) {
                    int64_t s = ids[e];
                    double dx = (double)px - sx[s], dy = (double)py - sy[s];
                    double q = inv_a[s] * dx * dx + 2.0 * inv_b[s] * dx * dy + inv_c[s] * dy * dy;
                    double g = exp(-0.5 * q);
                    double raw = opac[s] * g;
                    int clamped = raw > alpha_max;
                    double alpha = clamped ? alpha_max : raw;
                    if (alpha < ALPHA_CUTOFF) continue;
                    double one_m = 1.0 - alpha;
                    double t_k = t_next / one_m;
                    double w = t_k * alpha;
                    const double *a = attr + 3 * s;
                    g_attr[3 * e] += u0 * w;
                    g_attr[3 * e + 1] += u1 * w;
                    g_attr[3 * e + 2] += u2 * w;
                    double d_alpha = (u0 * (t_k * a[0] - s0 / one_m) + u1 * (t_k * a[1] - s1 / one_m) +
                                      u2 * (t_k * a[2] - s2 / one_m) - d_tfin * t_fin / one_m);
                    if (!clamped) {
                        g_opac[e] += d_alpha * g;
                        double d_q = -0.5 * opac[s] * g * d_alpha;
                        g_q[3 * e] += d_q * dx * dx;
                        g_q[3 * e + 1] += d_q * 2.0 * dx * dy;
                        g_q[3 * e + 2] += d_q * dy * dy;
                        double ddx = d_q * 2.0 * (inv_a[s] * dx + inv_b[s] * dy);
                        double ddy = d_q * 2.0 * (inv_b[s] * dx + inv_c[s] * dy);
                        g_mu[2 * e] -= ddx;
                        g_mu[2 * e + 1] -= ddy;
                    }
                    s0 += w * a[0];
                    s1 += w * a[1];
                    s2 += w * a[2];
                    t_next = t_k;
                }
            }
    }
}

/* bin_tiles + forward_kernel without materialising the CSR (full frames at
 * configs 2-5, whose random-init CSR holds ~1e9 entries). Per tile row, the
 * ranks whose tile range covers the row are collected in rank order — the
 * order bin_tiles scatters them in (_raster_kernels.py:137-142) — then each
 * tile of the row blends the ranks whose column range covers it, with
 * forward_kernel's per-pixel rules (_raster_kernels.py:146-201). With
 * terminate, a tile stops once every pixel has T < cutoff: forward_kernel
 * skips each later entry per pixel at that point, so the planes are
 * identical. attr2 (optional) is blended with the same weights in the same
 * pass (alpha and T do not depend on the attribute). */
void oracle_forward_stream(int64_t width, int64_t height, int64_t tile, int64_t k,
                           const double *sx, const double *sy, const double *radius,
                           const double *inv_a, const double *inv_b, const double *inv_c,
                           const double *opac, const double *attr, const double *attr2,
                           double alpha_max, int terminate, double *out, double *out2,
                           double *trans) {
    int64_t ntx = (width + tile - 1) / tile, nty = (height + tile - 1) / tile;
    double ft = (double)tile;
    int64_t *rx0 = (int64_t *)malloc(sizeof(int64_t) * (k > 0 ? k : 1));
    int64_t *rx1 = (int64_t *)malloc(sizeof(int64_t) * (k > 0 ? k : 1));
    int64_t *ry0 = (int64_t *)malloc(sizeof(int64_t) * (k > 0 ? k : 1));
    int64_t *ry1 = (int64_t *)malloc(sizeof(int64_t) * (k > 0 ? k : 1));
    int64_t *row = (int64_t *)malloc(sizeof(int64_t) * (k > 0 ? k : 1));
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < k; ++i)
        tile_range(sx[i], sy[i], radius[i], ft, ntx, nty, &rx0[i], &rx1[i], &ry0[i], &ry1[i]);
    for (int64_t ty = 0; ty < nty; ++ty) {
        int64_t nrow = 0;
        for (int64_t i = 0; i < k; ++i)
            if (ry0[i] <= ty && ty <= ry1[i] && rx0[i] <= rx1[i]) row[nrow++] = i;
#pragma omp parallel for schedule(dynamic, 1)
        for (int64_t tx = 0; tx < ntx; ++tx) {
            int64_t x_end = imin((tx + 1) * tile, width), y_end = imin((ty + 1) * tile, height);
            int64_t npix = (x_end - tx * tile) * (y_end - ty * tile), nsat = 0;
            for (int64_t e = 0; e < nrow; ++e) {
                int64_t s = row[e];
                if (tx < rx0[s] || tx > rx1[s]) continue;
                double rad = radius[s] + 1.0, rr = rad * rad;
                double mx = sx[s], my = sy[s];
                double ia = inv_a[s], ib = inv_b[s], ic = inv_c[s], op = opac[s];
                int64_t px0 = imax(tx * tile, (int64_t)ceil(mx - rad));
                int64_t px1 = imin(x_end - 1, (int64_t)floor(mx + rad));
                int64_t py0 = imax(ty * tile, (int64_t)ceil(my - rad));
                int64_t py1 = imin(y_end - 1, (int64_t)floor(my + rad));
                for (int64_t py = py0; py <= py1; ++py) {
                    double dy = (double)py - my;
                    for (int64_t px = px0; px <= px1; ++px) {
                        int64_t pix = py * width + px;
                        double tr = trans[pix];
                        if (terminate && tr < TRANS_CUTOFF) continue;
                        double dx = (double)px - mx;
                        if (dx * dx + dy * dy > rr) continue;
                        double q = ia * dx * dx + 2.0 * ib * dx * dy + ic * dy * dy;
                        double alpha = op * exp(-0.5 * q);
                        if (alpha > alpha_max) alpha = alpha_max;
                        if (alpha < ALPHA_CUTOFF) continue;
                        double w = tr * alpha;
                        out[3 * pix] += w * attr[3 * s];
                        out[3 * pix + 1] += w * attr[3 * s + 1];
                        out[3 * pix + 2] += w * attr[3 * s + 2];
                        if (attr2) {
                            out2[3 * pix] += w * attr2[3 * s];
                            out2[3 * pix + 1] += w * attr2[3 * s + 1];
                            out2[3 * pix + 2] += w * attr2[3 * s + 2];
                        }
                        trans[pix] = tr * (1.0 - alpha);
                        if (terminate && trans[pix] < TRANS_CUTOFF) ++nsat;
                    }
                }
                if (terminate && nsat == npix) break;
            }
        }
    }
    free(rx0);
    free(rx1);
    free(ry0);
    free(ry1);
    free(row);
}
