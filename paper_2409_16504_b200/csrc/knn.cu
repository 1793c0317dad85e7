// Analytic estimators on the device: exact k-nearest
// neighbours on a uniform grid (_neighbors.py:33-128), estimate_local_pca and
// estimate_global (estimators.py:41-211).
//
// kNN: cell size h = (V/N)^(1/3) formed on the host with the reference's
// float64 expression; points sorted by packed cell key (stable, so by index
// inside a cell); one thread per query expands Chebyshev shells, looks cells
// up by binary search in the sorted unique keys and keeps the k best
// (d2, index) pairs sorted with the index as the tie-break — the result is
// the unique k-prefix of that total order, so indices and distances are
// bit-identical to the reference (distances computed in the same float64
// order, no FMA: this file is compiled with -fmad=false).
#include "common.cuh"

namespace sfb {

constexpr int kKnnMax = 64;

struct KnnGrid {
    double lo[3], h;
    int64_t dims[3], cap[3];
};

__device__ __forceinline__ int64_t cell_of(double p, double lo, double h, int64_t cap) {
    const int64_t c = (int64_t)floor((p - lo) / h);
    return c < cap ? c : cap;
}

__global__ void k_knn_keys(const double *__restrict__ pos, int64_t n, KnnGrid G,
                           unsigned long long *__restrict__ keys, uint32_t *__restrict__ vals) {
    SFB_FOR(i, n) {
        const int64_t cx = cell_of(pos[3 * i], G.lo[0], G.h, G.cap[0]);
        const int64_t cy = cell_of(pos[3 * i + 1], G.lo[1], G.h, G.cap[1]);
        const int64_t cz = cell_of(pos[3 * i + 2], G.lo[2], G.h, G.cap[2]);
        keys[i] = ((unsigned long long)cz << 42) | ((unsigned long long)cy << 21) | (unsigned long long)cx;
        vals[i] = (uint32_t)i;
    }
}

__global__ void k_cell_heads(const unsigned long long *__restrict__ keys, int64_t n, int32_t *__restrict__ flag) {
    SFB_FOR(j, n) flag[j] = (j == 0 || keys[j] != keys[j - 1]) ? 1 : 0;
}

__global__ void k_cell_table(const unsigned long long *__restrict__ keys, const int32_t *__restrict__ incl,
                             int64_t n, unsigned long long *__restrict__ ukeys, int32_t *__restrict__ starts,
                             int64_t *__restrict__ d_cells) {
    SFB_FOR(j, n) {
        const int32_t u = incl[j] - 1;
        if (j == 0 || incl[j - 1] != incl[j]) {
            ukeys[u] = keys[j];
            starts[u] = (int32_t)j;
        }
        if (j == n - 1) {
            starts[u + 1] = (int32_t)n;
            *d_cells = u + 1;
        }
    }
}

__device__ __forceinline__ void knn_insert(double *bd, int32_t *bi, int k, double d2, int32_t j) {
    const double last = bd[k - 1];
    if (d2 > last || (d2 == last && 0 <= bi[k - 1] && bi[k - 1] < j)) return;
    int p = k - 1;
    while (p > 0 && (bd[p - 1] > d2 || (bd[p - 1] == d2 && bi[p - 1] > j))) {
        bd[p] = bd[p - 1];
        bi[p] = bi[p - 1];
        --p;
    }
    bd[p] = d2;
    bi[p] = j;
}

__global__ void __launch_bounds__(128)
k_knn_query(const double *__restrict__ pos, int64_t n, int k, KnnGrid G,
            const double *__restrict__ spos, const uint32_t *__restrict__ sidx,
            const unsigned long long *__restrict__ ukeys, const int32_t *__restrict__ starts,
            const int64_t *__restrict__ d_cells, double *__restrict__ out_d2,
            int64_t *__restrict__ out_idx) {
    const int64_t ncell = *d_cells;
    SFB_FOR(i, n) {
        double bd[kKnnMax];
        int32_t bi[kKnnMax];
        for (int q = 0; q < k; ++q) {
            bd[q] = __longlong_as_double(0x7ff0000000000000ll);   // +inf
            bi[q] = -1;
        }
        const double qx = pos[3 * i], qy = pos[3 * i + 1], qz = pos[3 * i + 2];
        auto clampc = [](int64_t c, int64_t d) { return c < 0 ? 0 : (c > d - 1 ? d - 1 : c); };
        const int64_t cx = clampc((int64_t)floor((qx - G.lo[0]) / G.h), G.dims[0]);
        const int64_t cy = clampc((int64_t)floor((qy - G.lo[1]) / G.h), G.dims[1]);
        const int64_t cz = clampc((int64_t)floor((qz - G.lo[2]) / G.h), G.dims[2]);
        const int64_t last_shell = max(max(cx, G.dims[0] - 1 - cx),
                                       max(max(cy, G.dims[1] - 1 - cy), max(cz, G.dims[2] - 1 - cz)));
        for (int64_t shell = 0;; ++shell) {
            for (int64_t dz = -shell; dz <= shell; ++dz) {
                const int64_t z = cz + dz;
                if (z < 0 || z >= G.dims[2]) continue;
                for (int64_t dy = -shell; dy <= shell; ++dy) {
                    const int64_t y = cy + dy;
                    if (y < 0 || y >= G.dims[1]) continue;
                    const bool face = llabs(dz) == shell || llabs(dy) == shell;
                    for (int64_t dx = -shell; dx <= shell; dx += (face || shell == 0) ? 1 : 2 * shell) {
                        const int64_t x = cx + dx;
                        if (x < 0 || x >= G.dims[0]) continue;
                        const unsigned long long key = ((unsigned long long)z << 42) |
                                                       ((unsigned long long)y << 21) | (unsigned long long)x;
                        int64_t lo = 0, hi = ncell;   // searchsorted
                        while (lo < hi) {
                            const int64_t mid = (lo + hi) >> 1;
                            if (ukeys[mid] < key) lo = mid + 1;
                            else hi = mid;
                        }
                        if (lo >= ncell || ukeys[lo] != key) continue;
                        for (int32_t row = starts[lo]; row < starts[lo + 1]; ++row) {
                            const int32_t j = (int32_t)sidx[row];
                            if (j == i) continue;
                            const double ex = spos[3 * (int64_t)row] - qx, ey = spos[3 * (int64_t)row + 1] - qy,
                                         ez = spos[3 * (int64_t)row + 2] - qz;
                            knn_insert(bd, bi, k, ex * ex + ey * ey + ez * ez, j);
                        }
                    }
                }
            }
            // points beyond this shell are at least shell*h away
            const double reach = (double)shell * G.h;
            if (bi[k - 1] >= 0 && bd[k - 1] <= reach * reach) break;
            if (shell >= last_shell) break;
        }
        for (int q = 0; q < k; ++q) {
            out_d2[(int64_t)i * k + q] = bd[q];
            out_idx[(int64_t)i * k + q] = bi[q];
        }
    }
}

__global__ void k_gather_sorted(const double *__restrict__ pos, const uint32_t *__restrict__ order, int64_t n,
                                double *__restrict__ spos) {
    SFB_FOR(j, n) {
        const int64_t i = order[j];
        spos[3 * j] = pos[3 * i];
        spos[3 * j + 1] = pos[3 * i + 1];
        spos[3 * j + 2] = pos[3 * i + 2];
    }
}

// host half: grid parameters with the reference's float64 expressions
// (_neighbors.py:100-111)
static KnnGrid knn_grid(const double *lo_hi, int64_t n) {
    KnnGrid G{};
    double ext[3], emax = 0.0;
    for (int a = 0; a < 3; ++a) {
        G.lo[a] = lo_hi[a];
        ext[a] = lo_hi[3 + a] - lo_hi[a];
        emax = std::max(emax, ext[a]);
    }
    const double volume = (ext[0] * ext[1]) * ext[2];
    double h = volume > 0 ? std::pow(volume / (double)n, 1.0 / 3.0) : emax;
    h = std::max(std::max(h, emax / (double)((1 << 21) - 2)), 1e-300);
    if (emax == 0.0) h = 1.0;
    G.h = h;
    for (int a = 0; a < 3; ++a) {
        G.cap[a] = std::max<int64_t>((int64_t)(ext[a] / h), 0);
        G.dims[a] = G.cap[a] + 1;
    }
    return G;
}

void knn_run(sfb_ctx *ctx, const double *pos, int64_t n, int k, double *out_d2, int64_t *out_idx) {
    SFB_REQUIRE(k >= 1 && k <= kKnnMax, "k must be in [1, 64]");
    SFB_REQUIRE(k < n, std::to_string(k) + " neighbors need at least " + std::to_string(k + 1) +
                           " points, got " + std::to_string(n));
    cudaStream_t st = ctx->stream;
    double lo_hi[6];
    bbox_run(ctx, pos, n, lo_hi);
    const KnnGrid G = knn_grid(lo_hi, n);
    auto *keys = ctx->arena.alloc<unsigned long long>(n), *keys2 = ctx->arena.alloc<unsigned long long>(n);
    uint32_t *vals = ctx->arena.alloc<uint32_t>(n), *vals2 = ctx->arena.alloc<uint32_t>(n);
    k_knn_keys<<<dgrid(n, 256), 256, 0, st>>>(pos, n, G, keys, vals);
    SFB_CHECK_LAUNCH();
    int bits = 0;
    while (bits < 64 && ((unsigned long long)(((uint64_t)G.cap[2] << 42) | ((uint64_t)G.cap[1] << 21) |
                                              (uint64_t)G.cap[0]) >> bits))
        ++bits;
    const bool second = dsort_pairs<unsigned long long>(ctx, keys, vals, keys2, vals2, nullptr, n,
                                                        bits > 0 ? bits : 1);
    const unsigned long long *ks = second ? keys2 : keys;
    const uint32_t *vs = second ? vals2 : vals;
    int32_t *flag = ctx->arena.alloc<int32_t>(n);
    k_cell_heads<<<dgrid(n, 256), 256, 0, st>>>(ks, n, flag);
    dscan(ctx, flag, flag, nullptr, n, nullptr, true);
    auto *ukeys = ctx->arena.alloc<unsigned long long>(n);
    int32_t *starts = ctx->arena.alloc<int32_t>(n + 1);
    int64_t *d_cells = ctx->arena.alloc<int64_t>(1);
    k_cell_table<<<dgrid(n, 256), 256, 0, st>>>(ks, flag, n, ukeys, starts, d_cells);
    double *spos = ctx->arena.alloc<double>(3 * (size_t)n);
    k_gather_sorted<<<dgrid(n, 256), 256, 0, st>>>(pos, vs, n, spos);
    k_knn_query<<<dgrid(n, 128, 16), 128, 0, st>>>(pos, n, k, G, spos, vs, ukeys, starts, d_cells, out_d2,
                                                   out_idx);
    SFB_CHECK_LAUNCH();
}

// ------------------------------------------------------------------ local PCA
// symeig3x3 (estimators.py:41-137): trigonometric closed form on the
// max-abs-scaled matrix, primary eigenvector = the better separated extreme
// one from the largest cross product of the rows of (A - lam I), secondary
// orthogonalised against it, exactly diagonal inputs sorted directly.
__device__ void cross3(const double *a, const double *b, double *c) {
    c[0] = a[1] * b[2] - a[2] * b[1];
    c[1] = a[2] * b[0] - a[0] * b[2];
    c[2] = a[0] * b[1] - a[1] * b[0];
}

__device__ bool cross_row_eigvec(const double a[3][3], double lam, double *v) {
    double b[3][3];
    for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) b[r][c] = a[r][c] - (r == c ? lam : 0.0);
    double cr[3][3];
    cross3(b[0], b[1], cr[0]);
    cross3(b[0], b[2], cr[1]);
    cross3(b[1], b[2], cr[2]);
    int pick = 0;
    double best = -1.0;
    for (int q = 0; q < 3; ++q) {
        const double nn = sqrt(cr[q][0] * cr[q][0] + cr[q][1] * cr[q][1] + cr[q][2] * cr[q][2]);
        if (nn > best) {   // argmax: first maximum
            best = nn;
            pick = q;
        }
    }
    const double d = fmax(best, 1e-300);
    for (int c = 0; c < 3; ++c) v[c] = cr[pick][c] / d;
    return best > 1e-12;
}

__device__ void any_perpendicular(const double *v, double *w) {
    int axis = 0;
    double m = fabs(v[0]);
    for (int a = 1; a < 3; ++a)
        if (fabs(v[a]) < m) {
            m = fabs(v[a]);
            axis = a;
        }
    double e[3] = {0.0, 0.0, 0.0};
    e[axis] = 1.0;
    const double dot = e[0] * v[0] + e[1] * v[1] + e[2] * v[2];
    for (int c = 0; c < 3; ++c) w[c] = e[c] - dot * v[c];
    const double nn = sqrt(w[0] * w[0] + w[1] * w[1] + w[2] * w[2]);
    for (int c = 0; c < 3; ++c) w[c] /= nn;
}

__device__ void symeig3x3(const double m[3][3], double lam[3], double fr[3][3]) {
    double scale = 0.0;
    for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) scale = fmax(scale, fabs(m[r][c]));
    const double s = scale > 0 ? scale : 1.0;
    double a[3][3];
    for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) a[r][c] = m[r][c] / s;
    const double a00 = a[0][0], a11 = a[1][1], a22 = a[2][2], a01 = a[0][1], a02 = a[0][2], a12 = a[1][2];
    const double off = a01 * a01 + a02 * a02 + a12 * a12;
    const double q = (a00 + a11 + a22) / 3.0;
    const double p2 = (a00 - q) * (a00 - q) + (a11 - q) * (a11 - q) + (a22 - q) * (a22 - q) + 2.0 * off;
    const double p = sqrt(fmax(p2 / 6.0, 0.0));
    const double sp = p > 0 ? p : 1.0;
    double b[3][3];
    for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) b[r][c] = (a[r][c] - (r == c ? q : 0.0)) / sp;
    const double det = b[0][0] * (b[1][1] * b[2][2] - b[1][2] * b[1][2]) -
                       b[0][1] * (b[0][1] * b[2][2] - b[1][2] * b[0][2]) +
                       b[0][2] * (b[0][1] * b[1][2] - b[1][1] * b[0][2]);
    const double phi = acos(fmin(fmax(det / 2.0, -1.0), 1.0)) / 3.0;
    const double hi = q + 2.0 * p * cos(phi);
    const double lo = q + 2.0 * p * cos(phi + 2.0 * 3.141592653589793 / 3.0);
    const double mid = 3.0 * q - hi - lo;
    lam[0] = lo;
    lam[1] = mid;
    lam[2] = hi;
    const bool hi_primary = (hi - mid) >= (mid - lo);
    double vp[3], vs[3];
    const bool okp = cross_row_eigvec(a, hi_primary ? hi : lo, vp);
    const bool oks = cross_row_eigvec(a, hi_primary ? lo : hi, vs);
    if (!okp) {
        vp[0] = 1.0;
        vp[1] = 0.0;
        vp[2] = 0.0;
    }
    const double dp = vs[0] * vp[0] + vs[1] * vp[1] + vs[2] * vp[2];
    for (int c = 0; c < 3; ++c) vs[c] -= dp * vp[c];
    const double sn = sqrt(vs[0] * vs[0] + vs[1] * vs[1] + vs[2] * vs[2]);
    if (oks && sn > 1e-8) {
        for (int c = 0; c < 3; ++c) vs[c] /= fmax(sn, 1e-300);
    } else {
        any_perpendicular(vp, vs);
    }
    const double *rh = hi_primary ? vp : vs, *rl = hi_primary ? vs : vp;
    for (int c = 0; c < 3; ++c) {
        fr[2][c] = rh[c];
        fr[0][c] = rl[c];
    }
    cross3(fr[2], fr[0], fr[1]);
    if (off == 0.0) {   // exactly diagonal: sorted diagonal, permutation frame
        double d[3] = {a00, a11, a22};
        int o[3] = {0, 1, 2};
        for (int x = 1; x < 3; ++x)   // stable insertion sort
            for (int y = x; y > 0 && d[o[y - 1]] > d[o[y]]; --y) {
                const int t = o[y];
                o[y] = o[y - 1];
                o[y - 1] = t;
            }
        for (int r = 0; r < 3; ++r) lam[r] = d[o[r]];
        for (int r = 0; r < 3; ++r)
            for (int c = 0; c < 3; ++c) fr[r][c] = 0.0;
        fr[0][o[0]] = 1.0;
        fr[2][o[2]] = 1.0;
        cross3(fr[2], fr[0], fr[1]);
    }
    for (int r = 0; r < 3; ++r) lam[r] *= s;
}

// rotmat_to_quat (gaussians.py:178-209): the largest of the four branches
__device__ void rotmat_to_quat(const double r[3][3], double *qo) {
    const double m[4] = {1.0 + r[0][0] + r[1][1] + r[2][2], 1.0 + r[0][0] - r[1][1] - r[2][2],
                         1.0 - r[0][0] + r[1][1] - r[2][2], 1.0 - r[0][0] - r[1][1] + r[2][2]};
    int b = 0;
    for (int q = 1; q < 4; ++q)
        if (m[q] > m[b]) b = q;
    const double big = 0.5 * sqrt(m[b]), quarter = 0.25 / big;
    const double wx = r[2][1] - r[1][2], wy = r[0][2] - r[2][0], wz = r[1][0] - r[0][1];
    const double xy = r[1][0] + r[0][1], xz = r[0][2] + r[2][0], yz = r[2][1] + r[1][2];
    double q[4];
    if (b == 0) {
        q[0] = big; q[1] = wx * quarter; q[2] = wy * quarter; q[3] = wz * quarter;
    } else if (b == 1) {
        q[0] = wx * quarter; q[1] = big; q[2] = xy * quarter; q[3] = xz * quarter;
    } else if (b == 2) {
        q[0] = wy * quarter; q[1] = xy * quarter; q[2] = big; q[3] = yz * quarter;
    } else {
        q[0] = wz * quarter; q[1] = xz * quarter; q[2] = yz * quarter; q[3] = big;
    }
    const double nn = sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
    for (int c = 0; c < 4; ++c) qo[c] = q[c] / nn;
}

// estimate_local_pca per point (estimators.py:166-211)
__global__ void k_local_pca(const double *__restrict__ pos, int64_t n, int k, const int64_t *__restrict__ idx,
                            const double *__restrict__ mean_c, double sigma_mult, double dbar,
                            double *__restrict__ scales, double *__restrict__ quats,
                            double *__restrict__ normals) {
    SFB_FOR(i, n) {
        const int64_t *nb = idx + i * k;
        double mu[3] = {0.0, 0.0, 0.0};
        for (int q = 0; q < k; ++q)
            for (int c = 0; c < 3; ++c) mu[c] += pos[3 * nb[q] + c];
        for (int c = 0; c < 3; ++c) mu[c] /= (double)k;
        double cov[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
        for (int q = 0; q < k; ++q) {
            double d[3];
            for (int c = 0; c < 3; ++c) d[c] = pos[3 * nb[q] + c] - mu[c];
            for (int r = 0; r < 3; ++r)
                for (int c = 0; c < 3; ++c) cov[r][c] += d[r] * d[c];
        }
        for (int r = 0; r < 3; ++r)
            for (int c = 0; c < 3; ++c) cov[r][c] /= (double)k;
        double lam[3], fr[3][3];
        symeig3x3(cov, lam, fr);
        for (int row = 0; row < 2; ++row) {   // largest-|component| positive
            int am = 0;
            for (int c = 1; c < 3; ++c)
                if (fabs(fr[row][c]) > fabs(fr[row][am])) am = c;
            if (fr[row][am] < 0)
                for (int c = 0; c < 3; ++c) fr[row][c] = -fr[row][c];
        }
        cross3(fr[0], fr[1], fr[2]);
        for (int c = 0; c < 3; ++c)
            scales[3 * i + c] = fmax(sigma_mult * sqrt(fmax(lam[c], 0.0)), 0.1 * dbar);
        double nv[3] = {fr[0][0], fr[0][1], fr[0][2]};
        const double out = nv[0] * (pos[3 * i] - mean_c[0]) + nv[1] * (pos[3 * i + 1] - mean_c[1]) +
                           nv[2] * (pos[3 * i + 2] - mean_c[2]);
        const double sg = out < 0 ? -1.0 : 1.0;
        for (int c = 0; c < 3; ++c) normals[3 * i + c] = nv[c] * sg;
        rotmat_to_quat(fr, quats + 4 * i);
    }
}

// per-point nearest-neighbour distance and per-column centroid partials
__global__ void k_nn_dist(const double *__restrict__ d2, int64_t n, int k, double *__restrict__ dist) {
    SFB_FOR(i, n) dist[i] = sqrt(d2[i * k]);
}

void local_pca_run(sfb_ctx *ctx, const double *pos, int64_t n, int k, double sigma_mult,
                   const int64_t *idx, double dbar, const double *mean_c, double *scales,
                   double *quats, double *normals) {
    k_local_pca<<<dgrid(n, 128, 16), 128, 0, ctx->stream>>>(pos, n, k, idx, mean_c, sigma_mult, dbar,
                                                            scales, quats, normals);
    SFB_CHECK_LAUNCH();
}

void nn_dist_run(sfb_ctx *ctx, const double *d2, int64_t n, int k, double *dist) {
    k_nn_dist<<<dgrid(n, 256), 256, 0, ctx->stream>>>(d2, n, k, dist);
    SFB_CHECK_LAUNCH();
}

}  // namespace sfb
