// Splatting pipeline on the device (compiled with -fmad=false).
//
// Reference: project_kernel / bin_tiles / forward_kernel
// (_raster_kernels.py:20-201) and _prepare / _compose / render
// (rasterizer.py:99-166). Contract kept bit-for-bit where the reference is
// integer or IEEE-exact: projection, covariance and depth in float64 with the
// numba expression order and no FMA contraction, blend order = stable sort of
// (depth, input index), tile ranges floor((s -+ r)/tile) on the alpha-support
// radius, per-pixel box/circle tests, "T < 1/255 is checked before each splat".
//
// B200 design:
//   1. project per geometry row (per splat, or per voxel in the fused frame);
//   2. compact kept points, stable LSD radix sort of float64 depth bits with
//      the point index as payload -> rank order (ties by index);
//   3. split the rank order into RUNS of consecutive points with identical
//      geometry (a voxel's points share centre/cov/opacity, so P2ENet splats
//      collapse ~33x); one alpha per (run, pixel), colours stay per point;
//   4. bin runs into a three-level tile pyramid — 16 px tiles, 8x8-tile super
//      tiles, one whole-image list — choosing per run the finest level with
//      <= 16 entries, so the giant random-init splats never expand into
//      billions of (tile, splat) keys;
//   5. one CTA per tile walks the three rank-sorted lists as a merge (rank
//      windows + a shared-memory bitmap), tests exact tile coverage, blends
//      RGB + normal (+ depth) + T in float64 registers in ONE pass, and stops
//      when every pixel of the tile has T < 1/255 — identical to the
//      reference, whose per-pixel skip makes all later splats no-ops.
#include <cstddef>
#include <utility>

#include "common.cuh"

namespace sfb {

constexpr double kCutoff = 1.0 / 255.0;
constexpr int kFineMax = 16;   // tiles per run at the fine level
constexpr int kSuper = 8;      // tiles per super-tile edge
constexpr int kSuperMax = 16;  // super tiles per run at the middle level
constexpr int kWin = 512;      // rank window of the merge
// compositor CTA: 128 threads, two pixels each for the default 16x16 tile
// (two independent per-pixel chains per thread), 8 CTAs per SM; A/B on
// config 2 with 8 frames in flight: 0.308 ms/frame vs 0.316 for 256 threads x
// one pixel (64 threads x 4 pixels: 0.34, register-starved). The rank window
// (512) and the chunk (64 runs) keep its shared memory at ~14 KB: the rest of
// the SM's 256 KB stays L1 for the runs' colour reads (0.0615 vs 0.0625 ms
// with a 2048-rank window and 128-run chunks)
constexpr int kCT = 128;       // compositor threads per CTA
constexpr int kCompMinBlocks = 8;
constexpr int kCompReps = 4;   // timed re-launches of the compositor in stage-timing mode
constexpr int kChunk = 64;     // candidate runs staged per compositing chunk

// ------------------------------------------------------------ 1. projection
__device__ __forceinline__ void project_one(const double *__restrict__ p, const double *__restrict__ q,
                                            const double *__restrict__ sc, const Cam &C, double z_near,
                                            double dil, double *o_sx, double *o_sy, double *o_d,
                                            double *o_a, double *o_b, double *o_c, double *o_r,
                                            uint8_t *o_keep) {
    const double *R = C.r;
    double px = R[0] * p[0] + R[1] * p[1] + R[2] * p[2] + C.t[0];
    double py = R[3] * p[0] + R[4] * p[1] + R[5] * p[2] + C.t[1];
    double pz = R[6] * p[0] + R[7] * p[1] + R[8] * p[2] + C.t[2];
    uint8_t ok = 0;
    double vsx = 0, vsy = 0, vd = 0, va = 0, vb = 0, vc = 0, vr = 0;
    if (pz > z_near) {
        double w = q[0], x = q[1], y = q[2], z = q[3];
        double qn = sqrt(w * w + x * x + y * y + z * z);
        w /= qn;
        x /= qn;
        y /= qn;
        z /= qn;
        double r[9] = {1.0 - 2.0 * (y * y + z * z), 2.0 * (x * y - w * z), 2.0 * (x * z + w * y),
                       2.0 * (x * y + w * z), 1.0 - 2.0 * (x * x + z * z), 2.0 * (y * z - w * x),
                       2.0 * (x * z - w * y), 2.0 * (y * z + w * x), 1.0 - 2.0 * (x * x + y * y)};
        double u[9];
#pragma unroll
        for (int a = 0; a < 3; ++a)
#pragma unroll
            for (int b = 0; b < 3; ++b)
                u[3 * a + b] = r[3 * a] * R[3 * b] + r[3 * a + 1] * R[3 * b + 1] + r[3 * a + 2] * R[3 * b + 2];
        double d0 = sc[0] * sc[0], d1 = sc[1] * sc[1], d2 = sc[2] * sc[2];
#define SIG(j, k) (d0 * u[j] * u[k] + d1 * u[3 + j] * u[3 + k] + d2 * u[6 + j] * u[6 + k])
        double s00 = SIG(0, 0), s01 = SIG(0, 1), s02 = SIG(0, 2);
        double s11 = SIG(1, 1), s12 = SIG(1, 2), s22 = SIG(2, 2);
#undef SIG
        double jx = C.fx / pz, jy = C.fy / pz;
        double jxz = -C.fx * px / (pz * pz), jyz = -C.fy * py / (pz * pz);
        double a = jx * jx * s00 + 2.0 * jx * jxz * s02 + jxz * jxz * s22 + dil;
        double b = jx * jy * s01 + jx * jyz * s02 + jxz * jy * s12 + jxz * jyz * s22;
        double c = jy * jy * s11 + 2.0 * jy * jyz * s12 + jyz * jyz * s22 + dil;
        double mid = 0.5 * (a + c);
        double gap = sqrt(fmax(0.25 * (a - c) * (a - c) + b * b, 0.0));
        double rr = 3.0 * sqrt(fmax(mid + gap, 0.0));
        double csx = jx * px + C.cx, csy = jy * py + C.cy;
        if (!(csx + rr < 0.0 || csx - rr > (double)C.w - 1.0 || csy + rr < 0.0 ||
              csy - rr > (double)C.h - 1.0)) {
            ok = 1;
            vsx = csx;
            vsy = csy;
            vd = pz;
            va = a;
            vb = b;
            vc = c;
            vr = rr;
        }
    }
    *o_sx = vsx;
    *o_sy = vsy;
    *o_d = vd;
    *o_a = va;
    *o_b = vb;
    *o_c = vc;
    *o_r = vr;
    *o_keep = ok;
}

__global__ void k_project(const double *__restrict__ centers, const double *__restrict__ quats,
                          const double *__restrict__ scales, const int64_t *__restrict__ d_n,
                          int64_t n_fixed, const FrameParams *__restrict__ FP, double z_near,
                          double dil, double *__restrict__ sx, double *__restrict__ sy,
                          double *__restrict__ depth, double *__restrict__ ca,
                          double *__restrict__ cb, double *__restrict__ cc,
                          double *__restrict__ rad3, uint8_t *__restrict__ keep,
                          unsigned long long *__restrict__ zr) {
    const int64_t n = d_n ? *d_n : n_fixed;
    const Cam C = FP->cam;
    // the kept depths' range for the depth-order keys, reduced here (zr:
    // DevCounts words, zero-initialised per frame) instead of a second pass
    unsigned long long lo = ~0ull, hi = 0ull;
    for (int64_t i0 = blockIdx.x * (int64_t)blockDim.x; i0 < n; i0 += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = i0 + threadIdx.x;
        if (i < n) {
            project_one(centers + 3 * i, quats + 4 * i, scales + 3 * i, C, z_near, dil, sx + i, sy + i,
                        depth + i, ca + i, cb + i, cc + i, rad3 + i, keep + i);
            if (zr && keep[i]) {
                const unsigned long long b = (unsigned long long)__double_as_longlong(depth[i]);
                lo = b < lo ? b : lo;
                hi = b > hi ? b : hi;
            }
        }
    }
    if (zr) {
        for (int o = 16; o; o >>= 1) {
            const unsigned long long l2 = __shfl_xor_sync(0xffffffffu, lo, o);
            const unsigned long long h2 = __shfl_xor_sync(0xffffffffu, hi, o);
            lo = l2 < lo ? l2 : lo;
            hi = h2 > hi ? h2 : hi;
        }
        if ((threadIdx.x & 31) == 0 && hi) {
            atomicMax(&zr[0], ~lo);
            atomicMax(&zr[1], hi);
        }
    }
}

void project_run(sfb_ctx *ctx, const double *centers, const double *quats, const double *scales,
                 const int64_t *d_n, int64_t n_bound, const FrameParams *FP, double z_near,
                 double dilation, double *sx, double *sy, double *depth, double *ca, double *cb,
                 double *cc, double *radius, uint8_t *keep, unsigned long long *zr) {
    if (n_bound == 0) return;
    k_project<<<dgrid(n_bound, 128), 128, 0, ctx->stream>>>(centers, quats, scales, d_n, n_bound, FP,
                                                            z_near, dilation, sx, sy, depth, ca, cb,
                                                            cc, radius, keep, zr);
    SFB_CHECK_LAUNCH();
}

// ------------------------------------------------------------ 2. depth order
struct Proj {
    double *sx, *sy, *depth, *a, *b, *c, *r3;
    uint8_t *keep;
};

static Proj project_inputs(sfb_ctx *ctx, const RenderInputs &in, const FrameParams *FP,
                           unsigned long long *zr = nullptr) {
    Proj P;
    const int64_t n = in.n_geom;   // bound
    double *blk = ctx->arena.alloc<double>(7 * (size_t)(n > 0 ? n : 1));
    P.sx = blk;
    P.sy = blk + n;
    P.depth = blk + 2 * n;
    P.a = blk + 3 * n;
    P.b = blk + 4 * n;
    P.c = blk + 5 * n;
    P.r3 = blk + 6 * n;
    P.keep = ctx->arena.alloc<uint8_t>(n > 0 ? n : 1);
    project_run(ctx, in.centers, in.quats, in.scales, in.d_n_geom, n, FP, 0.01, 0.3, P.sx, P.sy,
                P.depth, P.a, P.b, P.c, P.r3, P.keep, zr);
    return P;
}

// Depth order = stable sort of (float64 depth, point index) over kept points
// (rasterizer.py:105). Sorting 64-bit depth keys costs 8 radix passes, so the
// sort runs on a 32-bit MONOTONE quantisation q(d) = floor((d - zmin) * s)
// (4 passes); points with equal q keep index order (stable), and a fix-up
// pass re-sorts each equal-q group by the exact (depth bits, index) key.
// Equal-q groups are almost always one voxel's points (identical depth,
// already in index order: O(k) check) or exact ties.
__device__ __forceinline__ unsigned long long dbits(double d) {
    return (unsigned long long)__double_as_longlong(d);
}

__global__ void k_depth_keys(int64_t n, const int32_t *__restrict__ p2g, const Proj P,
                             const unsigned long long *__restrict__ zr, uint32_t *__restrict__ keys,
                             uint32_t *__restrict__ vals, int64_t *__restrict__ d_kept) {
    const double zmin = __longlong_as_double((long long)~zr[0]);
    const double zmax = __longlong_as_double((long long)zr[1]);
    const double scale = zmax > zmin ? 4294967294.0 / (zmax - zmin) : 0.0;
    SFB_FOR(i, ((n + 31) & ~int64_t(31))) {
        bool k = false;
        if (i < n) {
            const int64_t g = p2g ? p2g[i] : i;
            k = P.keep[g];
            uint32_t key = 0xffffffffu;
            if (k) key = (uint32_t)fmin(floor((P.depth[g] - zmin) * scale), 4294967294.0);
            keys[i] = key;
            vals[i] = (uint32_t)i;
        }
        const unsigned ball = __ballot_sync(0xffffffffu, k);
        if ((threadIdx.x & 31) == 0 && ball) atomicAdd((unsigned long long *)d_kept, (unsigned long long)__popc(ball));
    }
}

// exact (depth bits, index) order inside every group of equal quantised keys:
// (1) full depth bits per rank, (2) flag ranks that are out of order w.r.t.
// their predecessor in the same group and mark that group's head (rare),
// (3) heads of marked groups insertion-sort their group
__global__ void k_depth_full(const uint32_t *__restrict__ src, const int32_t *__restrict__ p2g,
                             const Proj P, const int64_t *__restrict__ d_kept,
                             unsigned long long *__restrict__ full) {
    const int64_t K = *d_kept;
    SFB_FOR(j, K) {
        const uint32_t i = src[j];
        full[j] = dbits(P.depth[p2g ? p2g[i] : (int64_t)i]);
    }
}

__global__ void k_depth_mark(const uint32_t *__restrict__ keys,
                             const unsigned long long *__restrict__ full,
                             const int64_t *__restrict__ d_kept, uint8_t *__restrict__ need,
                             uint32_t *__restrict__ heads, int64_t *__restrict__ n_heads) {
    const int64_t K = *d_kept;
    SFB_FOR(j, K) {
        if (j == 0 || keys[j] != keys[j - 1] || full[j] >= full[j - 1]) continue;
        // first element of the group: keys are sorted, so binary search
        int64_t lo = 0, hi = j;
        const uint32_t kj = keys[j];
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if (keys[mid] < kj) lo = mid + 1;
            else hi = mid;
        }
        if (atomicCAS((unsigned int *)(need + 4 * lo), 0u, 1u) == 0u) {
            const unsigned long long slot = atomicAdd((unsigned long long *)n_heads, 1ull);
            heads[slot] = (uint32_t)lo;
        }
    }
}

// one CTA per out-of-order group: rank sort of (depth bits, index) in smem
constexpr int kFixMax = 2048;
__global__ void __launch_bounds__(256)
k_depth_fixup(const uint32_t *__restrict__ keys, uint32_t *__restrict__ src,
              unsigned long long *__restrict__ full, const int64_t *__restrict__ d_kept,
              const uint32_t *__restrict__ heads, const int64_t *__restrict__ n_heads) {
    __shared__ unsigned long long s_full[kFixMax];
    __shared__ uint32_t s_src[kFixMax];
    __shared__ int64_t s_end;
    const int64_t K = *d_kept, H = *n_heads;
    for (int64_t gi = blockIdx.x; gi < H; gi += gridDim.x) {
        const int64_t h = heads[gi];
        // group end = first index after h with another key: all threads test
        // 256 positions per round (groups are short: one round, instead of a
        // ~15-step serial binary search by one thread)
        const uint32_t kh = keys[h];
        if (threadIdx.x == 0) s_end = K;
        __syncthreads();
        for (int64_t base = h + 1; base < K; base += blockDim.x) {
            const int64_t i = base + threadIdx.x;
            if (i < K && keys[i] != kh) atomicMin((unsigned long long *)&s_end, (unsigned long long)i);
            __syncthreads();
            if (s_end < K || base + (int64_t)blockDim.x >= K) break;
            __syncthreads();
        }
        __syncthreads();
        const int64_t e = s_end, cnt = e - h;
        if (cnt <= kFixMax) {
            for (int64_t i = threadIdx.x; i < cnt; i += blockDim.x) {
                s_full[i] = full[h + i];
                s_src[i] = src[h + i];
            }
            __syncthreads();
            for (int64_t i = threadIdx.x; i < cnt; i += blockDim.x) {
                const unsigned long long d = s_full[i];
                const uint32_t x = s_src[i];
                int64_t r = 0;
                for (int64_t k = 0; k < cnt; ++k) {
                    const unsigned long long dk = s_full[k];
                    r += (dk < d) || (dk == d && s_src[k] < x);
                }
                src[h + r] = x;
                full[h + r] = d;
            }
        } else if (threadIdx.x == 0) {   // pathological huge group: serial insertion sort
            for (int64_t a = h + 1; a < e; ++a) {
                const uint32_t ia = src[a];
                const unsigned long long da = full[a];
                int64_t b = a - 1;
                while (b >= h && (full[b] > da || (full[b] == da && src[b] > ia))) {
                    src[b + 1] = src[b];
                    full[b + 1] = full[b];
                    --b;
                }
                src[b + 1] = ia;
                full[b + 1] = da;
            }
        }
        __syncthreads();
    }
}

// returns the rank -> point array (first *d_kept entries valid)
static uint32_t *depth_order(sfb_ctx *ctx, const RenderInputs &in, const Proj &P, DevCounts *C) {
    const int64_t n = in.n_points;
    uint32_t *k0 = ctx->arena.alloc<uint32_t>(n), *k1 = ctx->arena.alloc<uint32_t>(n);
    uint32_t *v0 = ctx->arena.alloc<uint32_t>(n), *v1 = ctx->arena.alloc<uint32_t>(n);
    k_depth_keys<<<dgrid(n, 256), 256, 0, ctx->stream>>>(n, in.point_to_geom, P, C->zr, k0, v0, &C->kept);
    SFB_CHECK_LAUNCH();
    // stable by point index within equal keys (devprims.cu radix sort)
    const bool second = dsort_pairs<uint32_t>(ctx, k0, v0, k1, v1, nullptr, n, 32);
    uint32_t *ks = second ? k1 : k0, *vs = second ? v1 : v0;
    auto *full = ctx->arena.alloc<unsigned long long>(n);
    uint8_t *need = ctx->arena.alloc<uint8_t>(4 * n);
    uint32_t *heads = ctx->arena.alloc<uint32_t>(n);
    SFB_CUDA(cudaMemsetAsync(need, 0, 4 * n, ctx->stream));
    const unsigned g = dgrid(n, 256);
    k_depth_full<<<g, 256, 0, ctx->stream>>>(vs, in.point_to_geom, P, &C->kept, full);
    k_depth_mark<<<g, 256, 0, ctx->stream>>>(ks, full, &C->kept, need, heads, &C->scratch[2]);
    k_depth_fixup<<<2 * 148, 256, 0, ctx->stream>>>(ks, vs, full, &C->kept, heads, &C->scratch[2]);
    SFB_CHECK_LAUNCH();
    return vs;
}

// ------------------------------------------------------------ 3. runs
// alpha-support radius of rasterizer.py:115-123 (gap uses square-then-scale)
__device__ __forceinline__ double support_radius(double a, double b, double c, double op) {
    double mid = 0.5 * (a + c);
    double amc = a - c;
    double gap = sqrt(fmax(0.25 * (amc * amc) + b * b, 0.0));
    double lam = fmax(mid + gap, 0.0);
    double sup = 2.0 * log(fmax(255.0 * op, 1e-300));
    return sqrt(fmax(sup, 0.0) * lam) + 1e-9;
}

struct TileRect {
    int32_t x0, x1, y0, y1;
};

__device__ __forceinline__ TileRect tile_rect(double sx, double sy, double r, double ft,
                                              int64_t ntx, int64_t nty) {
    // int(np.floor(v / tile)) clamped (_raster_kernels.py:123-130); clamp in
    // double first so non-finite extents cannot overflow the integer cast
    double lim = 4.0e9;
    double fx0 = fmin(fmax(floor((sx - r) / ft), -1.0), lim);
    double fx1 = fmin(fmax(floor((sx + r) / ft), -lim), (double)ntx);
    double fy0 = fmin(fmax(floor((sy - r) / ft), -1.0), lim);
    double fy1 = fmin(fmax(floor((sy + r) / ft), -lim), (double)nty);
    TileRect t;
    t.x0 = (int32_t)fmax(fx0, 0.0);
    t.x1 = (int32_t)fmin(fx1, (double)(ntx - 1));
    t.y0 = (int32_t)fmax(fy0, 0.0);
    t.y1 = (int32_t)fmin(fy1, (double)(nty - 1));
    return t;
}

__global__ void k_run_heads(const uint32_t *__restrict__ src, const int64_t *__restrict__ d_k,
                            const int32_t *__restrict__ p2g, Proj P, const double *__restrict__ opac,
                            int32_t *__restrict__ head) {
    const int64_t K = *d_k;
    SFB_FOR(j, K) {
        int h = 1;
        if (j > 0) {
            const uint32_t i = src[j], k = src[j - 1];
            if (p2g) {
                h = p2g[i] != p2g[k];
            } else {
                h = !(P.sx[i] == P.sx[k] && P.sy[i] == P.sy[k] && P.depth[i] == P.depth[k] &&
                      P.a[i] == P.a[k] && P.b[i] == P.b[k] && P.c[i] == P.c[k] && opac[i] == opac[k]);
            }
        }
        head[j] = h;
    }
}

// Alpha-support test of a whole tile. forward_kernel blends a splat at a
// pixel only if alpha = min(o exp(-q/2), alpha_max) >= 1/255, i.e. only if
// q <= 2 ln(255 o). q_cut widens that bound by a relative 1e-6 (+1e-6), far
// beyond the float64 rounding of q and of the exp, so skipping a run whose
// q exceeds q_cut at every pixel of a tile never drops a contribution.
__device__ __forceinline__ double q_cut(double op) {
    return 2.0 * log(fmax(255.0 * op, 1e-300)) * (1.0 + 1e-6) + 1e-6;
}

// What the compositor stages per candidate run, packed so a run costs a few
// 16-byte loads: geometry (conic, centre, opacity, support radius, depth)
// and the attribute side (first normal, point range, uniform-normal flag).
struct __align__(16) RunRec {
    double mx, my, ia, ib, ic, op, rad, dep;
};
struct __align__(16) RunAux {
    double rn[3];          // normal of the run's first point
    int32_t start, count;  // the run's points in rank order
    int32_t uni, pad;      // 1 when every point of the run has the same normal
    double qcut;           // q_cut(opacity): the run's alpha-support bound
};
static_assert(sizeof(RunAux) == 48 && offsetof(RunAux, start) == 24 && offsetof(RunAux, uni) == 32 &&
                  offsetof(RunAux, qcut) == 40,
              "the compositor stages RunAux as three double2 loads");

struct Runs {
    RunRec *rec;
    RunAux *aux;
    int32_t *start, *count;
    int4 *rect;
    uint8_t *level;  // 0 fine, 1 super, 2 global, 3 dead
    int32_t *nf, *ns, *ng;  // per-run entry counts
    const int64_t *d_R;
};

// geometry of run r from geometry row g: conic, support radius, tile rect
// and pyramid level (rasterizer.py:112-127)
__device__ __forceinline__ void run_geometry(Runs &R, int64_t r, int64_t g, const Proj &P,
                                             const double *__restrict__ opac, double ft, int64_t ntx,
                                             int64_t nty, double alpha_max) {
    const double a = P.a[g], b = P.b[g], c = P.c[g];
    const double op = opac[g];
    const double det = a * c - b * b;
    const double rad = support_radius(a, b, c, op);
    RunRec &q = R.rec[r];
    q.mx = P.sx[g];
    q.my = P.sy[g];
    q.ia = c / det;
    q.ib = -b / det;
    q.ic = a / det;
    q.op = op;
    q.rad = rad;
    const TileRect t = tile_rect(P.sx[g], P.sy[g], rad, ft, ntx, nty);
    R.rect[r] = make_int4(t.x0, t.x1, t.y0, t.y1);
    int lvl = 3, nf = 0, ns = 0, ng = 0;
    const bool live = !(op < kCutoff) && !(alpha_max < kCutoff) && t.x0 <= t.x1 && t.y0 <= t.y1;
    if (live) {
        const int64_t cnt = (int64_t)(t.x1 - t.x0 + 1) * (t.y1 - t.y0 + 1);
        if (cnt <= kFineMax) {
            lvl = 0;
            nf = (int)cnt;
        } else {
            const int64_t scnt =
                (int64_t)(t.x1 / kSuper - t.x0 / kSuper + 1) * (t.y1 / kSuper - t.y0 / kSuper + 1);
            if (scnt <= kSuperMax) {
                lvl = 1;
                ns = (int)scnt;
            } else {
                lvl = 2;
                ng = 1;
            }
        }
    }
    R.level[r] = (uint8_t)lvl;
    R.nf[r] = nf;
    R.ns[r] = ns;
    R.ng[r] = ng;
}

__global__ void k_run_build(const uint32_t *__restrict__ src, DevCounts *__restrict__ C,
                            const int32_t *__restrict__ incl, const int32_t *__restrict__ p2g, Proj P,
                            const double *__restrict__ opac, double ft, int64_t ntx, int64_t nty,
                            double alpha_max, Runs R) {
    const int64_t K = C->kept;
    SFB_FOR(j, K) {
        const int32_t r = incl[j] - 1;
        const bool last = j == K - 1 || incl[j + 1] != incl[j];
        if (last) R.count[r] = (int32_t)(j + 1);   // end of run r; start subtracted in k_emit
        if (j == K - 1) {
            C->runs = r + 1;
            C->runs1 = r + 2;
        }
        const bool head = j == 0 || incl[j - 1] != incl[j];
        if (!head) continue;
        R.start[r] = (int32_t)j;
        const uint32_t i = src[j];
        run_geometry(R, r, p2g ? p2g[i] : (int64_t)i, P, opac, ft, ntx, nty, alpha_max);
    }
}

// ------------------------------------------------------------ 2b. voxel-level order
// Fused frame: every point of a voxel shares the voxel's geometry, hence its
// depth, so the stable (depth, point index) order of the points is the depth
// order of the VOXELS with each voxel's points in index order (its CSR list),
// except inside groups of voxels whose depths are exactly equal, where the
// points of the group interleave by index (rasterizer.py:105). Sorting the
// M0 voxels instead of the N points replaces an 800k-key sort by a ~30k one,
// and runs come out per voxel (one run per voxel outside tie groups).
__global__ void k_vdepth_keys(const int64_t *__restrict__ d_ng, const Proj P,
                              const unsigned long long *__restrict__ zr, uint32_t *__restrict__ keys,
                              uint32_t *__restrict__ vals, int32_t *__restrict__ vpos,
                              int64_t *__restrict__ d_kept_geom) {
    const int64_t ng = *d_ng;
    const double zmin = __longlong_as_double((long long)~zr[0]);
    const double zmax = __longlong_as_double((long long)zr[1]);
    // 24-bit monotone quantisation (3 radix passes over ~30k voxels; exact
    // order restored inside equal-key groups by the fix-up), culled last
    const double scale = zmax > zmin ? 16777214.0 / (zmax - zmin) : 0.0;
    SFB_FOR(g, ((ng + 31) & ~int64_t(31))) {
        bool k = false;
        if (g < ng) {
            k = P.keep[g];
            keys[g] = k ? (uint32_t)fmin(floor((P.depth[g] - zmin) * scale), 16777214.0) : 0xffffffu;
            vals[g] = (uint32_t)g;
            vpos[g] = -1;
        }
        const unsigned ball = __ballot_sync(0xffffffffu, k);
        if ((threadIdx.x & 31) == 0 && ball) atomicAdd((unsigned long long *)d_kept_geom, (unsigned long long)__popc(ball));
    }
}

// per sorted kept voxel: its point count and its sorted position
__global__ void k_vcounts(const uint32_t *__restrict__ vs, const int64_t *__restrict__ d_kg,
                          const int32_t *__restrict__ goff, int32_t *__restrict__ cnt,
                          int32_t *__restrict__ vpos) {
    const int64_t KG = *d_kg;
    SFB_FOR(i, KG) {
        const uint32_t v = vs[i];
        cnt[i] = goff[v + 1] - goff[v];
        vpos[v] = (int32_t)i;
    }
}

// [gs, ge) = the group of sorted voxels with depth bits equal to full[i]
__device__ __forceinline__ bool tie_group(const unsigned long long *__restrict__ full, int64_t i,
                                          int64_t KG, int64_t &gs, int64_t &ge) {
    const unsigned long long d = full[i];
    gs = i;
    while (gs > 0 && full[gs - 1] == d) --gs;
    ge = i + 1;
    while (ge < KG && full[ge] == d) ++ge;
    return ge - gs > 1;
}

// number of points of a sorted index list below p
__device__ __forceinline__ int32_t count_below(const int32_t *__restrict__ lst, int32_t n, int32_t p) {
    int32_t lo = 0, hi = n;
    while (lo < hi) {
        const int32_t mid = (lo + hi) >> 1;
        if (lst[mid] < p) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

// CSR slot -> rank: src[rank] = point, colours gathered in rank order.
// thead[rank] = 1 where a tie group's merged order switches voxel (its first
// rank included): the predecessor of p in the group is the largest group
// point index below p, found with the same per-voxel binary searches. Also
// records every sorted voxel's group bounds (gspan) for the run builders.
template <int G>   // lanes per voxel (32: one warp; 8 / 16: several voxels per warp)
__global__ void k_vranks(const int32_t *__restrict__ order, const int32_t *__restrict__ goff,
                         const int32_t *__restrict__ off, const unsigned long long *__restrict__ full,
                         const uint32_t *__restrict__ vs, const int64_t *__restrict__ d_kg,
                         const double *__restrict__ colors, float4 *__restrict__ scol,
                         uint32_t *__restrict__ src, int32_t *__restrict__ thead,
                         int2 *__restrict__ gspan) {
    // one warp per sorted kept voxel, lanes over its points (CSR slots):
    // the voxel's offsets are loaded once, the point reads / rank writes
    // are coalesced, only the colour gather is random
    const int64_t KG = *d_kg;
    const int lane = threadIdx.x % G;
    const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / G;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) / G;
    for (int64_t i = w0; i < KG; i += nw) {
        const uint32_t v = vs[i];
        const int32_t s0 = goff[v], s1 = goff[v + 1];
        int64_t gs, ge;
        const bool tie = tie_group(full, i, KG, gs, ge);
        if (lane == 0) gspan[i] = make_int2((int32_t)gs, (int32_t)ge);
        const int64_t base = tie ? (int64_t)off[gs] : (int64_t)off[i];
        for (int32_t s = s0 + lane; s < s1; s += G) {
            const int32_t p = order[s];
            const int32_t w = s - s0;
            int64_t rank = base + w;
            int32_t h = 0;
            if (tie) {
                int32_t own = w > 0 ? order[s - 1] : -1, other = -1;   // predecessors of p
                for (int64_t u = gs; u < ge; ++u) {
                    const uint32_t vu = vs[u];
                    if (vu == v) continue;
                    const int32_t *lst = order + goff[vu];
                    const int32_t cb = count_below(lst, goff[vu + 1] - goff[vu], p);
                    rank += cb;
                    if (cb > 0) other = max(other, lst[cb - 1]);
                }
                h = other > own || (own < 0 && other < 0);
            }
            src[rank] = (uint32_t)p;
            thead[rank] = h;
            if (scol)
                scol[rank] = make_float4((float)colors[3 * (size_t)p], (float)colors[3 * (size_t)p + 1],
                                         (float)colors[3 * (size_t)p + 2], 0.f);
        }
    }
}

// Runs per sorted voxel: 1 outside tie groups; the first voxel of a tie
// group holds the group's block count (inclusive scan of thead over ranks).
__global__ void k_vblocks(const int2 *__restrict__ gspan, const int64_t *__restrict__ d_kg,
                          const int32_t *__restrict__ off, const int32_t *__restrict__ cnt,
                          const int32_t *__restrict__ hincl, int32_t *__restrict__ nblk) {
    const int64_t KG = *d_kg;
    SFB_FOR(i, KG) {
        const int2 sp = gspan[i];
        const int64_t gs = sp.x, ge = sp.y;
        int32_t b = 1;
        if (ge - gs > 1) {
            b = 0;
            if (gs == i) {
                const int64_t j0 = off[gs], j1 = off[ge - 1] + cnt[ge - 1];
                b = hincl[j1 - 1] - (j0 > 0 ? hincl[j0 - 1] : 0);
            }
        }
        nblk[i] = b;
    }
}

// Run records. x < KG: one run per non-tie sorted voxel; x < K: a tie-group
// head rank starts run ro[group] + (heads of the group before it), ending at
// the next head or the group end.
__global__ void k_vbuild(const uint32_t *__restrict__ vs, const int2 *__restrict__ gspan,
                         DevCounts *__restrict__ C, const int64_t *__restrict__ d_kg,
                         const int32_t *__restrict__ off, const int32_t *__restrict__ cnt,
                         const int32_t *__restrict__ ro, const int32_t *__restrict__ vpos,
                         const int32_t *__restrict__ thead, const int32_t *__restrict__ hincl,
                         const uint32_t *__restrict__ src, const int32_t *__restrict__ p2g, Proj P,
                         const double *__restrict__ opac, double ft, int64_t ntx, int64_t nty,
                         double alpha_max, Runs R) {
    const int64_t KG = *d_kg, K = C->kept;
    if (blockIdx.x == 0 && threadIdx.x == 0) C->runs1 = C->runs + 1;
    SFB_FOR(x, max(KG, K)) {
        if (x < KG && gspan[x].y - gspan[x].x == 1) {
            const int64_t r = ro[x];
            R.start[r] = off[x];
            R.count[r] = off[x] + cnt[x];   // run end; k_emit subtracts the start
            run_geometry(R, r, vs[x], P, opac, ft, ntx, nty, alpha_max);
        }
        if (x < K && thead[x]) {
            const int32_t g = p2g[src[x]];
            const int2 sp = gspan[vpos[g]];
            const int64_t gs = sp.x, ge = sp.y;
            const int64_t j0 = off[gs], j1 = off[ge - 1] + cnt[ge - 1];
            const int64_t r = ro[gs] + (hincl[x] - (j0 > 0 ? hincl[j0 - 1] : 0)) - 1;
            int64_t e = x + 1;
            while (e < j1 && !thead[e]) ++e;
            R.start[r] = (int32_t)x;
            R.count[r] = (int32_t)e;
            run_geometry(R, r, g, P, opac, ft, ntx, nty, alpha_max);
        }
    }
}

// Pyramid capacity check: the fine / super entry buffers hold `cap` entries
// (sized from the previous eager frame, not from the point count). When a
// frame's runs ask for more, every run goes to the global list instead (all
// runs in rank order; dead runs get an empty rect) — slower compositing for
// that frame, identical planes.
__global__ void k_entry_guard(DevCounts *__restrict__ C, int64_t cap) {
    C->ef_req = C->ef;
    C->es_req = C->es;
    if (C->ef > cap || C->es > cap) {
        C->overflow = 1;
        C->ef = C->es = 0;
        C->g = C->runs;
    }
}

__global__ void k_emit(Runs R, const int32_t *__restrict__ fpos, const int32_t *__restrict__ spos,
                       const int32_t *__restrict__ gpos, int64_t ntx, int64_t nsx,
                       uint32_t *__restrict__ fkey, uint32_t *__restrict__ fval,
                       uint32_t *__restrict__ skey, uint32_t *__restrict__ sval,
                       uint32_t *__restrict__ glist, int4 *__restrict__ grect,
                       const DevCounts *__restrict__ C) {
    const int64_t nr = *R.d_R;
    const bool all_global = C->overflow != 0;
    SFB_FOR(r, nr) {
        R.count[r] -= R.start[r];   // k_run_build stored the run's end
        const int lvl = R.level[r];
        const int4 t = R.rect[r];
        if (all_global) {
            glist[r] = (uint32_t)r;
            grect[r] = lvl == 3 ? make_int4(1, 0, 1, 0) : t;
        } else if (lvl == 0) {
            int32_t p = fpos[r];
            for (int y = t.z; y <= t.w; ++y)
                for (int x = t.x; x <= t.y; ++x) {
                    fkey[p] = (uint32_t)(y * ntx + x);
                    fval[p++] = (uint32_t)r;
                }
        } else if (lvl == 1) {
            int32_t p = spos[r];
            for (int y = t.z / kSuper; y <= t.w / kSuper; ++y)
                for (int x = t.x / kSuper; x <= t.y / kSuper; ++x) {
                    skey[p] = (uint32_t)(y * nsx + x);
                    sval[p++] = (uint32_t)r;
                }
        } else if (lvl == 2) {
            glist[gpos[r]] = (uint32_t)r;
            grect[gpos[r]] = t;
        }
    }
}

// once per frame, per run: its depth, its first point's normal and whether
// the normal is uniform over the run (always, for per-voxel geometry)
__global__ void k_stage_runs(Runs R, const uint32_t *__restrict__ src, const int32_t *__restrict__ p2g,
                             const double *__restrict__ normals, const double *__restrict__ gdepth,
                             int want_n) {
    const int64_t nr = *R.d_R;
    SFB_FOR(r, nr) {
        const uint32_t i0 = src[R.start[r]];
        const int64_t g0 = p2g ? p2g[i0] : (int64_t)i0;
        R.rec[r].dep = gdepth[g0];
        RunAux &x = R.aux[r];
        x.qcut = q_cut(R.rec[r].op);
        x.start = R.start[r];
        x.count = R.count[r];
        x.pad = 0;
        uint8_t u = 1;
        if (want_n) {
            for (int c = 0; c < 3; ++c) x.rn[c] = normals[3 * g0 + c];
            if (!p2g)   // generic splats: compare every point's normal
                for (int32_t j = R.start[r] + 1; j < R.start[r] + R.count[r] && u; ++j) {
                    const uint32_t i = src[j];
                    u = normals[3 * (size_t)i] == normals[3 * (size_t)i0] &&
                        normals[3 * (size_t)i + 1] == normals[3 * (size_t)i0 + 1] &&
                        normals[3 * (size_t)i + 2] == normals[3 * (size_t)i0 + 2];
                }
        }
        x.uni = u;
    }
}

// per-point attributes in rank order as float4 (one 16-byte load per point in
// the compositor); normals only for per-point geometry (runs may mix them)
__global__ void k_gather_attrs(const uint32_t *__restrict__ src, const int32_t *__restrict__ p2g,
                               const double *__restrict__ colors, const double *__restrict__ normals,
                               const int64_t *__restrict__ d_k, float4 *__restrict__ scol,
                               float4 *__restrict__ snrm) {
    const int64_t K = *d_k;
    SFB_FOR(j, K) {
        const size_t i = src[j];
        if (scol)
            scol[j] = make_float4((float)colors[3 * i], (float)colors[3 * i + 1], (float)colors[3 * i + 2], 0.f);
        if (snrm && !p2g)
            snrm[j] = make_float4((float)normals[3 * i], (float)normals[3 * i + 1], (float)normals[3 * i + 2], 0.f);
    }
}

// tile rects of a sorted list's entries, in list order (the compositor then
// loads an entry's id and rect side by side instead of rect[id])
__global__ void k_list_rects(const uint32_t *__restrict__ ids, const int64_t *__restrict__ d_n,
                             const int4 *__restrict__ rect, int4 *__restrict__ out) {
    const int64_t n = *d_n;
    SFB_FOR(i, n) out[i] = rect[ids[i]];
}

__global__ void k_tile_index(const uint32_t *__restrict__ fk, const int64_t *__restrict__ d_ef,
                             const uint32_t *__restrict__ sk, const int64_t *__restrict__ d_es,
                             const uint32_t *__restrict__ s_ids, const int4 *__restrict__ rect, int64_t nt,
                             int64_t ns, int32_t *__restrict__ f_off, int32_t *__restrict__ s_off,
                             int4 *__restrict__ srect) {
    const int64_t ef = *d_ef, es = *d_es;
    auto lower = [](const uint32_t *k, int64_t n, uint32_t v) {
        int64_t lo = 0, hi = n;
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if (k[mid] < v) lo = mid + 1;
            else hi = mid;
        }
        return (int32_t)lo;
    };
    SFB_FOR(x, max(es, nt + ns + 2)) {
        if (x < es) srect[x] = rect[s_ids[x]];
        if (x <= nt) f_off[x] = lower(fk, ef, (uint32_t)x);
        else if (x <= nt + ns + 1) s_off[x - nt - 1] = lower(sk, es, (uint32_t)(x - nt - 1));
    }
}

__global__ void k_histogram(const uint32_t *__restrict__ keys, const int64_t *__restrict__ d_n,
                            int32_t *__restrict__ cnt) {
    const int64_t n = *d_n;
    SFB_FOR(j, n) atomicAdd(&cnt[keys[j]], 1);
}

// ------------------------------------------------------------ 5. compositor
struct CompParams {
    int64_t W, H, ntx, nty, nsx;
    int tile;
    int terminate;
    double alpha_max;
    int plane_mask;
    const FrameParams *fp;
    // lists
    const int32_t *f_off;
    const uint32_t *f_ids;
    const int32_t *s_off;
    const uint32_t *s_ids;
    const uint32_t *g_ids;
    const int4 *s_rect, *g_rect;   // tile rects of the super / global entries, in list order
    const int64_t *d_G;
    Runs R;
    // per-point attributes in rank order (float4: x, y, z, pad)
    const float4 *scol;   // colours (rgb plane)
    const float4 *snrm;   // normals of per-point geometry (runs with mixed normals)
    // outputs
    float *rgb, *normal, *depth, *trans;
    uint8_t *rgba;   // render_pose RGBA8 (FrameParams shading), or null
    int64_t *dbg;   // optional per-tile counters: windows, list entries, alpha evals, point blends
};

// exp(x) for x <= 0 in float64 (the compositor's alpha = o * exp(-q/2)):
// x = k ln2 + r, |r| <= ln2/2, with ln2 split hi/lo (Cody-Waite), exp(r) by
// a degree-12 Taylor polynomial in FMA Horner form (truncation < 2^-60), then
// scaled by 2^k through the exponent bits. Within ~1 ulp like the libm exp
// (the reference's numba kernel uses LLVM's), at ~25 instructions instead of
// the ~50 of the general-purpose CUDA exp with its special-case paths.
// Branch-free (the compositor evaluates it for both of a thread's pixels in
// one straight-line block): x is clamped to [-708, 0] (x > 0 only through
// rounding of a degenerate conic, where the result is 1 to within rounding)
// and 0 is selected below -708 (alpha < 1/255 there anyway).
__device__ __forceinline__ double exp_nonpos(double x) {
    const bool under = x < -708.0;
    x = fmin(fmax(x, -708.0), 0.0);
    const double kd = rint(x * 1.4426950408889634);
    const double r = __fma_rn(-kd, 6.93147180369123816490e-01, x);
    const double rr = __fma_rn(-kd, 1.90821492927058770002e-10, r);
    double p = 2.08767569878680989792e-09;            // 1/12!
    p = __fma_rn(p, rr, 2.50521083854417187751e-08);  // 1/11!
    p = __fma_rn(p, rr, 2.75573192239858906526e-07);  // 1/10!
    p = __fma_rn(p, rr, 2.75573192239858906526e-06);  // 1/9!
    p = __fma_rn(p, rr, 2.48015873015873015873e-05);  // 1/8!
    p = __fma_rn(p, rr, 1.98412698412698412698e-04);  // 1/7!
    p = __fma_rn(p, rr, 1.38888888888888888889e-03);  // 1/6!
    p = __fma_rn(p, rr, 8.33333333333333333333e-03);  // 1/5!
    p = __fma_rn(p, rr, 4.16666666666666666667e-02);  // 1/4!
    p = __fma_rn(p, rr, 1.66666666666666666667e-01);  // 1/3!
    p = __fma_rn(p, rr, 0.5);
    p = __fma_rn(p, rr, 1.0);
    p = __fma_rn(p, rr, 1.0);
    const int k = (int)kd;   // in [-1022, 0]: 2^k is a normal double
    return under ? 0.0 : p * __longlong_as_double((long long)(k + 1023) << 52);
}


// min over the rectangle [x0,x1] x [y0,y1] (offsets from the centre) of the
// positive-definite form q(d) = ia dx^2 + 2 ib dx dy + ic dy^2: 0 when the
// centre is inside, else the least of the four edge minima (a 1-D quadratic
// per edge, minimised at its clamped stationary point). Returns 0 (no cull)
// for a degenerate conic. The stationary point is fixed * slope with the
// slope -b/c divided once per pair of parallel edges (its rounding moves the
// evaluated point by ~1e-16 relative: q changes quadratically, far inside
// q_cut's 1e-6 margin).
__device__ __forceinline__ double edge_min(double a, double b, double c, double slope, double fixed,
                                           double lo, double hi) {
    // q(t) = a fixed^2 + 2 b fixed t + c t^2 over t in [lo, hi]
    const double t = fmin(fmax(slope * fixed, lo), hi);
    return a * fixed * fixed + 2.0 * b * fixed * t + c * t * t;
}
__device__ __forceinline__ double tile_min_q(double ia, double ib, double ic, double x0, double x1,
                                             double y0, double y1) {
    if (!(ia > 0.0) || !(ic > 0.0) || !(ia * ic - ib * ib > 0.0)) return 0.0;
    if (x0 <= 0.0 && 0.0 <= x1 && y0 <= 0.0 && 0.0 <= y1) return 0.0;
    const double sx = -ib / ic, sy = -ib / ia;
    double m = edge_min(ia, ib, ic, sx, x0, y0, y1);
    m = fmin(m, edge_min(ia, ib, ic, sx, x1, y0, y1));
    m = fmin(m, edge_min(ic, ib, ia, sy, y0, x0, x1));
    m = fmin(m, edge_min(ic, ib, ia, sy, y1, x0, x1));
    return m;
}

// sum_{j<m} om^j v_j (float32; v in rank order). Two interleaved Horner
// chains in om^2 (even and odd points), S = E + om * O, so two independent
// chains and four 16-byte loads are in flight per step; the (x, y) channels
// go through one paired FFMA2 (sm_100), z through an FFMA.
__device__ __forceinline__ void hstep(float2 &xy, float &z, float2 om2v, float om2, float4 a) {
    xy = __ffma2_rn(xy, om2v, make_float2(a.x, a.y));
    z = fmaf(z, om2, a.z);
}
__device__ __forceinline__ float3 horner3(const float4 *__restrict__ v, int m, float om) {
    const float om2 = om * om;
    const float2 om2v = make_float2(om2, om2);
    float2 exy = make_float2(0.f, 0.f), oxy = make_float2(0.f, 0.f);
    float ez = 0.f, oz = 0.f;
    int j = m - 1;
    if (!(m & 1) && j >= 0) {   // make the last point an even one
        const float4 a = __ldg(v + j);
        oxy = make_float2(a.x, a.y);
        oz = a.z;
        --j;
    }
    // j is even here: pairs (j-1 odd, j even) ... down to (-, 0)
    for (; j >= 4; j -= 4) {
        const float4 a = __ldg(v + j), b = __ldg(v + j - 1), c = __ldg(v + j - 2), d = __ldg(v + j - 3);
        hstep(exy, ez, om2v, om2, a);
        hstep(oxy, oz, om2v, om2, b);
        hstep(exy, ez, om2v, om2, c);
        hstep(oxy, oz, om2v, om2, d);
    }
    for (; j >= 2; j -= 2) {
        const float4 a = __ldg(v + j), b = __ldg(v + j - 1);
        hstep(exy, ez, om2v, om2, a);
        hstep(oxy, oz, om2v, om2, b);
    }
    if (j == 0) hstep(exy, ez, om2v, om2, __ldg(v));
    return make_float3(fmaf(om, oxy.x, exy.x), fmaf(om, oxy.y, exy.y), fmaf(om, oz, ez));
}

// Colour / normal accumulators of the compositor (T, the depth sums and every
// alpha / cutoff decision stay float64)
using CompAcc = float;
__device__ __forceinline__ double acc_fma(double w, double v, double c) { return __fma_rn(w, v, c); }
__device__ __forceinline__ float acc_fma(double w, double v, float c) {
    return __fmaf_rn((float)w, (float)v, c);
}

// The same sums for two pixels that blend the same m points of a run (the
// usual case: a thread's two pixels share the tile's runs): one load of each
// point feeds both pixels, one Horner chain per pixel ((x, y) paired FFMA2s,
// the two pixels' z in a third).
__device__ __forceinline__ void horner3x2(const float4 *__restrict__ v, int m, float om0, float om1,
                                          float3 &S0, float3 &S1) {
    const float2 o0 = make_float2(om0, om0), o1 = make_float2(om1, om1), oz = make_float2(om0, om1);
    float2 xy0 = make_float2(0.f, 0.f), xy1 = make_float2(0.f, 0.f), z = make_float2(0.f, 0.f);
    auto step = [&](const float4 a) {
        const float2 axy = make_float2(a.x, a.y);
        xy0 = __ffma2_rn(xy0, o0, axy);
        xy1 = __ffma2_rn(xy1, o1, axy);
        z = __ffma2_rn(z, oz, make_float2(a.z, a.z));
    };
    int j = m - 1;
    for (; j >= 3; j -= 4) {
        const float4 a = __ldg(v + j), b = __ldg(v + j - 1), c = __ldg(v + j - 2), d = __ldg(v + j - 3);
        step(a);
        step(b);
        step(c);
        step(d);
    }
    for (; j >= 0; --j) step(__ldg(v + j));
    S0 = make_float3(xy0.x, xy0.y, z.x);
    S1 = make_float3(xy1.x, xy1.y, z.y);
}

// One CTA per tile. The rank-ordered fine / super / global lists are merged
// in rank windows (bitmap + ordered compaction), candidate runs are staged
// in chunks, and every pixel blends each covering run in closed form: a
// run's points share alpha, so before point j of the run T = T0 (1-a)^j and
//   sum_j T_j a c_j = T0 a sum_{j<m} (1-a)^j c_j       (Horner, float32)
//   sum_j T_j a     = T0 - T_m                         (normal / depth of
//                                                       uniform runs)
// where m = points blended before T < 1/255 (forward_kernel's per-point
// check, _raster_kernels.py:185-187). m = run length unless T crosses the
// cutoff inside the run; then T is iterated point by point exactly as the
// reference does. Alpha, T and the thresholds stay float64.
// MASK: the planes accumulated (SFB_PLANE_*), a compile-time constant so
// unused accumulators and branches disappear from the hot loop
template <int NPIX, int MASK>
__global__ void __launch_bounds__(kCT, kCompMinBlocks) k_composite(CompParams P) {
    constexpr uint32_t NONE = 0xffffffffu;
    __shared__ uint32_t bitmap[kWin / 32];
    __shared__ uint32_t list[kWin];
    __shared__ uint32_t s_add[3];
    __shared__ uint32_t s_head;
    __shared__ unsigned s_bal[kCT / 32];
    __shared__ uint8_t r_idx[kChunk];   // staged slot of the chunk's e-th surviving run
    // the current chunk's run records (pixel box precomputed per run)
    __shared__ double r_mx[kChunk], r_my[kChunk], r_rr[kChunk], r_ia[kChunk], r_ib[kChunk],
        r_ic[kChunk], r_op[kChunk], r_dep[kChunk], r_rn[3][kChunk];
    __shared__ int32_t r_x0[kChunk], r_x1[kChunk], r_y0[kChunk], r_y1[kChunk], r_start[kChunk],
        r_count[kChunk];
    __shared__ uint8_t r_uni[kChunk];
    __shared__ uint8_t r_full[kChunk];   // run's pixel box and circle cover the whole tile

    const int64_t t = blockIdx.x;
    const uint32_t ntx32 = (uint32_t)P.ntx;   // 32-bit division: the grid is < 2^31 tiles
    const int32_t tx = (int32_t)(blockIdx.x % ntx32), ty = (int32_t)(blockIdx.x / ntx32);
    const int32_t st = (ty / kSuper) * (int32_t)P.nsx + tx / kSuper;
    const int TS = P.tile;
    // pixel coordinates fit 32 bits (images are < 2^31 pixels wide and high)
    const int32_t x_lo = tx * TS, y_lo = ty * TS;
    const int32_t x_end = (int32_t)min((int64_t)x_lo + TS, P.W), y_end = (int32_t)min((int64_t)y_lo + TS, P.H);
    constexpr bool want_rgb = MASK & SFB_PLANE_RGB, want_n = MASK & SFB_PLANE_NORMAL;
    constexpr bool want_d = MASK & SFB_PLANE_DEPTH;
    const bool term = P.terminate;

    int32_t pxs[NPIX], pys[NPIX];
    bool valid[NPIX];
    double T[NPIX];
    CompAcc c0[NPIX], c1[NPIX], c2[NPIX], n0[NPIX], n1[NPIX], n2[NPIX];
    double dd[NPIX];   // depth keeps float64 sums: its values are O(scene depth), not O(1)
#pragma unroll
    for (int k = 0; k < NPIX; ++k) {
        const uint32_t p = threadIdx.x + k * kCT;
        pxs[k] = (int32_t)(x_lo + p % (uint32_t)TS);
        pys[k] = (int32_t)(y_lo + p / (uint32_t)TS);
        valid[k] = p < TS * TS && pxs[k] < x_end && pys[k] < y_end;
        T[k] = 1.0;
        c0[k] = c1[k] = c2[k] = n0[k] = n1[k] = n2[k] = dd[k] = 0.0;
    }
    auto saturated = [&]() {
        int mine = 1;
#pragma unroll
        for (int k = 0; k < NPIX; ++k)
            if (valid[k] && !(T[k] < kCutoff)) mine = 0;
        return mine;
    };

    const double2 *__restrict__ Rrec = reinterpret_cast<const double2 *>(P.R.rec);
    const double2 *__restrict__ Raux = reinterpret_cast<const double2 *>(P.R.aux);
    const float4 *__restrict__ scol = P.scol, *__restrict__ snrm = P.snrm;
    const double alpha_max = P.alpha_max;
    const uint32_t *ids[3] = {P.f_ids, P.s_ids, P.g_ids};
    // list positions as 32-bit (the entry lists are int32-indexed)
    // list cursors and ends are CTA-uniform: kept in shared memory (registers
    // go to the per-pixel state)
    __shared__ int32_t cur[3], end[3];
    if (threadIdx.x < 3) {
        const int s = threadIdx.x;
        cur[s] = s == 0 ? P.f_off[t] : s == 1 ? P.s_off[st] : 0;
        end[s] = s == 0 ? P.f_off[t + 1] : s == 1 ? P.s_off[st + 1] : (int32_t)*P.d_G;
    }
    __syncthreads();
    __shared__ int s_ws;   // rank window size: 128 -> kWin (most tiles saturate in the first)
    if (threadIdx.x == 0) s_ws = 128;
    bool done = false;
    while (!done) {
        // the window's first 256-rank slice (ids and, in list order, rects)
        // is loaded before the window is known: thread 0's ids are the list
        // heads, so the window start costs no extra dependent round trip
        uint32_t id[3];
        int4 rc[2];
#pragma unroll
        for (int s = 0; s < 3; ++s) {
            const int32_t idx = cur[s] + (int32_t)threadIdx.x;
            id[s] = idx < end[s] ? ids[s][idx] : NONE;
            if (s) rc[s - 1] = idx < end[s] ? (s == 1 ? P.s_rect : P.g_rect)[idx] : make_int4(1, 0, 1, 0);
        }
        if (threadIdx.x == 0) s_head = min(id[0], min(id[1], id[2]));
        for (int i = threadIdx.x; i < kWin / 32; i += kCT) bitmap[i] = 0;
        if (threadIdx.x < 3) s_add[threadIdx.x] = 0;
        __syncthreads();
        const uint32_t w0 = s_head;
        if (w0 == NONE) break;
        const int ws = s_ws;   // written again only after the compaction's barrier
        const uint32_t w1 = w0 + (uint32_t)ws;
        // one 256-rank slice of the window at a time: 3 id loads + 2 rect
        // loads in flight per thread, few registers (occupancy)
        for (int k = 0; k * kCT < ws; ++k) {
            if (k) {
#pragma unroll
                for (int s = 0; s < 3; ++s) {
                    const int32_t idx = cur[s] + k * kCT + (int32_t)threadIdx.x;
                    id[s] = idx < end[s] ? ids[s][idx] : NONE;
                }
#pragma unroll
                for (int s = 1; s < 3; ++s) {   // rects stored in list order: no dependent load
                    const int32_t idx = cur[s] + k * kCT + (int32_t)threadIdx.x;
                    rc[s - 1] = idx < end[s] ? (s == 1 ? P.s_rect : P.g_rect)[idx] : make_int4(1, 0, 1, 0);
                }
            }
#pragma unroll
            for (int s = 0; s < 3; ++s) {
                const uint32_t r = id[s];
                const bool in = r < w1;
                bool cover = in;
                if (s && in) {
                    const int4 q = rc[s - 1];
                    cover = tx >= q.x && tx <= q.y && ty >= q.z && ty <= q.w;
                }
                if (cover) atomicOr(&bitmap[(r - w0) >> 5], 1u << ((r - w0) & 31));
                const unsigned ball = __ballot_sync(0xffffffffu, in);
                if ((threadIdx.x & 31) == 0 && ball) atomicAdd(&s_add[s], (uint32_t)__popc(ball));
            }
        }
        __syncthreads();
        // read again only after the compaction's barrier
        if (threadIdx.x < 3) cur[threadIdx.x] += (int32_t)s_add[threadIdx.x];
        // ordered compaction of the bitmap by all threads: every warp forms
        // the words' prefix counts (2 words per lane, shuffle scan), then
        // each thread places the set bits among its rank positions
        // p = tid + kCT k (a warp's 32 positions are one word)
        int nlist;
        {
            const int lane = threadIdx.x & 31;
            const int nw = ws / 32;
            const uint32_t wa = 2 * lane < nw ? bitmap[2 * lane] : 0u;
            const uint32_t wb = 2 * lane + 1 < nw ? bitmap[2 * lane + 1] : 0u;
            const int ca = __popc(wa), cb = __popc(wb);
            int incl = ca + cb;
            for (int o = 1; o < 32; o <<= 1) {
                const int v = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += v;
            }
            const int pre = incl - ca - cb;   // set bits before word 2 * lane
            nlist = __shfl_sync(0xffffffffu, incl, 31);
            for (int p0 = threadIdx.x & ~31; p0 < ws; p0 += kCT) {
                const int wi = p0 >> 5;   // warp-uniform
                const int base = __shfl_sync(0xffffffffu, pre, wi >> 1) +
                                 ((wi & 1) ? __shfl_sync(0xffffffffu, ca, wi >> 1) : 0);
                const uint32_t word = (wi & 1) ? __shfl_sync(0xffffffffu, wb, wi >> 1)
                                               : __shfl_sync(0xffffffffu, wa, wi >> 1);
                if ((word >> lane) & 1u) list[base + __popc(word & ((1u << lane) - 1u))] = w0 + p0 + lane;
            }
        }
        __syncthreads();
        // chunks of candidate runs grow 16 -> kChunk: most tiles saturate within
        // the first few contributing runs. Each candidate is staged by one
        // thread, which also drops it when its alpha-support ellipse misses the
        // tile's pixels (tile_min_q): such a run has alpha < 1/255 at every
        // pixel of the tile, so forward_kernel's per-pixel test skips it
        // everywhere (_raster_kernels.py:193-194). Survivors are compacted in
        // rank order.
        int chunk = 16;
        for (int base = 0; base < nlist && !done; base += chunk, chunk = min(2 * chunk, kChunk)) {
            const int nc = min(chunk, nlist - base);
            bool keep = false;
            if (threadIdx.x < nc) {
                const uint32_t r = list[base + threadIdx.x];
                const int j = threadIdx.x;
                const double2 q0 = Rrec[4 * (size_t)r], q1 = Rrec[4 * (size_t)r + 1],
                              q2 = Rrec[4 * (size_t)r + 2], q3 = Rrec[4 * (size_t)r + 3];
                const double2 a0 = Raux[3 * (size_t)r], a1 = Raux[3 * (size_t)r + 1],
                              a2 = Raux[3 * (size_t)r + 2];
                const double mx = q0.x, my = q0.y;
                const double rad = q3.x + 1.0;
                r_mx[j] = mx;
                r_my[j] = my;
                r_rr[j] = rad * rad;
                r_ia[j] = q1.x;
                r_ib[j] = q1.y;
                r_ic[j] = q2.x;
                r_op[j] = q2.y;
                r_dep[j] = q3.y;
                // RunAux as double2: {rn0, rn1}, {rn2, (start, count)}, {(uni, pad), qcut}
                r_start[j] = __double2loint(a1.y);
                r_count[j] = __double2hiint(a1.y);
                r_uni[j] = (uint8_t)__double2loint(a2.x);
                if (want_n) {
                    r_rn[0][j] = a0.x;
                    r_rn[1][j] = a0.y;
                    r_rn[2][j] = a1.x;
                }
                // pixel box of forward_kernel (_raster_kernels.py:178-181), clamped to the tile
                const int32_t bx0 = (int32_t)fmin(fmax((double)x_lo, ceil(mx - rad)), (double)x_end);
                const int32_t bx1 = (int32_t)fmax(fmin((double)(x_end - 1), floor(mx + rad)), (double)(x_lo - 1));
                const int32_t by0 = (int32_t)fmin(fmax((double)y_lo, ceil(my - rad)), (double)y_end);
                const int32_t by1 = (int32_t)fmax(fmin((double)(y_end - 1), floor(my + rad)), (double)(y_lo - 1));
                r_x0[j] = bx0;
                r_x1[j] = bx1;
                r_y0[j] = by0;
                r_y1[j] = by1;
                // whole tile inside the box and the circle (farthest corner
                // within the radius): the per-pixel tests are then all true
                const double fx = fmax(fabs((double)x_lo - mx), fabs((double)(x_end - 1) - mx));
                const double fy = fmax(fabs((double)y_lo - my), fabs((double)(y_end - 1) - my));
                r_full[j] = bx0 == x_lo && bx1 == x_end - 1 && by0 == y_lo && by1 == y_end - 1 &&
                            fx * fx + fy * fy <= rad * rad;
                keep = bx0 <= bx1 && by0 <= by1 &&
                       !(tile_min_q(q1.x, q1.y, q2.x, bx0 - mx, bx1 - mx, by0 - my, by1 - my) >
                         a2.y);   // q_cut(opacity), precomputed per run
            }
            const unsigned ball = __ballot_sync(0xffffffffu, keep);
            if ((threadIdx.x & 31) == 0) s_bal[threadIdx.x >> 5] = ball;
            __syncthreads();
            int slot = __popc(ball & ((1u << (threadIdx.x & 31)) - 1u)), nb = 0;
#pragma unroll
            for (int w = 0; w < kCT / 32; ++w) {
                const int c = __popc(s_bal[w]);
                slot += w < (int)(threadIdx.x >> 5) ? c : 0;
                nb += c;
            }
            if (keep) r_idx[slot] = (uint8_t)threadIdx.x;   // survivors in rank order
            __syncthreads();
            for (int e = 0; e < nb; ++e) {
                if (term && e && (e & 31) == 0 && __syncthreads_and(saturated())) {
                    done = true;
                    break;
                }
                if (term && __all_sync(0xffffffffu, saturated())) {
                    e |= 31;   // my warp is finished: skip to the next block checkpoint
                    continue;
                }
                const int f = r_idx[e];
                // the pixels' tests and alphas in one branch-free block (two
                // independent float64 chains interleave), then the blends
                double al[NPIX];
                bool use[NPIX];
                {
                    const double mx = r_mx[f], my = r_my[f], ia = r_ia[f], ib = r_ib[f], ic = r_ic[f];
                    const double op = r_op[f];
                    const bool full = r_full[f];
#pragma unroll
                    for (int k = 0; k < NPIX; ++k) {
                        const double dx = (double)pxs[k] - mx, dy = (double)pys[k] - my;
                        bool ok = valid[k] && !(term && T[k] < kCutoff);
                        if (!full)   // forward_kernel's pixel box and circle (_raster_kernels.py:178-184)
                            ok = ok && !(pxs[k] < r_x0[f] || pxs[k] > r_x1[f] || pys[k] < r_y0[f] ||
                                         pys[k] > r_y1[f]) &&
                                 !(dx * dx + dy * dy > r_rr[f]);
                        const double q = ia * dx * dx + 2.0 * ib * dx * dy + ic * dy * dy;
                        double alpha = op * exp_nonpos(-0.5 * q);
                        if (alpha > alpha_max) alpha = alpha_max;
                        use[k] = ok && !(alpha < kCutoff);
                        al[k] = alpha;
                    }
                }
                // per pixel: points blended (m) and the weights, in float64
                int mm[NPIX];
                double wa[NPIX], wsum[NPIX];
                float omf[NPIX];
                const int32_t b0 = r_start[f], cnt = r_count[f];
                // (1-alpha)^e for all pixels in one square-and-multiply loop
                // (e is the run's: uniform across the warp)
                double pw[NPIX];
                {
                    double bb[NPIX];
#pragma unroll
                    for (int k = 0; k < NPIX; ++k) {
                        pw[k] = 1.0;
                        bb[k] = 1.0 - al[k];
                    }
                    for (int ex = term ? cnt - 1 : cnt; ex; ex >>= 1) {
                        if (ex & 1) {
#pragma unroll
                            for (int k = 0; k < NPIX; ++k) pw[k] = pw[k] * bb[k];
                        }
#pragma unroll
                        for (int k = 0; k < NPIX; ++k) bb[k] = bb[k] * bb[k];
                    }
                }
#pragma unroll
                for (int k = 0; k < NPIX; ++k) {
                    mm[k] = 0;
                    wa[k] = wsum[k] = 0.0;
                    omf[k] = 0.f;
                    if (!use[k]) continue;
                    const double alpha = al[k];
                    const double om = 1.0 - alpha;
                    const double T0 = T[k];
                    int m = cnt;
                    double Tend;
                    if (term) {
                        const double Tl = T0 * pw[k];   // T before the last point
                        if (Tl >= kCutoff * (1.0 + 1e-12)) {
                            Tend = Tl * om;
                        } else {   // the run crosses the cutoff: exact per-point iteration
                            double Tt = T0;
                            int j = 0;
                            while (j < cnt && !(Tt < kCutoff)) {
                                Tt = Tt * om;
                                ++j;
                            }
                            m = j;
                            Tend = Tt;
                        }
                    } else {
                        Tend = T0 * pw[k];
                    }
                    if (P.dbg) {
                        atomicAdd((unsigned long long *)&P.dbg[4 * t + 2], 1ull);
                        atomicAdd((unsigned long long *)&P.dbg[4 * t + 3], (unsigned long long)m);
                    }
                    mm[k] = m;
                    wa[k] = T0 * alpha;    // weight of the run's first point
                    wsum[k] = T0 - Tend;   // total weight of its m points
                    omf[k] = (float)om;
                    T[k] = Tend;
                }
                // colour (and non-uniform normal) sums: pixel pairs with the
                // same m share the loads of the run's points
                auto sums = [&](const float4 *__restrict__ v, CompAcc *a0, CompAcc *a1, CompAcc *a2) {
#pragma unroll
                    for (int k = 0; k < NPIX; k += 2) {
                        if (k + 1 < NPIX && use[k] && use[k + 1] && mm[k] == mm[k + 1]) {
                            float3 S0, S1;
                            horner3x2(v, mm[k], omf[k], omf[k + 1], S0, S1);
                            a0[k] = acc_fma(wa[k], S0.x, a0[k]);
                            a1[k] = acc_fma(wa[k], S0.y, a1[k]);
                            a2[k] = acc_fma(wa[k], S0.z, a2[k]);
                            a0[k + 1] = acc_fma(wa[k + 1], S1.x, a0[k + 1]);
                            a1[k + 1] = acc_fma(wa[k + 1], S1.y, a1[k + 1]);
                            a2[k + 1] = acc_fma(wa[k + 1], S1.z, a2[k + 1]);
                            continue;
                        }
#pragma unroll
                        for (int u = k; u < k + 2 && u < NPIX; ++u) {
                            if (!use[u]) continue;
                            const float3 S = horner3(v, mm[u], omf[u]);
                            a0[u] = acc_fma(wa[u], S.x, a0[u]);
                            a1[u] = acc_fma(wa[u], S.y, a1[u]);
                            a2[u] = acc_fma(wa[u], S.z, a2[u]);
                        }
                    }
                };
                if (want_rgb) sums(scol + b0, c0, c1, c2);
                if (want_n) {
                    if (r_uni[f]) {
#pragma unroll
                        for (int k = 0; k < NPIX; ++k) {
                            if (!use[k]) continue;
                            n0[k] = acc_fma(wsum[k], r_rn[0][f], n0[k]);
                            n1[k] = acc_fma(wsum[k], r_rn[1][f], n1[k]);
                            n2[k] = acc_fma(wsum[k], r_rn[2][f], n2[k]);
                        }
                    } else {
                        sums(snrm + b0, n0, n1, n2);
                    }
                }
                if (want_d) {
#pragma unroll
                    for (int k = 0; k < NPIX; ++k)
                        if (use[k]) dd[k] = acc_fma(wsum[k], r_dep[f], dd[k]);
                }
            }
            if (done) break;
            if (term) done = __syncthreads_and(saturated());
            else __syncthreads();
        }
        if (threadIdx.x == 0) s_ws = min(s_ws * 2, kWin);
        if (P.dbg && threadIdx.x == 0) {
            atomicAdd((unsigned long long *)&P.dbg[4 * t + 0], 1ull);
            atomicAdd((unsigned long long *)&P.dbg[4 * t + 1], (unsigned long long)nlist);
        }
    }
    // planes (rasterizer.py:140-149; FrameBuffer clips T to [0,1])
    const double bgc[3] = {P.fp->bg[0], P.fp->bg[1], P.fp->bg[2]};
#pragma unroll
    for (int k = 0; k < NPIX; ++k) {
        if (!valid[k]) continue;
        const int64_t pix = (int64_t)pys[k] * P.W + pxs[k];
        if (P.rgba) {   // service.py:116-136 render_pose + to_rgba (+ relight)
            const FrameParams &F = *P.fp;
            const double tc = fmin(fmax(T[k], 0.0), 1.0);
            double v[3];
            if (F.shade_mode == SFB_MODE_RGB || F.shade_mode == SFB_MODE_RELIT) {
                v[0] = c0[k] + T[k] * bgc[0];
                v[1] = c1[k] + T[k] * bgc[1];
                v[2] = c2[k] + T[k] * bgc[2];
            }
            if (F.shade_mode != SFB_MODE_RGB) {
                const double nrm = sqrt(n0[k] * n0[k] + n1[k] * n1[k] + n2[k] * n2[k]);
                const bool z = !(nrm > 0.0);
                const double inv = 1.0 / nrm;   // one division (the planes are float32)
                const double u0 = z ? 0.0 : n0[k] * inv, u1 = z ? 0.0 : n1[k] * inv,
                             u2 = z ? 0.0 : n2[k] * inv;
                if (F.shade_mode == SFB_MODE_NORMAL) {
                    v[0] = u0 * 0.5 + 0.5;
                    v[1] = u1 * 0.5 + 0.5;
                    v[2] = u2 * 0.5 + 0.5;
                } else if (!(tc > 0.999)) {   // relight (rasterizer.py:209-226)
                    const double lam = fmax(u0 * F.light[0] + u1 * F.light[1] + u2 * F.light[2], 0.0);
                    const double g = F.ambient + F.diffuse * lam;
#pragma unroll
                    for (int a = 0; a < 3; ++a) v[a] = fmin(fmax(v[a] * g, 0.0), 1.0);
                } else {
#pragma unroll
                    for (int a = 0; a < 3; ++a) v[a] = fmin(fmax(v[a], 0.0), 1.0);
                }
            }
            uchar4 q;
            q.x = (unsigned char)fmin(fmax(rint(v[0] * 255.0), 0.0), 255.0);
            q.y = (unsigned char)fmin(fmax(rint(v[1] * 255.0), 0.0), 255.0);
            q.z = (unsigned char)fmin(fmax(rint(v[2] * 255.0), 0.0), 255.0);
            q.w = (unsigned char)fmin(fmax(rint((1.0 - tc) * 255.0), 0.0), 255.0);
            reinterpret_cast<uchar4 *>(P.rgba)[pix] = q;
        }
        if (P.rgb) {
            P.rgb[3 * pix + 0] = (float)(c0[k] + T[k] * bgc[0]);
            P.rgb[3 * pix + 1] = (float)(c1[k] + T[k] * bgc[1]);
            P.rgb[3 * pix + 2] = (float)(c2[k] + T[k] * bgc[2]);
        }
        if (P.normal) {
            const double nrm = sqrt(n0[k] * n0[k] + n1[k] * n1[k] + n2[k] * n2[k]);
            const bool z = !(nrm > 0.0);
            const double inv = 1.0 / nrm;   // one division (the planes are float32)
            P.normal[3 * pix + 0] = z ? 0.f : (float)(n0[k] * inv);
            P.normal[3 * pix + 1] = z ? 0.f : (float)(n1[k] * inv);
            P.normal[3 * pix + 2] = z ? 0.f : (float)(n2[k] * inv);
        }
        if (P.depth) P.depth[pix] = (float)dd[k];
        if (P.trans) P.trans[pix] = (float)fmin(fmax(T[k], 0.0), 1.0);
    }
}

// ------------------------------------------------------------ driver
__global__ void k_widen(const uint32_t *__restrict__ a, int64_t n, int64_t *__restrict__ b);

// voxel-level depth order (see k_vdepth_keys): fills src (rank -> point) and
// the rank-ordered colours; returns the sorted kept voxels, their exact depth
// bits, rank offsets and point counts, and the device count of kept voxels
static void voxel_order(sfb_ctx *ctx, const RenderInputs &in, const Proj &P, DevCounts *C,
                        uint32_t *src, float4 *scol, uint32_t *&vs, unsigned long long *&full,
                        int32_t *&off, int32_t *&cnt, int64_t *&d_kg, int32_t *&vpos,
                        int32_t *thead, int2 *&gspan) {
    cudaStream_t st = ctx->stream;
    const int64_t nbg = in.n_geom > 0 ? in.n_geom : 1;
    const unsigned gv = dgrid(ctx->grid_bound(nbg, ctx->hint_m[0]), 256);
    uint32_t *k0 = ctx->arena.alloc<uint32_t>(nbg), *k1 = ctx->arena.alloc<uint32_t>(nbg);
    uint32_t *v0 = ctx->arena.alloc<uint32_t>(nbg), *v1 = ctx->arena.alloc<uint32_t>(nbg);
    vpos = ctx->arena.alloc<int32_t>(nbg);
    d_kg = &C->scratch[3];
    // the depth range came with the projection (DevCounts::zr)
    k_vdepth_keys<<<gv, 256, 0, st>>>(in.d_n_geom, P, C->zr, k0, v0, vpos, d_kg);
    SFB_CHECK_LAUNCH();
    // stable by voxel id within equal quantised keys; culled voxels (key ~0) last
    const bool second = dsort_pairs<uint32_t>(ctx, k0, v0, k1, v1, in.d_n_geom, nbg, 24);
    uint32_t *ks = second ? k1 : k0;
    vs = second ? v1 : v0;
    // exact (depth bits, voxel id) order inside equal-quantised-key groups
    full = ctx->arena.alloc<unsigned long long>(nbg);
    uint8_t *need = ctx->arena.alloc<uint8_t>(4 * nbg);
    uint32_t *heads = ctx->arena.alloc<uint32_t>(nbg);
    SFB_CUDA(cudaMemsetAsync(need, 0, 4 * nbg, st));
    k_depth_full<<<gv, 256, 0, st>>>(vs, nullptr, P, d_kg, full);
    k_depth_mark<<<gv, 256, 0, st>>>(ks, full, d_kg, need, heads, &C->scratch[2]);
    k_depth_fixup<<<2 * 148, 256, 0, st>>>(ks, vs, full, d_kg, heads, &C->scratch[2]);
    SFB_CHECK_LAUNCH();
    cnt = ctx->arena.alloc<int32_t>(nbg);
    off = ctx->arena.alloc<int32_t>(nbg);
    k_vcounts<<<gv, 256, 0, st>>>(vs, d_kg, in.geom_offsets, cnt, vpos);
    SFB_CHECK_LAUNCH();
    dscan(ctx, cnt, off, d_kg, nbg, &C->kept, false);
    gspan = ctx->arena.alloc<int2>(nbg);
    k_vranks<32><<<dgrid(32 * ctx->grid_bound(nbg, ctx->hint_m[0]), 256), 256, 0, st>>>(
        in.geom_order, in.geom_offsets, off, full, vs, d_kg, in.colors, scol, src, thead, gspan);
    SFB_CHECK_LAUNCH();
}

// No host synchronisation: every size (kept points, runs, pyramid entries)
// stays on the device; buffers are sized from host bounds.
void render_run(sfb_ctx *ctx, const RenderInputs &in, const FrameParams *FP, int64_t width,
                int64_t height, const sfb_render_options &opts, int plane_mask, DevCounts *C,
                float *rgb, float *normal, float *depth, float *trans, uint8_t *rgba) {
    SFB_REQUIRE(width >= 1 && height >= 1, "image must have positive dimensions");
    SFB_REQUIRE(opts.tile_size >= 1 && opts.tile_size <= 32, "tile_size must be in [1, 32]");
    cudaStream_t st = ctx->stream;
    const int TS = opts.tile_size;
    const int64_t ntx = (width + TS - 1) / TS, nty = (height + TS - 1) / TS;
    const int64_t nsx = (ntx + kSuper - 1) / kSuper, nsy = (nty + kSuper - 1) / kSuper;
    const int64_t nt = ntx * nty, ns = nsx * nsy;
    const int64_t n = in.n_points;
    Proj P = project_inputs(ctx, in, FP, C->zr);
    ctx->mark(ST_PROJECT);
    const int64_t nb = n > 0 ? n : 1;
    const bool want_rgb = plane_mask & SFB_PLANE_RGB, want_n = plane_mask & SFB_PLANE_NORMAL;
    float4 *scol = want_rgb ? ctx->arena.alloc<float4>(nb) : nullptr;
    float4 *snrm = (want_n && !in.point_to_geom) ? ctx->arena.alloc<float4>(nb) : nullptr;
    // voxel-level order (fused frame): sorted kept voxels, their point offsets
    const bool by_voxel = in.point_to_geom && in.geom_offsets && in.geom_order && n > 0;
    uint32_t *vs = nullptr;
    unsigned long long *vfull = nullptr;
    int32_t *voff = nullptr, *vcnt = nullptr;
    int64_t *d_kg = nullptr;
    int32_t *vpos = nullptr, *thead = nullptr;
    int2 *gspan = nullptr;
    uint32_t *src;
    if (by_voxel) {
        src = ctx->arena.alloc<uint32_t>(nb);
        thead = ctx->arena.alloc<int32_t>(nb);
        voxel_order(ctx, in, P, C, src, scol, vs, vfull, voff, vcnt, d_kg, vpos, thead, gspan);
    } else {
        src = n > 0 ? depth_order(ctx, in, P, C) : ctx->arena.alloc<uint32_t>(1);
    }
    ctx->mark(ST_SORT);

    Runs R{};
    R.d_R = &C->runs;
    int32_t *head = ctx->arena.alloc<int32_t>(nb);
    R.rec = ctx->arena.alloc<RunRec>(nb);
    R.aux = ctx->arena.alloc<RunAux>(nb);
    R.start = ctx->arena.alloc<int32_t>(nb);
    R.count = ctx->arena.alloc<int32_t>(nb);

    R.rect = ctx->arena.alloc<int4>(nb);
    R.level = ctx->arena.alloc<uint8_t>(nb);
    int32_t *cnts = ctx->arena.alloc<int32_t>(3 * (nb + 1));
    R.nf = cnts;
    R.ns = cnts + (nb + 1);
    R.ng = cnts + 2 * (nb + 1);
    int32_t *pos = ctx->arena.alloc<int32_t>(3 * (nb + 1));
    // fine / super entry capacity: at most kFineMax per run and level; sized
    // from the last eager frame's demand (x2, >= 64k), 4 M entries before
    // any hint; a frame that needs more falls back to the global list
    // (k_entry_guard), so the bound never has to cover kFineMax x points
    const int64_t ebound =
        ctx->entry_cap_override > 0
            ? ctx->entry_cap_override
            : std::min<int64_t>(kFineMax * nb, ctx->hint_e > 0
                                                   ? std::max<int64_t>(2 * ctx->hint_e, int64_t(1) << 16)
                                                   : int64_t(1) << 22);
    uint32_t *fkey = ctx->arena.alloc<uint32_t>(ebound), *fval = ctx->arena.alloc<uint32_t>(ebound);
    uint32_t *fkey2 = ctx->arena.alloc<uint32_t>(ebound), *fval2 = ctx->arena.alloc<uint32_t>(ebound);
    uint32_t *skey = ctx->arena.alloc<uint32_t>(ebound), *sval = ctx->arena.alloc<uint32_t>(ebound);
    uint32_t *skey2 = ctx->arena.alloc<uint32_t>(ebound), *sval2 = ctx->arena.alloc<uint32_t>(ebound);
    uint32_t *glist = ctx->arena.alloc<uint32_t>(nb);
    int4 *grect = ctx->arena.alloc<int4>(nb);
    int4 *srect = ctx->arena.alloc<int4>(ebound);
    int32_t *f_off = ctx->arena.alloc<int32_t>(nt + 1);
    int32_t *s_off = ctx->arena.alloc<int32_t>(ns + 1);
    const uint32_t *fk_sorted = fkey, *sk_sorted = skey;
    SFB_CUDA(cudaMemsetAsync(cnts, 0, sizeof(int32_t) * 3 * (nb + 1), st));
    const uint32_t *f_ids = fval, *s_ids = sval;
    if (n > 0) {
        if (by_voxel) {
            const unsigned gv = dgrid(ctx->grid_bound(in.n_geom, ctx->hint_m[0]), 256);
            int32_t *hincl = head;   // inclusive count of tie-group run heads per rank
            dscan(ctx, thead, hincl, &C->kept, n, nullptr, true);
            int32_t *nblk = ctx->arena.alloc<int32_t>(in.n_geom + 1);   // then run offsets
            k_vblocks<<<gv, 256, 0, st>>>(gspan, d_kg, voff, vcnt, hincl, nblk);
            SFB_CHECK_LAUNCH();
            dscan(ctx, nblk, nblk, d_kg, in.n_geom, &C->runs, false);
            k_vbuild<<<dgrid(n, 256), 256, 0, st>>>(vs, gspan, C, d_kg, voff, vcnt, nblk, vpos, thead,
                                                   hincl, src, in.point_to_geom, P, in.opac,
                                                   (double)TS, ntx, nty, opts.alpha_max, R);
            SFB_CHECK_LAUNCH();
        } else {
            const unsigned g = dgrid(n, 256);
            k_run_heads<<<g, 256, 0, st>>>(src, &C->kept, in.point_to_geom, P, in.opac, head);
            SFB_CHECK_LAUNCH();
            dscan(ctx, head, head, &C->kept, n, nullptr, true);
            k_run_build<<<g, 256, 0, st>>>(src, C, head, in.point_to_geom, P, in.opac, (double)TS, ntx,
                                           nty, opts.alpha_max, R);
            SFB_CHECK_LAUNCH();
        }
        dscan3(ctx, R.nf, R.ns, R.ng, pos, pos + (nb + 1), pos + 2 * (nb + 1), &C->runs1, nb + 1,
               &C->ef, &C->es, &C->g);
        k_entry_guard<<<1, 1, 0, st>>>(C, ebound);
        k_emit<<<dgrid(ctx->grid_bound(n, ctx->hint_runs), 256), 256, 0, st>>>(
            R, pos, pos + (nb + 1), pos + 2 * (nb + 1), ntx, nsx, fkey, fval, skey, sval, glist, grect,
            C);
        SFB_CHECK_LAUNCH();
        if ((scol && !by_voxel) || snrm) {
            k_gather_attrs<<<dgrid(n, 256), 256, 0, st>>>(src, in.point_to_geom, in.colors,
                                                          in.normals, &C->kept, scol, snrm);
            SFB_CHECK_LAUNCH();
        }
        // side stream: the run staging and the super-tile list sort run beside
        // the fine-tile list sort (all three need only k_emit's output)
        const int fbits = bits_for((uint64_t)nt), sbits = bits_for((uint64_t)ns);
        SFB_CUDA(cudaEventRecord(ctx->side_ev[sfb_ctx::kEvBinFork], st));
        SFB_CUDA(cudaStreamWaitEvent(ctx->side_stream, ctx->side_ev[sfb_ctx::kEvBinFork], 0));
        ctx->stream = ctx->side_stream;
        try {
            k_stage_runs<<<dgrid(ctx->grid_bound(n, ctx->hint_runs), 256), 256, 0, ctx->stream>>>(
                R, src, in.point_to_geom, in.normals, P.depth, want_n ? 1 : 0);
            SFB_CHECK_LAUNCH();
            // stable sort by tile id keeps each tile's runs in rank order
            s_ids = dsort_pairs<uint32_t>(ctx, skey, sval, skey2, sval2, &C->es, ebound, sbits) ? sval2 : sval;
            SFB_CUDA(cudaEventRecord(ctx->side_ev[sfb_ctx::kEvBinJoin], ctx->stream));
        } catch (...) {
            ctx->stream = st;
            throw;
        }
        ctx->stream = st;
        sk_sorted = (s_ids == sval2) ? skey2 : skey;
        f_ids = dsort_pairs<uint32_t>(ctx, fkey, fval, fkey2, fval2, &C->ef, ebound, fbits) ? fval2 : fval;
        fk_sorted = (f_ids == fval2) ? fkey2 : fkey;
        SFB_CUDA(cudaStreamWaitEvent(st, ctx->side_ev[sfb_ctx::kEvBinJoin], 0));
    }
    // tile offsets by binary search in the sorted keys (no histogram / scan),
    // and the super-list rects in list order, in one launch
    k_tile_index<<<dgrid(std::max<int64_t>(ebound, nt + ns + 2), 256), 256, 0, st>>>(
        fk_sorted, &C->ef, sk_sorted, &C->es, s_ids, R.rect, nt, ns, f_off, s_off, srect);
    SFB_CHECK_LAUNCH();
    ctx->mark(ST_BIN);

    CompParams CP{};
    CP.W = width;
    CP.H = height;
    CP.ntx = ntx;
    CP.nty = nty;
    CP.nsx = nsx;
    CP.tile = TS;
    CP.terminate = opts.early_termination;
    CP.alpha_max = opts.alpha_max;
    CP.plane_mask = plane_mask;
    CP.fp = FP;
    CP.f_off = f_off;
    CP.f_ids = f_ids;
    CP.s_off = s_off;
    CP.s_ids = s_ids;
    CP.g_ids = glist;
    CP.s_rect = srect;
    CP.g_rect = grect;
    CP.d_G = &C->g;
    CP.R = R;
    CP.scol = scol;
    CP.snrm = snrm;
    CP.rgb = (plane_mask & SFB_PLANE_RGB) ? rgb : nullptr;
    CP.normal = (plane_mask & SFB_PLANE_NORMAL) ? normal : nullptr;
    CP.depth = (plane_mask & SFB_PLANE_DEPTH) ? depth : nullptr;
    CP.trans = trans;
    CP.rgba = rgba;
    CP.dbg = ctx->debug_counters;
    const int cm = plane_mask & 7;
    // stage timing only: after the frame's own launch, kCompReps more
    // back-to-back launches (idempotent: same lists in, same planes out)
    // between two events give the kernel's per-launch duration free of the
    // eager frame's launch gaps (sfb_stage_times stage 8)
    const int reps = ctx->timing ? 2 + kCompReps : 1;
    for (int rep = 0; rep < reps; ++rep) {
    if (rep == 1) {   // untimed: the host queues the timed reps behind it
        ctx->mark(ST_COMPOSITE);
        SFB_CUDA(cudaStreamSynchronize(st));
    }
    if (rep == 2) ctx->mark(ST_BEGIN_REPS);
    constexpr int kNpixMid = (256 + kCT - 1) / kCT, kNpixMax = (1024 + kCT - 1) / kCT;
#define SFB_COMP_CASE(M)                                                          \
    if (cm == M) {                                                                \
        if (TS * TS <= kCT) k_composite<1, M><<<(unsigned)nt, kCT, 0, st>>>(CP);  \
        else if (TS * TS <= 256) k_composite<kNpixMid, M><<<(unsigned)nt, kCT, 0, st>>>(CP); \
        else k_composite<kNpixMax, M><<<(unsigned)nt, kCT, 0, st>>>(CP);          \
    }
    SFB_COMP_CASE(0) SFB_COMP_CASE(1) SFB_COMP_CASE(2) SFB_COMP_CASE(3)
    SFB_COMP_CASE(4) SFB_COMP_CASE(5) SFB_COMP_CASE(6) SFB_COMP_CASE(7)
    }
#undef SFB_COMP_CASE
    SFB_CHECK_LAUNCH();
    ctx->mark(reps > 1 ? ST_COMPOSITE_REPS : ST_COMPOSITE);
    const FrameDebug &D = ctx->frame_debug;
    if (D.cap > 0 && D.source && n > 0) {   // parity export: rank order and runs
        SFB_REQUIRE(nb <= D.cap, "frame debug buffers are smaller than the cloud");
        k_widen<<<dgrid(nb, 256), 256, 0, st>>>(src, nb, D.source);
        SFB_CHECK_LAUNCH();
        if (D.run_start) SFB_CUDA(cudaMemcpyAsync(D.run_start, R.start, sizeof(int32_t) * nb,
                                                  cudaMemcpyDeviceToDevice, st));
        if (D.run_count) SFB_CUDA(cudaMemcpyAsync(D.run_count, R.count, sizeof(int32_t) * nb,
                                                  cudaMemcpyDeviceToDevice, st));
        if (D.run_rect) SFB_CUDA(cudaMemcpyAsync(D.run_rect, R.rect, sizeof(int4) * nb,
                                                 cudaMemcpyDeviceToDevice, st));
    }
}

// ------------------------------------------------------------ debug CSR (bin_tiles parity)
__global__ void k_rank_rects(const uint32_t *__restrict__ src, int64_t K, const int32_t *__restrict__ p2g,
                             Proj P, const double *__restrict__ opac, double ft, int64_t ntx,
                             int64_t nty, double *__restrict__ radius, int4 *__restrict__ rect,
                             int32_t *__restrict__ cnt, int64_t *__restrict__ source) {
    SFB_FOR(j, K) {
        const uint32_t i = src[j];
        const int64_t g = p2g ? p2g[i] : (int64_t)i;
        const double r = support_radius(P.a[g], P.b[g], P.c[g], opac[g]);
        radius[j] = r;
        source[j] = i;
        const TileRect t = tile_rect(P.sx[g], P.sy[g], r, ft, ntx, nty);
        rect[j] = make_int4(t.x0, t.x1, t.y0, t.y1);
        cnt[j] = (t.x0 <= t.x1 && t.y0 <= t.y1) ? (t.x1 - t.x0 + 1) * (t.y1 - t.y0 + 1) : 0;
    }
}

__global__ void k_rank_emit(const int4 *__restrict__ rect, const int32_t *__restrict__ pos, int64_t K,
                            int64_t ntx, uint32_t *__restrict__ key, uint32_t *__restrict__ val) {
    SFB_FOR(j, K) {
        const int4 t = rect[j];
        int64_t p = pos[j];
        for (int y = t.z; y <= t.w; ++y)
            for (int x = t.x; x <= t.y; ++x) {
                key[p] = (uint32_t)(y * ntx + x);
                val[p++] = (uint32_t)j;
            }
    }
}

__global__ void k_widen(const uint32_t *__restrict__ a, int64_t n, int64_t *__restrict__ b) {
    SFB_FOR(j, n) b[j] = a[j];
}
__global__ void k_widen32(const int32_t *__restrict__ a, int64_t n, int64_t *__restrict__ b) {
    SFB_FOR(j, n) b[j] = a[j];
}

// The reference CSR of _prepare + bin_tiles (rasterizer.py:99-130,
// _raster_kernels.py:108-143): rank -> splat, per-rank support radius, per-tile
// offsets and rank lists. Host-synchronising by design (it sizes buffers from
// K and E); used by the parity seam and by render_backward.
struct Csr {
    Proj P;
    uint32_t *src = nullptr;        // rank -> splat (first K)
    int64_t K = 0, E = 0;
    double *radius = nullptr;       // per rank
    int32_t *toff = nullptr;        // (nt+1) tile offsets
    const uint32_t *ids = nullptr;  // (E) ranks, tile-major, ascending within a tile
    int64_t ntx = 0, nty = 0;
};

static Csr build_csr(sfb_ctx *ctx, const RenderInputs &in, const FrameParams *FP, int64_t width,
                     int64_t height, int tile, DevCounts *C, int64_t *source) {
    cudaStream_t st = ctx->stream;
    Csr R;
    R.ntx = (width + tile - 1) / tile;
    R.nty = (height + tile - 1) / tile;
    const int64_t nt = R.ntx * R.nty;
    R.P = project_inputs(ctx, in, FP, C->zr);
    R.toff = ctx->arena.alloc<int32_t>(nt + 1);
    SFB_CUDA(cudaMemsetAsync(R.toff, 0, sizeof(int32_t) * (nt + 1), st));
    if (in.n_points > 0) {
        R.src = depth_order(ctx, in, R.P, C);
        ctx->read_back(&C->kept, sizeof(int64_t));
        R.K = ctx->pinned[0];
    }
    if (R.K == 0) return R;
    const int64_t K = R.K;
    int4 *rect = ctx->arena.alloc<int4>(K);
    int32_t *cnt = ctx->arena.alloc<int32_t>(K + 1);
    int32_t *pos = ctx->arena.alloc<int32_t>(K + 1);
    R.radius = ctx->arena.alloc<double>(K);
    int64_t *src64 = source ? source : ctx->arena.alloc<int64_t>(K);
    SFB_CUDA(cudaMemsetAsync(cnt, 0, sizeof(int32_t) * (K + 1), st));
    k_rank_rects<<<dgrid(K, 256), 256, 0, st>>>(R.src, K, in.point_to_geom, R.P, in.opac, (double)tile,
                                                R.ntx, R.nty, R.radius, rect, cnt, src64);
    dscan(ctx, cnt, pos, nullptr, K + 1, &C->scratch[0], false);
    ctx->read_back(&C->scratch[0], sizeof(int64_t));
    R.E = ctx->pinned[0];
    SFB_REQUIRE(R.E < (int64_t(1) << 31), "CSR larger than 2^31 entries");
    const int64_t E = R.E;
    uint32_t *key = ctx->arena.alloc<uint32_t>(E + 1), *val = ctx->arena.alloc<uint32_t>(E + 1);
    uint32_t *key2 = ctx->arena.alloc<uint32_t>(E + 1), *val2 = ctx->arena.alloc<uint32_t>(E + 1);
    k_rank_emit<<<dgrid(K, 256), 256, 0, st>>>(rect, pos, K, R.ntx, key, val);
    SFB_CHECK_LAUNCH();
    const int bits = bits_for((uint64_t)nt);
    const bool second = dsort_pairs<uint32_t>(ctx, key, val, key2, val2, nullptr, E, bits);
    const uint32_t *ks = second ? key2 : key;
    R.ids = second ? val2 : val;
    k_histogram<<<dgrid(E, 256), 256, 0, st>>>(ks, &C->scratch[0], R.toff);
    dscan(ctx, R.toff, R.toff, nullptr, nt + 1, nullptr, false);
    SFB_CHECK_LAUNCH();
    return R;
}

void prepare_debug_run(sfb_ctx *ctx, const RenderInputs &in, const FrameParams *FP, int64_t width,
                       int64_t height, int tile, DevCounts *C, int64_t *source, double *radius,
                       int64_t *offsets, int64_t *ids, int64_t cap, int64_t *k_host,
                       int64_t *e_host) {
    cudaStream_t st = ctx->stream;
    Csr R = build_csr(ctx, in, FP, width, height, tile, C, source);
    const int64_t nt = R.ntx * R.nty;
    *k_host = R.K;
    *e_host = R.E;
    k_widen32<<<dgrid(nt + 1, 256), 256, 0, st>>>(R.toff, nt + 1, offsets);
    if (R.K > 0) {
        SFB_CUDA(cudaMemcpyAsync(radius, R.radius, sizeof(double) * R.K, cudaMemcpyDeviceToDevice, st));
        if (R.E <= cap && ids) k_widen<<<dgrid(R.E, 256), 256, 0, st>>>(R.ids, R.E, ids);
    }
    SFB_CHECK_LAUNCH();
}

// ------------------------------------------------------------ render_backward
// Analytic gradients of render() (rasterizer.py:229-354). Per-rank inputs of
// the reference's backward_kernel (_raster_kernels.py:204-310) in rank order.
struct BwdRank {
    double *sx, *sy, *ia, *ib, *ic, *op, *attr;   // attr (K,3)
};

__global__ void k_bwd_rank_inputs(const Proj P, const uint32_t *__restrict__ src, int64_t K,
                                  const double *__restrict__ opac, const double *__restrict__ colors,
                                  const double *__restrict__ normals, int mode, BwdRank B) {
    SFB_FOR(j, K) {
        const int64_t i = src[j];
        const double a = P.a[i], b = P.b[i], c = P.c[i];
        const double det = a * c - b * b;
        B.sx[j] = P.sx[i];
        B.sy[j] = P.sy[i];
        B.ia[j] = c / det;
        B.ib[j] = -b / det;
        B.ic[j] = a / det;
        B.op[j] = opac[i];
        for (int k = 0; k < 3; ++k)
            B.attr[3 * j + k] = mode == 0 ? colors[3 * i + k]
                                : mode == 1 ? normals[3 * i + k] : (k == 0 ? P.depth[i] : 0.0);
    }
}

// block-wide sum of NV doubles in a fixed order (warp trees, then warps in
// order): deterministic run to run
template <int NV>
__device__ __forceinline__ void block_sum(double (&v)[NV], double (*s_part)[NV], double *out) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int k = 0; k < NV; ++k)
        for (int o = 16; o; o >>= 1) v[k] += __shfl_down_sync(0xffffffffu, v[k], o);
    if (lane == 0)
#pragma unroll
        for (int k = 0; k < NV; ++k) s_part[warp][k] = v[k];
    __syncthreads();
    if (threadIdx.x < NV) {
        double t = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += s_part[w][threadIdx.x];
        out[threadIdx.x] = t;
    }
    __syncthreads();
}

// One CTA per tile, one thread per pixel (tile <= 16): forward replay of the
// tile list, then the reverse sweep walked in lockstep over the entries; the
// 9 per-entry partials (g_attr 3, g_opac, g_q 3, g_mu 2) are block-summed.
__global__ void __launch_bounds__(256)
k_backward(int64_t W, int64_t H, int tile, int64_t ntx, const int32_t *__restrict__ toff,
           const uint32_t *__restrict__ ids, BwdRank B, double alpha_max, int terminate, int mode,
           const FrameParams *__restrict__ FP, const double *__restrict__ upstream,
           double *__restrict__ g_ent /* (E, 9) */) {
    __shared__ double s_part[8][9];
    __shared__ double s_out[9];
    __shared__ int s_elast;
    const int64_t t = blockIdx.x;
    const int64_t tx = t % ntx, ty = t / ntx;
    const int64_t px = tx * tile + threadIdx.x % tile, py = ty * tile + threadIdx.x / tile;
    const bool valid = (int)threadIdx.x < tile * tile && px < W && py < H;
    const int64_t start = toff[t], end = toff[t + 1];
    double tr = 1.0, n0 = 0.0, n1 = 0.0, n2 = 0.0;
    int64_t e_last = start - 1;
    if (valid)
        for (int64_t e = start; e < end; ++e) {
            const uint32_t s = ids[e];
            const double dx = (double)px - B.sx[s], dy = (double)py - B.sy[s];
            const double q = B.ia[s] * dx * dx + 2.0 * B.ib[s] * dx * dy + B.ic[s] * dy * dy;
            double alpha = B.op[s] * exp(-0.5 * q);
            if (alpha > alpha_max) alpha = alpha_max;
            if (alpha < kCutoff) continue;
            const double w = tr * alpha;
            n0 += w * B.attr[3 * s];
            n1 += w * B.attr[3 * s + 1];
            n2 += w * B.attr[3 * s + 2];
            tr *= 1.0 - alpha;
            e_last = e;
            if (terminate && tr < kCutoff) break;
        }
    const double t_fin = tr;
    double u0 = 0.0, u1 = 0.0, u2 = 0.0, d_tfin = 0.0;
    if (valid) {
        const double *up = upstream + 3 * (py * W + px);
        u0 = up[0];
        u1 = up[1];
        u2 = up[2];
        if (mode == 1) {
            const double nn = sqrt(n0 * n0 + n1 * n1 + n2 * n2);
            if (nn > 1e-12) {
                const double dot = (n0 * u0 + n1 * u1 + n2 * u2) / (nn * nn * nn);
                u0 = u0 / nn - n0 * dot;
                u1 = u1 / nn - n1 * dot;
                u2 = u2 / nn - n2 * dot;
            }
        }
        if (mode == 0) d_tfin = u0 * FP->bg[0] + u1 * FP->bg[1] + u2 * FP->bg[2];
    }
    const bool live = valid && !(u0 == 0.0 && u1 == 0.0 && u2 == 0.0);
    if (!live) e_last = start - 1;
    // lockstep reverse sweep from the largest e_last of the tile
    if (threadIdx.x == 0) s_elast = (int)(start - 1);
    __syncthreads();
    if (e_last >= start) atomicMax(&s_elast, (int)e_last);
    __syncthreads();
    const int64_t e_top = s_elast;
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, t_next = t_fin;
    for (int64_t e = e_top; e >= start; --e) {
        double v[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
        bool any = false;
        if (e <= e_last) {
            const uint32_t s = ids[e];
            const double dx = (double)px - B.sx[s], dy = (double)py - B.sy[s];
            const double ia = B.ia[s], ib = B.ib[s], ic = B.ic[s], op = B.op[s];
            const double q = ia * dx * dx + 2.0 * ib * dx * dy + ic * dy * dy;
            const double g = exp(-0.5 * q);
            const double raw = op * g;
            const bool clamped = raw > alpha_max;
            const double alpha = clamped ? alpha_max : raw;
            if (!(alpha < kCutoff)) {
                any = true;
                const double one_m = 1.0 - alpha;
                const double t_k = t_next / one_m;
                const double w = t_k * alpha;
                const double a0 = B.attr[3 * s], a1 = B.attr[3 * s + 1], a2 = B.attr[3 * s + 2];
                v[0] = u0 * w;
                v[1] = u1 * w;
                v[2] = u2 * w;
                const double d_alpha = (u0 * (t_k * a0 - s0 / one_m) + u1 * (t_k * a1 - s1 / one_m) +
                                        u2 * (t_k * a2 - s2 / one_m) - d_tfin * t_fin / one_m);
                if (!clamped) {
                    v[3] = d_alpha * g;
                    const double d_q = -0.5 * op * g * d_alpha;
                    v[4] = d_q * dx * dx;
                    v[5] = d_q * 2.0 * dx * dy;
                    v[6] = d_q * dy * dy;
                    v[7] = -(d_q * 2.0 * (ia * dx + ib * dy));
                    v[8] = -(d_q * 2.0 * (ib * dx + ic * dy));
                }
                s0 += w * a0;
                s1 += w * a1;
                s2 += w * a2;
                t_next = t_k;
            }
        }
        if (!__syncthreads_or(any)) continue;
        block_sum<9>(v, s_part, s_out);
        if (threadIdx.x < 9) g_ent[9 * e + threadIdx.x] = s_out[threadIdx.x];
    }
}

// per rank: sum of its entries' slots in CSR order (np.add.at walks ids in order)
__global__ void k_bwd_reduce(const uint32_t *__restrict__ ent_sorted, const int32_t *__restrict__ roff,
                             int64_t K, const double *__restrict__ g_ent, double *__restrict__ g_rank) {
    SFB_FOR(j, K) {
        double acc[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
        for (int32_t q = roff[j]; q < roff[j + 1]; ++q) {
            const double *g = g_ent + 9 * (size_t)ent_sorted[q];
#pragma unroll
            for (int k = 0; k < 9; ++k) acc[k] += g[k];
        }
#pragma unroll
        for (int k = 0; k < 9; ++k) g_rank[9 * j + k] = acc[k];
    }
}

// chain rule per rank (rasterizer.py:286-354): inverse-covariance partials ->
// screen covariance -> EWA Jacobian / camera point -> world covariance ->
// scales and the normalised quaternion; written at the splat's input index
__global__ void k_bwd_chain(const uint32_t *__restrict__ src, int64_t K, const double *__restrict__ g_rank,
                            const BwdRank B, const double *__restrict__ centers,
                            const double *__restrict__ scales, const double *__restrict__ quats,
                            const FrameParams *__restrict__ FP, int mode, double *__restrict__ d_centers,
                            double *__restrict__ d_scales, double *__restrict__ d_quats,
                            double *__restrict__ d_opac, double *__restrict__ d_colors,
                            double *__restrict__ d_normals) {
    const Cam C = FP->cam;
    SFB_FOR(j, K) {
        const int64_t i = src[j];
        const double *g = g_rank + 9 * j;   // attr 0-2, opac 3, q 4-6, mu 7-8
        const double ia = B.ia[j], ib = B.ib[j], ic = B.ic[j];
        const double im[2][2] = {{ia, ib}, {ib, ic}};
        const double gi[2][2] = {{g[4], 0.5 * g[5]}, {0.5 * g[5], g[6]}};
        double tmp[2][2], gcov[2][2];
        for (int r = 0; r < 2; ++r)
            for (int c = 0; c < 2; ++c) tmp[r][c] = im[r][0] * gi[0][c] + im[r][1] * gi[1][c];
        for (int r = 0; r < 2; ++r)
            for (int c = 0; c < 2; ++c) gcov[r][c] = -(tmp[r][0] * im[0][c] + tmp[r][1] * im[1][c]);
        const double *R = C.r;
        const double *ce = centers + 3 * i;
        double pc[3];
        for (int r = 0; r < 3; ++r) pc[r] = ce[0] * R[3 * r] + ce[1] * R[3 * r + 1] + ce[2] * R[3 * r + 2] + C.t[r];
        const double x = pc[0], y = pc[1], z = pc[2];
        double jac[2][3] = {{C.fx / z, 0.0, -C.fx * x / (z * z)}, {0.0, C.fy / z, -C.fy * y / (z * z)}};
        double a2m[2][3];
        for (int r = 0; r < 2; ++r)
            for (int c = 0; c < 3; ++c)
                a2m[r][c] = jac[r][0] * R[c] + jac[r][1] * R[3 + c] + jac[r][2] * R[6 + c];
        double gs3[3][3];
        for (int a = 0; a < 3; ++a)
            for (int m = 0; m < 3; ++m) {
                double acc = 0.0;
                for (int jj = 0; jj < 2; ++jj)
                    for (int l = 0; l < 2; ++l) acc += a2m[jj][a] * gcov[jj][l] * a2m[l][m];
                gs3[a][m] = acc;
            }
        // rotation of the (normalised) quaternion, sigma3 = rot^T diag(s^2) rot
        const double *qq = quats + 4 * i;
        const double qn = sqrt(qq[0] * qq[0] + qq[1] * qq[1] + qq[2] * qq[2] + qq[3] * qq[3]);
        const double w = qq[0] / qn, qx = qq[1] / qn, qy = qq[2] / qn, qz = qq[3] / qn;
        const double rot[3][3] = {{1 - 2 * (qy * qy + qz * qz), 2 * (qx * qy - w * qz), 2 * (qx * qz + w * qy)},
                                  {2 * (qx * qy + w * qz), 1 - 2 * (qx * qx + qz * qz), 2 * (qy * qz - w * qx)},
                                  {2 * (qx * qz - w * qy), 2 * (qy * qz + w * qx), 1 - 2 * (qx * qx + qy * qy)}};
        const double *sc = scales + 3 * i;
        const double s2[3] = {sc[0] * sc[0], sc[1] * sc[1], sc[2] * sc[2]};
        double sig[3][3];
        for (int a = 0; a < 3; ++a)
            for (int l = 0; l < 3; ++l)
                sig[a][l] = rot[0][a] * s2[0] * rot[0][l] + rot[1][a] * s2[1] * rot[1][l] + rot[2][a] * s2[2] * rot[2][l];
        double mcam[3][3];
        for (int a = 0; a < 3; ++a)
            for (int m = 0; m < 3; ++m) {
                double acc = 0.0;
                for (int jj = 0; jj < 3; ++jj)
                    for (int l = 0; l < 3; ++l) acc += R[3 * a + jj] * sig[jj][l] * R[3 * m + l];
                mcam[a][m] = acc;
            }
        double gjac[2][3];
        for (int a = 0; a < 2; ++a)
            for (int m = 0; m < 3; ++m) {
                double acc = 0.0;
                for (int jj = 0; jj < 2; ++jj)
                    for (int l = 0; l < 3; ++l) acc += gcov[a][jj] * jac[jj][l] * mcam[l][m];
                gjac[a][m] = 2.0 * acc;
            }
        double dp[3];
        dp[0] = gjac[0][2] * (-C.fx / (z * z));
        dp[1] = gjac[1][2] * (-C.fy / (z * z));
        dp[2] = gjac[0][0] * (-C.fx / (z * z)) + gjac[0][2] * (2.0 * C.fx * x / (z * z * z)) +
                gjac[1][1] * (-C.fy / (z * z)) + gjac[1][2] * (2.0 * C.fy * y / (z * z * z));
        dp[0] += g[7] * C.fx / z;
        dp[1] += g[8] * C.fy / z;
        dp[2] += g[7] * (-C.fx * x / (z * z)) + g[8] * (-C.fy * y / (z * z));
        if (mode == 2) dp[2] += g[0];
        for (int c = 0; c < 3; ++c) d_centers[3 * i + c] = dp[0] * R[c] + dp[1] * R[3 + c] + dp[2] * R[6 + c];
        // g_d = rot gs3 rot^T ; d_scales = 2 s diag(g_d)
        for (int a = 0; a < 3; ++a) {
            double acc = 0.0;
            for (int jj = 0; jj < 3; ++jj)
                for (int l = 0; l < 3; ++l) acc += rot[a][jj] * gs3[jj][l] * rot[a][l];
            d_scales[3 * i + a] = 2.0 * sc[a] * acc;
        }
        // g_r = 2 s^2 (rot gs3); d_qhat = <g_r, dR/dq>
        double gr[3][3];
        for (int a = 0; a < 3; ++a)
            for (int c = 0; c < 3; ++c)
                gr[a][c] = 2.0 * s2[a] * (rot[a][0] * gs3[0][c] + rot[a][1] * gs3[1][c] + rot[a][2] * gs3[2][c]);
        const double dr[4][9] = {{0, -qz, qy, qz, 0, -qx, -qy, qx, 0},
                                 {0, qy, qz, qy, -2 * qx, -w, qz, w, -2 * qx},
                                 {-2 * qy, qx, w, qx, 0, qz, -w, qz, -2 * qy},
                                 {-2 * qz, -w, qx, w, -2 * qz, qy, qx, qy, 0}};
        double dq[4];
        for (int k = 0; k < 4; ++k) {
            double acc = 0.0;
            for (int e = 0; e < 9; ++e) acc += gr[e / 3][e % 3] * 2.0 * dr[k][e];
            dq[k] = acc;
        }
        const double qh[4] = {w, qx, qy, qz};
        const double dot = qh[0] * dq[0] + qh[1] * dq[1] + qh[2] * dq[2] + qh[3] * dq[3];
        for (int k = 0; k < 4; ++k) d_quats[4 * i + k] = (dq[k] - qh[k] * dot) / qn;
        d_opac[i] = g[3];
        if (mode == 0 && d_colors)
            for (int c = 0; c < 3; ++c) d_colors[3 * i + c] = g[c];
        if (mode == 1 && d_normals)
            for (int c = 0; c < 3; ++c) d_normals[3 * i + c] = g[c];
    }
}

__global__ void k_upcast_ranks(const uint32_t *__restrict__ ids, int64_t E, uint32_t *__restrict__ key,
                               uint32_t *__restrict__ val) {
    SFB_FOR(e, E) {
        key[e] = ids[e];
        val[e] = (uint32_t)e;
    }
}

void render_backward_run(sfb_ctx *ctx, const RenderInputs &in, const FrameParams *FP, int64_t width,
                         int64_t height, const sfb_render_options &opts, int mode, DevCounts *C,
                         const double *upstream, double *d_centers, double *d_scales,
                         double *d_quats, double *d_opac, double *d_colors, double *d_normals) {
    SFB_REQUIRE(mode >= 0 && mode <= 2, "mode must be rgb, normal or depth");
    SFB_REQUIRE(opts.tile_size >= 1 && opts.tile_size <= 16, "render_backward supports tile_size <= 16");
    cudaStream_t st = ctx->stream;
    const int64_t n = in.n_points;
    for (auto pr : {std::make_pair(d_centers, 3), std::make_pair(d_scales, 3), std::make_pair(d_quats, 4),
                    std::make_pair(d_opac, 1), std::make_pair(d_colors, 3), std::make_pair(d_normals, 3)})
        if (pr.first) SFB_CUDA(cudaMemsetAsync(pr.first, 0, sizeof(double) * pr.second * (size_t)n, st));
    if (n == 0) return;
    Csr R = build_csr(ctx, in, FP, width, height, opts.tile_size, C, nullptr);
    if (R.K == 0) return;
    const int64_t K = R.K, E = R.E;
    BwdRank B;
    double *blk = ctx->arena.alloc<double>(9 * (size_t)K);
    B.sx = blk;
    B.sy = blk + K;
    B.ia = blk + 2 * K;
    B.ib = blk + 3 * K;
    B.ic = blk + 4 * K;
    B.op = blk + 5 * K;
    B.attr = blk + 6 * K;
    k_bwd_rank_inputs<<<dgrid(K, 256), 256, 0, st>>>(R.P, R.src, K, in.opac, in.colors, in.normals, mode, B);
    double *g_ent = ctx->arena.alloc<double>(9 * (size_t)(E > 0 ? E : 1));
    SFB_CUDA(cudaMemsetAsync(g_ent, 0, sizeof(double) * 9 * (size_t)(E > 0 ? E : 1), st));
    k_backward<<<(unsigned)(R.ntx * R.nty), 256, 0, st>>>(width, height, opts.tile_size, R.ntx, R.toff,
                                                         R.ids, B, opts.alpha_max, opts.early_termination,
                                                         mode, FP, upstream, g_ent);
    SFB_CHECK_LAUNCH();
    // entries -> ranks in CSR order: stable sort of (rank, entry)
    uint32_t *key = ctx->arena.alloc<uint32_t>(E + 1), *val = ctx->arena.alloc<uint32_t>(E + 1);
    uint32_t *key2 = ctx->arena.alloc<uint32_t>(E + 1), *val2 = ctx->arena.alloc<uint32_t>(E + 1);
    k_upcast_ranks<<<dgrid(E, 256), 256, 0, st>>>(R.ids, E, key, val);
    const bool second = dsort_pairs<uint32_t>(ctx, key, val, key2, val2, nullptr, E,
                                              bits_for((uint64_t)K));
    const uint32_t *ks = second ? key2 : key, *vs = second ? val2 : val;
    int32_t *roff = ctx->arena.alloc<int32_t>(K + 1);
    SFB_CUDA(cudaMemsetAsync(roff, 0, sizeof(int32_t) * (K + 1), st));
    k_histogram<<<dgrid(E, 256), 256, 0, st>>>(ks, &C->scratch[0], roff);   // scratch[0] = E
    dscan(ctx, roff, roff, nullptr, K + 1, nullptr, false);
    double *g_rank = ctx->arena.alloc<double>(9 * (size_t)K);
    k_bwd_reduce<<<dgrid(K, 256), 256, 0, st>>>(vs, roff, K, g_ent, g_rank);
    k_bwd_chain<<<dgrid(K, 128), 128, 0, st>>>(R.src, K, g_rank, B, in.centers, in.scales, in.quats, FP,
                                              mode, d_centers, d_scales, d_quats, d_opac, d_colors,
                                              d_normals);
    SFB_CHECK_LAUNCH();
}

}  // namespace sfb
