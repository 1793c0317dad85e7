// Density-1 voxelization on the device (reference: voxelgrid.py:125-168).
//
//   bbox reduce -> (host) s -> keygen: floor(p*s) packed into a compact
//   (z,y,x)-ordered key of only the bits the cloud needs -> stable LSD radix
//   sort of (key, point index) -> run-length segmentation -> per-voxel ordered
//   float64 sums (bit-identical to np.add.at, which walks points in increasing
//   index) -> 9 feature channels.
// HBM-bound integer/byte work; no tensor cores.
#include <cub/cub.cuh>

#include "common.cuh"

namespace sfb {

__device__ __forceinline__ unsigned long long ord_bits(double v) {
    unsigned long long u = __double_as_longlong(v);
    return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}
static inline double unord_bits(unsigned long long u) {
    u = (u >> 63) ? (u & 0x7fffffffffffffffull) : ~u;
    double d;
    std::memcpy(&d, &u, 8);
    return d;
}

__global__ void k_bbox_init(unsigned long long *mm) {
    int t = threadIdx.x;
    if (t < 3) mm[t] = ~0ull;
    else if (t < 6) mm[t] = 0ull;
}

__global__ void k_bbox(const double *__restrict__ pos, int64_t n, unsigned long long *mm) {
    unsigned long long lo[3] = {~0ull, ~0ull, ~0ull}, hi[3] = {0, 0, 0};
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            unsigned long long u = ord_bits(pos[3 * i + a]);
            lo[a] = u < lo[a] ? u : lo[a];
            hi[a] = u > hi[a] ? u : hi[a];
        }
    }
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        for (int o = 16; o; o >>= 1) {
            unsigned long long l2 = __shfl_xor_sync(0xffffffffu, lo[a], o);
            unsigned long long h2 = __shfl_xor_sync(0xffffffffu, hi[a], o);
            lo[a] = l2 < lo[a] ? l2 : lo[a];
            hi[a] = h2 > hi[a] ? h2 : hi[a];
        }
    }
    if ((threadIdx.x & 31) == 0) {
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            atomicMin(&mm[a], lo[a]);
            atomicMax(&mm[3 + a], hi[a]);
        }
    }
}

void bbox_run(sfb_ctx *ctx, const double *pos, int64_t n, double *lo_hi_host) {
    SFB_REQUIRE(n > 0, "empty cloud has no bbox");
    auto *mm = ctx->arena.alloc<unsigned long long>(6);
    k_bbox_init<<<1, 32, 0, ctx->stream>>>(mm);
    k_bbox<<<grid_for(n, 256, ctx->num_sms * 8), 256, 0, ctx->stream>>>(pos, n, mm);
    SFB_CHECK_LAUNCH();
    ctx->read_back(mm, 6 * sizeof(unsigned long long));
    for (int a = 0; a < 6; ++a) lo_hi_host[a] = unord_bits((unsigned long long)ctx->pinned[a]);
}

struct KeyLayout {
    int64_t lo[3];
    int bits[3];
    int total;
};

template <class K>
__global__ void k_keygen(const double *__restrict__ pos, int64_t n, double s, KeyLayout L,
                         K *__restrict__ keys, uint32_t *__restrict__ vals) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    int64_t ix = (int64_t)floor(__dmul_rn(pos[3 * i + 0], s)) - L.lo[0];
    int64_t iy = (int64_t)floor(__dmul_rn(pos[3 * i + 1], s)) - L.lo[1];
    int64_t iz = (int64_t)floor(__dmul_rn(pos[3 * i + 2], s)) - L.lo[2];
    keys[i] = (K)(((uint64_t)iz << (L.bits[0] + L.bits[1])) | ((uint64_t)iy << L.bits[0]) |
                  (uint64_t)ix);
    vals[i] = (uint32_t)i;
}

template <class K>
__global__ void k_heads(const K *__restrict__ keys, int64_t n, int32_t *__restrict__ flag) {
    int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (j >= n) return;
    flag[j] = (j == 0 || keys[j] != keys[j - 1]) ? 1 : 0;
}

template <class K>
__global__ void k_segments(const K *__restrict__ keys, const uint32_t *__restrict__ vals,
                           const int32_t *__restrict__ incl, int64_t n, KeyLayout L,
                           int32_t *__restrict__ coords, int64_t *__restrict__ pkeys,
                           int32_t *__restrict__ p2v, int32_t *__restrict__ order,
                           int32_t *__restrict__ offsets) {
    int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (j >= n) return;
    int32_t v = incl[j] - 1;
    uint32_t i = vals[j];
    order[j] = (int32_t)i;
    p2v[i] = v;
    if (j == n - 1) offsets[v + 1] = (int32_t)n;
    if (j == 0 || incl[j - 1] != incl[j]) {
        uint64_t k = (uint64_t)keys[j];
        int64_t x = (int64_t)(k & ((1ull << L.bits[0]) - 1)) + L.lo[0];
        int64_t y = (int64_t)((k >> L.bits[0]) & ((1ull << L.bits[1]) - 1)) + L.lo[1];
        int64_t z = (int64_t)(k >> (L.bits[0] + L.bits[1])) + L.lo[2];
        coords[3 * v + 0] = (int32_t)x;
        coords[3 * v + 1] = (int32_t)y;
        coords[3 * v + 2] = (int32_t)z;
        pkeys[v] = pack_key(x, y, z);
        offsets[v] = (int32_t)j;
    }
}

// One thread per voxel: ordered float64 sums over its points (ascending index).
__global__ void k_voxel_feats(const double *__restrict__ pos, const double *__restrict__ col,
                              const int32_t *__restrict__ order, const int32_t *__restrict__ offsets,
                              const int32_t *__restrict__ coords, int64_t m, double s,
                              double *__restrict__ feats) {
    int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (v >= m) return;
    int32_t b = offsets[v], e = offsets[v + 1];
    double c0 = 0.0, c1 = 0.0, c2 = 0.0, r0 = 0.0, r1 = 0.0, r2 = 0.0;
    for (int32_t j = b; j < e; ++j) {
        int64_t i = order[j];
        c0 = __dadd_rn(c0, __dmul_rn(pos[3 * i + 0], s));
        c1 = __dadd_rn(c1, __dmul_rn(pos[3 * i + 1], s));
        c2 = __dadd_rn(c2, __dmul_rn(pos[3 * i + 2], s));
        r0 = __dadd_rn(r0, col[3 * i + 0]);
        r1 = __dadd_rn(r1, col[3 * i + 1]);
        r2 = __dadd_rn(r2, col[3 * i + 2]);
    }
    double cnt = (double)(e - b);
    double cen[3] = {__ddiv_rn(c0, cnt), __ddiv_rn(c1, cnt), __ddiv_rn(c2, cnt)};
    double *f = feats + 9 * v;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        double res = __dsub_rn(cen[a], __dadd_rn((double)coords[3 * v + a], 0.5));
        res = fmin(fmax(res, -0.5), 0.5);
        f[a] = __ddiv_rn(cen[a], s);
        f[6 + a] = res;
    }
    f[3] = __ddiv_rn(r0, cnt);
    f[4] = __ddiv_rn(r1, cnt);
    f[5] = __ddiv_rn(r2, cnt);
}

template <class K>
static void voxelize_typed(sfb_ctx *ctx, const double *pos, const double *col, int64_t n, double s,
                           const KeyLayout &L, VoxelOut &out) {
    cudaStream_t st = ctx->stream;
    K *keys = ctx->arena.alloc<K>(n), *keys2 = ctx->arena.alloc<K>(n);
    uint32_t *vals = ctx->arena.alloc<uint32_t>(n), *vals2 = ctx->arena.alloc<uint32_t>(n);
    int32_t *flag = ctx->arena.alloc<int32_t>(n), *incl = ctx->arena.alloc<int32_t>(n);
    unsigned g = grid_for(n, 256);
    k_keygen<K><<<g, 256, 0, st>>>(pos, n, s, L, keys, vals);
    SFB_CHECK_LAUNCH();
    size_t tb = 0, tb2 = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tb, keys, keys2, vals, vals2, (int)n, 0, L.total, st);
    cub::DeviceScan::InclusiveSum(nullptr, tb2, flag, incl, (int)n, st);
    void *tmp = ctx->arena.alloc_bytes(tb > tb2 ? tb : tb2);
    SFB_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tb, keys, keys2, vals, vals2, (int)n, 0,
                                             L.total > 0 ? L.total : 1, st));
    k_heads<K><<<g, 256, 0, st>>>(keys2, n, flag);
    SFB_CUDA(cub::DeviceScan::InclusiveSum(tmp, tb2, flag, incl, (int)n, st));
    k_segments<K><<<g, 256, 0, st>>>(keys2, vals2, incl, n, L, out.coords, out.keys, out.p2v,
                                     out.order, out.offsets);
    SFB_CHECK_LAUNCH();
    ctx->read_back(incl + (n - 1), sizeof(int32_t));
    out.m = *reinterpret_cast<int32_t *>(ctx->pinned);
    k_voxel_feats<<<grid_for(out.m, 128), 128, 0, st>>>(pos, col, out.order, out.offsets,
                                                        out.coords, out.m, s, out.feats);
    SFB_CHECK_LAUNCH();
}

void voxelize_run(sfb_ctx *ctx, const double *pos, const double *col, int64_t n, double s,
                  const double *lo_hi, VoxelOut &out) {
    SFB_REQUIRE(n >= 2, "voxelization needs at least 2 points");
    SFB_REQUIRE(n < (int64_t(1) << 31), "at most 2^31-1 points per cloud");
    SFB_REQUIRE(s > 0.0 && s == s, "voxel scale must be positive");
    KeyLayout L{};
    L.total = 0;
    for (int a = 0; a < 3; ++a) {
        // floor(lo*s) .. floor(hi*s) bounds floor(p*s) for every point (monotone rounding)
        int64_t lo = (int64_t)std::floor(lo_hi[a] * s);
        int64_t hi = (int64_t)std::floor(lo_hi[3 + a] * s);
        SFB_REQUIRE(lo > -(int64_t(1) << 20) && hi < (int64_t(1) << 20),
                    "voxel coordinates must satisfy |c| < 1048576");
        L.lo[a] = lo;
        L.bits[a] = bits_for((uint64_t)(hi - lo));
        L.total += L.bits[a];
    }
    if (L.total <= 32) voxelize_typed<uint32_t>(ctx, pos, col, n, s, L, out);
    else voxelize_typed<uint64_t>(ctx, pos, col, n, s, L, out);
}

}  // namespace sfb
