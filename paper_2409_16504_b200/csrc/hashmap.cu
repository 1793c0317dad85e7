// Voxel hashing, sparse-conv kernel maps and 2x2x2 pooling on the device.
//
// Reference: SparseVoxelGrid.lookup (voxelgrid.py:88-94, a searchsorted over
// the sorted key array), _lookup_clipped (sparsenet.py:178-184), the tap
// loops of sparse_conv / transposed_conv_pruned (sparsenet.py:201-207,
// 233-238) and pool_2x2x2 (voxelgrid.py:171-185).
//
// B200 design: an open-addressing table of packed 64-bit keys -> canonical
// row (one CAS insert per voxel, 1-2 probes per lookup, sized to 2x the
// voxel count so it stays L2-resident), kernel maps written tap-major
// (taps x rows, int32) so the gather-GEMM reads them coalesced, and pooling
// as a stable radix sort of compact parent keys + ordered segment means
// (children summed in increasing child row, as np.add.at does).
#include <cub/cub.cuh>

#include "common.cuh"

namespace sfb {

static constexpr unsigned long long kEmpty = ~0ull;

__device__ __forceinline__ uint32_t hash64(unsigned long long k) {
    k ^= k >> 33;
    k *= 0xff51afd7ed558ccdull;
    k ^= k >> 33;
    k *= 0xc4ceb9fe1a85ec53ull;
    k ^= k >> 33;
    return (uint32_t)k;
}

__global__ void k_hash_insert(const int32_t *__restrict__ coords, int64_t m,
                              unsigned long long *__restrict__ keys, int32_t *__restrict__ vals,
                              uint32_t mask) {
    int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (r >= m) return;
    unsigned long long key =
        (unsigned long long)pack_key(coords[3 * r], coords[3 * r + 1], coords[3 * r + 2]);
    uint32_t h = hash64(key) & mask;
    while (true) {
        unsigned long long prev = atomicCAS(&keys[h], kEmpty, key);
        if (prev == kEmpty || prev == key) {
            vals[h] = (int32_t)r;
            return;
        }
        h = (h + 1) & mask;
    }
}

__device__ __forceinline__ int32_t hash_find(const unsigned long long *__restrict__ keys,
                                             const int32_t *__restrict__ vals, uint32_t mask,
                                             int64_t x, int64_t y, int64_t z) {
    if (!key_in_range(x, y, z)) return -1;
    unsigned long long key = (unsigned long long)pack_key(x, y, z);
    uint32_t h = hash64(key) & mask;
    while (true) {
        unsigned long long k = keys[h];
        if (k == key) return vals[h];
        if (k == kEmpty) return -1;
        h = (h + 1) & mask;
    }
}

HashTable hash_build(sfb_ctx *ctx, const int32_t *coords, int64_t m) {
    HashTable h;
    uint64_t cap = 64;
    while (cap < (uint64_t)(2 * m)) cap <<= 1;
    h.mask = (uint32_t)(cap - 1);
    h.keys = ctx->arena.alloc<unsigned long long>(cap);
    h.vals = ctx->arena.alloc<int32_t>(cap);
    SFB_CUDA(cudaMemsetAsync(h.keys, 0xff, cap * sizeof(unsigned long long), ctx->stream));
    if (m > 0) {
        k_hash_insert<<<grid_for(m, 256), 256, 0, ctx->stream>>>(coords, m, h.keys, h.vals, h.mask);
        SFB_CHECK_LAUNCH();
    }
    return h;
}

// map[t*m + r] = row of coords[r] + offset(t)*stride, -1 when empty/out of range
__global__ void k_kernel_map(const int32_t *__restrict__ coords, int64_t m, int stride, int kernel,
                             const unsigned long long *__restrict__ keys,
                             const int32_t *__restrict__ vals, uint32_t mask,
                             int32_t *__restrict__ map) {
    int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    int t = blockIdx.y;
    if (r >= m) return;
    int k2 = kernel * kernel, rad = kernel / 2;
    int a = t / k2, b = (t / kernel) % kernel, c = t % kernel;  // (dz, dy, dx) lexicographic
    int64_t x = coords[3 * r] + (int64_t)(c - rad) * stride;
    int64_t y = coords[3 * r + 1] + (int64_t)(b - rad) * stride;
    int64_t z = coords[3 * r + 2] + (int64_t)(a - rad) * stride;
    map[(int64_t)t * m + r] = hash_find(keys, vals, mask, x, y, z);
}

void kernel_map_build(sfb_ctx *ctx, const HashTable &h, const int32_t *coords, int64_t m,
                      int stride, int kernel, int32_t *map_tap_major) {
    if (m == 0) return;
    int taps = kernel * kernel * kernel;
    dim3 grid(grid_for(m, 128), taps);
    k_kernel_map<<<grid, 128, 0, ctx->stream>>>(coords, m, stride, kernel, h.keys, h.vals, h.mask,
                                                map_tap_major);
    SFB_CHECK_LAUNCH();
}

__global__ void k_transposed_lookup(const int32_t *__restrict__ targets, int64_t m, int ps,
                                    const unsigned long long *__restrict__ keys,
                                    const int32_t *__restrict__ vals, uint32_t mask,
                                    int32_t *__restrict__ parent, int32_t *__restrict__ tap) {
    int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (r >= m) return;
    int64_t t[3], p[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        t[a] = targets[3 * r + a];
        p[a] = floor_div(t[a], ps) * ps;
    }
    int half = ps / 2;
    tap[r] = (int32_t)(((t[2] - p[2]) / half) * 4 + ((t[1] - p[1]) / half) * 2 + (t[0] - p[0]) / half);
    parent[r] = hash_find(keys, vals, mask, p[0], p[1], p[2]);
}

void transposed_lookup(sfb_ctx *ctx, const HashTable &h, int parent_stride,
                       const int32_t *targets, int64_t m, int32_t *parent_out, int32_t *tap_out) {
    if (m == 0) return;
    k_transposed_lookup<<<grid_for(m, 256), 256, 0, ctx->stream>>>(
        targets, m, parent_stride, h.keys, h.vals, h.mask, parent_out, tap_out);
    SFB_CHECK_LAUNCH();
}

// ---------------------------------------------------------------- pooling
struct ParentLayout {
    int64_t lo[3];
    int bits[3];
    int total;
    int64_t step;
};

__global__ void k_int_bbox(const int32_t *__restrict__ c, int64_t m, int *mm) {
    int lo[3] = {INT_MAX, INT_MAX, INT_MAX}, hi[3] = {INT_MIN, INT_MIN, INT_MIN};
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
         i += (int64_t)gridDim.x * blockDim.x)
        for (int a = 0; a < 3; ++a) {
            lo[a] = min(lo[a], c[3 * i + a]);
            hi[a] = max(hi[a], c[3 * i + a]);
        }
    for (int a = 0; a < 3; ++a) {
        atomicMin(&mm[a], lo[a]);
        atomicMax(&mm[3 + a], hi[a]);
    }
}
__global__ void k_int_bbox_init(int *mm) {
    if (threadIdx.x < 3) mm[threadIdx.x] = INT_MAX;
    else if (threadIdx.x < 6) mm[threadIdx.x] = INT_MIN;
}

template <class K>
__global__ void k_parent_keys(const int32_t *__restrict__ coords, int64_t m, ParentLayout L,
                              K *__restrict__ keys, uint32_t *__restrict__ vals) {
    int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (j >= m) return;
    uint64_t q[3];
#pragma unroll
    for (int a = 0; a < 3; ++a)
        q[a] = (uint64_t)((floor_div(coords[3 * j + a], L.step) * L.step - L.lo[a]) / L.step);
    keys[j] = (K)((q[2] << (L.bits[0] + L.bits[1])) | (q[1] << L.bits[0]) | q[0]);
    vals[j] = (uint32_t)j;
}

template <class K>
__global__ void k_flag_heads(const K *__restrict__ k, int64_t n, int32_t *__restrict__ f) {
    int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (j < n) f[j] = (j == 0 || k[j] != k[j - 1]) ? 1 : 0;
}

template <class K>
__global__ void k_pool_segments(const K *__restrict__ keys, const uint32_t *__restrict__ vals,
                                const int32_t *__restrict__ incl, int64_t m, ParentLayout L,
                                int32_t *__restrict__ pcoords, int32_t *__restrict__ seg_start,
                                int32_t *__restrict__ child_to_parent) {
    int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (j >= m) return;
    int32_t v = incl[j] - 1;
    child_to_parent[vals[j]] = v;
    if (j == m - 1) seg_start[v + 1] = (int32_t)m;
    if (j == 0 || incl[j - 1] != incl[j]) {
        uint64_t k = (uint64_t)keys[j];
        int64_t qx = (int64_t)(k & ((1ull << L.bits[0]) - 1));
        int64_t qy = (int64_t)((k >> L.bits[0]) & ((1ull << L.bits[1]) - 1));
        int64_t qz = (int64_t)(k >> (L.bits[0] + L.bits[1]));
        pcoords[3 * v + 0] = (int32_t)(qx * L.step + L.lo[0]);
        pcoords[3 * v + 1] = (int32_t)(qy * L.step + L.lo[1]);
        pcoords[3 * v + 2] = (int32_t)(qz * L.step + L.lo[2]);
        seg_start[v] = (int32_t)j;
    }
}

// thread per (parent, channel): ordered float32 mean of its children
__global__ void k_pool_means(const float *__restrict__ feats, int ld_in, int c,
                             const uint32_t *__restrict__ child_rows,
                             const int32_t *__restrict__ seg_start, int64_t mp,
                             float *__restrict__ out, int ld_out) {
    int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (idx >= mp * c) return;
    int64_t v = idx / c;
    int ch = (int)(idx % c);
    int32_t b = seg_start[v], e = seg_start[v + 1];
    float acc = 0.f;
    for (int32_t j = b; j < e; ++j) acc = __fadd_rn(acc, feats[(int64_t)child_rows[j] * ld_in + ch]);
    out[v * ld_out + ch] = __fdiv_rn(acc, (float)(e - b));
}

template <class K>
static int64_t pool_typed(sfb_ctx *ctx, const int32_t *coords, int64_t m, const ParentLayout &L,
                          const float *feats, int c, int ld_in, int32_t *parent_coords,
                          float *parent_feats, int ld_out, int32_t *child_to_parent) {
    cudaStream_t st = ctx->stream;
    K *keys = ctx->arena.alloc<K>(m), *keys2 = ctx->arena.alloc<K>(m);
    uint32_t *vals = ctx->arena.alloc<uint32_t>(m), *vals2 = ctx->arena.alloc<uint32_t>(m);
    int32_t *flag = ctx->arena.alloc<int32_t>(m), *incl = ctx->arena.alloc<int32_t>(m);
    int32_t *seg = ctx->arena.alloc<int32_t>(m + 1);
    unsigned g = grid_for(m, 256);
    k_parent_keys<K><<<g, 256, 0, st>>>(coords, m, L, keys, vals);
    size_t tb = 0, tb2 = 0;
    int bits = L.total > 0 ? L.total : 1;
    cub::DeviceRadixSort::SortPairs(nullptr, tb, keys, keys2, vals, vals2, (int)m, 0, bits, st);
    cub::DeviceScan::InclusiveSum(nullptr, tb2, flag, incl, (int)m, st);
    void *tmp = ctx->arena.alloc_bytes(tb > tb2 ? tb : tb2);
    SFB_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tb, keys, keys2, vals, vals2, (int)m, 0, bits, st));
    k_flag_heads<K><<<g, 256, 0, st>>>(keys2, m, flag);
    SFB_CUDA(cub::DeviceScan::InclusiveSum(tmp, tb2, flag, incl, (int)m, st));
    k_pool_segments<K><<<g, 256, 0, st>>>(keys2, vals2, incl, m, L, parent_coords, seg,
                                          child_to_parent);
    SFB_CHECK_LAUNCH();
    ctx->read_back(incl + (m - 1), sizeof(int32_t));
    int64_t mp = *reinterpret_cast<int32_t *>(ctx->pinned);
    if (feats && c > 0) {
        k_pool_means<<<grid_for(mp * c, 256), 256, 0, st>>>(feats, ld_in, c, vals2, seg, mp,
                                                            parent_feats, ld_out);
        SFB_CHECK_LAUNCH();
    }
    return mp;
}

int64_t pool_build(sfb_ctx *ctx, const int32_t *coords, int64_t m, int stride, const float *feats,
                   int c, int ld_in, int32_t *parent_coords, float *parent_feats, int ld_out,
                   int32_t *child_to_parent) {
    SFB_REQUIRE(m > 0, "cannot pool an empty grid");
    int *mm = ctx->arena.alloc<int>(6);
    k_int_bbox_init<<<1, 32, 0, ctx->stream>>>(mm);
    k_int_bbox<<<grid_for(m, 256, 256), 256, 0, ctx->stream>>>(coords, m, mm);
    SFB_CHECK_LAUNCH();
    ctx->read_back(mm, 6 * sizeof(int));
    const int *h = reinterpret_cast<const int *>(ctx->pinned);
    ParentLayout L{};
    L.step = 2 * (int64_t)stride;
    L.total = 0;
    for (int a = 0; a < 3; ++a) {
        int64_t lo = floor_div(h[a], L.step) * L.step, hi = floor_div(h[3 + a], L.step) * L.step;
        L.lo[a] = lo;
        L.bits[a] = bits_for((uint64_t)((hi - lo) / L.step));
        L.total += L.bits[a];
    }
    if (L.total <= 32)
        return pool_typed<uint32_t>(ctx, coords, m, L, feats, c, ld_in, parent_coords,
                                    parent_feats, ld_out, child_to_parent);
    return pool_typed<uint64_t>(ctx, coords, m, L, feats, c, ld_in, parent_coords, parent_feats,
                                ld_out, child_to_parent);
}

}  // namespace sfb
