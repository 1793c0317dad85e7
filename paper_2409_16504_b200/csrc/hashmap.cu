// Voxel hashing, sparse-conv kernel maps and 2x2x2 pooling on the device.
//
// Reference: SparseVoxelGrid.lookup (voxelgrid.py:88-94, a searchsorted over
// the sorted key array), _lookup_clipped (sparsenet.py:178-184), the tap
// loops of sparse_conv / transposed_conv_pruned (sparsenet.py:201-207,
// 233-238) and pool_2x2x2 (voxelgrid.py:171-185).
//
// B200 design: an open-addressing table of packed 64-bit keys -> canonical
// row (one CAS insert per voxel, 1-2 probes per lookup, sized on the device
// to 2x the voxel count so it stays L2-resident), kernel maps written
// tap-major (taps x rows, int32) so the gather-GEMM reads them coalesced,
// and pooling as a stable radix sort of compact parent keys + ordered
// segment means (children summed in increasing child row, as np.add.at
// does). Every size is a device count: no host round trip per level.
#include "common.cuh"

namespace sfb {

static constexpr unsigned long long kEmpty = ~0ull;
// level-0 voxel table capacity >= kHashSpread x rows (power of two): most
// kernel-map lookups are misses, and a linear-probing miss costs
// (1 + 1/(1-a)^2)/2 probes at load a (A/B on config 2: 4x gives 0.286 vs
// 0.290 ms/frame and 0.779 vs 0.787 ms latency against 2x)
static constexpr int kHashSpread = 4;

__device__ __forceinline__ uint32_t hash64(unsigned long long k) {
    k ^= k >> 33;
    k *= 0xff51afd7ed558ccdull;
    k ^= k >> 33;
    k *= 0xc4ceb9fe1a85ec53ull;
    k ^= k >> 33;
    return (uint32_t)k;
}

__global__ void k_hash_clear(HashTable h, const int64_t *__restrict__ d_m, int64_t m_fixed) {
    const int64_t m = d_m ? *d_m : m_fixed;
    uint64_t cap = 64;
    while (cap < (uint64_t)(kHashSpread * m)) cap <<= 1;
    if (blockIdx.x == 0 && threadIdx.x == 0) *h.mask = (uint32_t)(cap - 1);
    SFB_FOR(i, (int64_t)cap) h.keys[i] = kEmpty;
}

__global__ void k_hash_insert(const int32_t *__restrict__ coords, const int64_t *__restrict__ d_m,
                              int64_t m_fixed, HashTable h) {
    const int64_t m = d_m ? *d_m : m_fixed;
    const uint32_t mask = *h.mask;
    SFB_FOR(r, m) {
        unsigned long long key =
            (unsigned long long)pack_key(coords[3 * r], coords[3 * r + 1], coords[3 * r + 2]);
        uint32_t slot = hash64(key) & mask;
        while (true) {
            unsigned long long prev = atomicCAS(&h.keys[slot], kEmpty, key);
            if (prev == kEmpty || prev == key) {
                h.vals[slot] = (int32_t)r;
                break;
            }
            slot = (slot + 1) & mask;
        }
    }
}

__device__ __forceinline__ int32_t hash_find(const HashTable &h, uint32_t mask, int64_t x, int64_t y,
                                             int64_t z) {
    if (!key_in_range(x, y, z)) return -1;
    unsigned long long key = (unsigned long long)pack_key(x, y, z);
    uint32_t slot = hash64(key) & mask;
    while (true) {
        unsigned long long k = h.keys[slot];
        if (k == key) return h.vals[slot];
        if (k == kEmpty) return -1;
        slot = (slot + 1) & mask;
    }
}

HashTable hash_build(sfb_ctx *ctx, const int32_t *coords, const int64_t *d_m, int64_t m_bound,
                     int64_t m_grid) {
    if (m_grid < 0) m_grid = m_bound;
    HashTable h;
    uint64_t cap = 64, capg = 64;
    while (cap < (uint64_t)(kHashSpread * m_bound)) cap <<= 1;
    while (capg < (uint64_t)(kHashSpread * m_grid)) capg <<= 1;
    h.keys = ctx->arena.alloc<unsigned long long>(cap);
    h.vals = ctx->arena.alloc<int32_t>(cap);
    h.mask = ctx->arena.alloc<uint32_t>(1);
    k_hash_clear<<<dgrid((int64_t)capg, 256), 256, 0, ctx->stream>>>(h, d_m, m_bound);
    k_hash_insert<<<dgrid(m_grid, 256), 256, 0, ctx->stream>>>(coords, d_m, m_bound, h);
    SFB_CHECK_LAUNCH();
    return h;
}

// map[t*m_cap + r] = row of coords[r] + offset(t)*stride, -1 when empty/out of range
__global__ void k_kernel_map(const int32_t *__restrict__ coords, const int64_t *__restrict__ d_m,
                             int64_t m_fixed, int64_t ld, int stride, int kernel, HashTable h,
                             int32_t *__restrict__ map) {
    const int64_t m = d_m ? *d_m : m_fixed;
    const uint32_t mask = *h.mask;
    const int taps = kernel * kernel * kernel, k2 = kernel * kernel, rad = kernel / 2;
    const bool narrow = m * taps < (int64_t(1) << 31);   // 32-bit index arithmetic (the usual case)
    SFB_FOR(idx, m * taps) {
        int64_t r;
        int t;
        if (narrow) {   // 32-bit division: a 64-bit one is ~4x the instructions
            const uint32_t i32 = (uint32_t)idx, m32 = (uint32_t)m;
            t = (int)(i32 / m32);
            r = (int64_t)(i32 - (uint32_t)t * m32);
        } else {
            r = idx % m;
            t = (int)(idx / m);
        }
        const int a = t / k2, b = (t / kernel) % kernel, c = t % kernel;  // (dz, dy, dx)
        const int64_t x = coords[3 * r] + (int64_t)(c - rad) * stride;
        const int64_t y = coords[3 * r + 1] + (int64_t)(b - rad) * stride;
        const int64_t z = coords[3 * r + 2] + (int64_t)(a - rad) * stride;
        map[(int64_t)t * ld + r] = hash_find(h, mask, x, y, z);
    }
}

void kernel_map_build(sfb_ctx *ctx, const HashTable &h, const int32_t *coords, const int64_t *d_m,
                      int64_t m_bound, int stride, int kernel, int32_t *map_tap_major,
                      int64_t m_grid) {
    if (m_grid < 0) m_grid = m_bound;
    const int taps = kernel * kernel * kernel;
    k_kernel_map<<<dgrid(m_grid * taps, 256), 256, 0, ctx->stream>>>(
        coords, d_m, m_bound, m_bound, stride, kernel, h, map_tap_major);
    SFB_CHECK_LAUNCH();
}

__global__ void k_transposed_lookup(const int32_t *__restrict__ targets,
                                    const int64_t *__restrict__ d_m, int64_t m_fixed, int ps,
                                    HashTable h, int32_t *__restrict__ parent,
                                    int32_t *__restrict__ tap) {
    const int64_t m = d_m ? *d_m : m_fixed;
    const uint32_t mask = *h.mask;
    SFB_FOR(r, m) {
        int64_t t[3], p[3];
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            t[a] = targets[3 * r + a];
            p[a] = floor_div(t[a], ps) * ps;
        }
        const int half = ps / 2;
        tap[r] = (int32_t)(floor_div(t[2] - p[2], half) * 4 + floor_div(t[1] - p[1], half) * 2 +
                           floor_div(t[0] - p[0], half));
        parent[r] = hash_find(h, mask, p[0], p[1], p[2]);
    }
}

void transposed_lookup(sfb_ctx *ctx, const HashTable &h, int parent_stride,
                       const int32_t *targets, const int64_t *d_m, int64_t m_bound,
                       int32_t *parent_out, int32_t *tap_out) {
    k_transposed_lookup<<<dgrid(m_bound, 256), 256, 0, ctx->stream>>>(
        targets, d_m, m_bound, parent_stride, h, parent_out, tap_out);
    SFB_CHECK_LAUNCH();
}

// ---------------------------------------------------------------- pooling
// parent layout at step S from the level-0 key layout: the lattice of every
// level lies inside [lo, lo + 2^bits - 1] per axis
__device__ __forceinline__ void parent_layout(const FrameParams *P, int64_t S, int64_t *plo,
                                              int *pbits) {
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        const int64_t lo = P->lo[a], hi = lo + ((int64_t)1 << P->bits[a]) - 1;
        plo[a] = floor_div(lo, S) * S;
        const int64_t span = floor_div(floor_div(hi, S) * S - plo[a], S);
        int b = 0;
        while (b < 63 && (span >> b) != 0) ++b;
        pbits[a] = b;
    }
}

template <class K>
__global__ void k_parent_keys(const int32_t *__restrict__ coords, const int64_t *__restrict__ d_m,
                              int64_t S, const FrameParams *__restrict__ P, K *__restrict__ keys,
                              uint32_t *__restrict__ vals) {
    int64_t plo[3];
    int pb[3];
    parent_layout(P, S, plo, pb);
    const int64_t m = *d_m;
    SFB_FOR(j, m) {
        uint64_t q[3];
#pragma unroll
        for (int a = 0; a < 3; ++a) q[a] = (uint64_t)floor_div(floor_div(coords[3 * j + a], S) * S - plo[a], S);
        keys[j] = (K)((q[2] << (pb[0] + pb[1])) | (q[1] << pb[0]) | q[0]);
        vals[j] = (uint32_t)j;
    }
}

template <class K>
__global__ void k_flag_heads(const K *__restrict__ k, const int64_t *__restrict__ d_n,
                             int32_t *__restrict__ f) {
    const int64_t n = *d_n;
    SFB_FOR(j, n) f[j] = (j == 0 || k[j] != k[j - 1]) ? 1 : 0;
}

template <class K>
__global__ void k_pool_segments(const K *__restrict__ keys, const uint32_t *__restrict__ vals,
                                const int32_t *__restrict__ incl, const int64_t *__restrict__ d_m,
                                int64_t S, const FrameParams *__restrict__ P,
                                int32_t *__restrict__ pcoords, int32_t *__restrict__ seg_start,
                                int32_t *__restrict__ child_to_parent, int64_t *__restrict__ d_mp) {
    int64_t plo[3];
    int pb[3];
    parent_layout(P, S, plo, pb);
    const int64_t m = *d_m;
    SFB_FOR(j, m) {
        const int32_t v = incl[j] - 1;
        child_to_parent[vals[j]] = v;
        if (j == m - 1) {
            seg_start[v + 1] = (int32_t)m;
            *d_mp = v + 1;
        }
        if (j == 0 || incl[j - 1] != incl[j]) {
            const uint64_t k = (uint64_t)keys[j];
            const int64_t qx = (int64_t)(k & ((1ull << pb[0]) - 1));
            const int64_t qy = (int64_t)((k >> pb[0]) & ((1ull << pb[1]) - 1));
            const int64_t qz = (int64_t)(k >> (pb[0] + pb[1]));
            pcoords[3 * v + 0] = (int32_t)(qx * S + plo[0]);
            pcoords[3 * v + 1] = (int32_t)(qy * S + plo[1]);
            pcoords[3 * v + 2] = (int32_t)(qz * S + plo[2]);
            seg_start[v] = (int32_t)j;
        }
    }
}

// thread per (parent, channel): ordered mean of its children in child-row
// order (np.add.at, voxelgrid.py:181-183), float32 in the network, float64
// through the pool_2x2x2 API
template <class T>
__global__ void k_pool_means(const T *__restrict__ feats, int ld_in, int c,
                             const uint32_t *__restrict__ child_rows,
                             const int32_t *__restrict__ seg_start, const int64_t *__restrict__ d_mp,
                             T *__restrict__ out, int ld_out) {
    const int64_t mp = *d_mp;
    SFB_FOR(idx, mp * c) {
        const int64_t v = idx / c;
        const int ch = (int)(idx % c);
        const int32_t b = seg_start[v], e = seg_start[v + 1];
        T acc = T(0);
        for (int32_t j = b; j < e; ++j) acc = acc + feats[(int64_t)child_rows[j] * ld_in + ch];
        out[v * ld_out + ch] = acc / (T)(e - b);
    }
}

template <class K, class T>
static void pool_typed(sfb_ctx *ctx, const int32_t *coords, const int64_t *d_m, int64_t m_bound,
                       int stride, const FrameParams *P, int key_bits, const T *feats, int c,
                       int ld_in, int32_t *parent_coords, T *parent_feats, int ld_out,
                       int32_t *child_to_parent, int64_t *d_mp) {
    cudaStream_t st = ctx->stream;
    const int64_t S = 2 * (int64_t)stride;
    K *keys = ctx->arena.alloc<K>(m_bound), *keys2 = ctx->arena.alloc<K>(m_bound);
    uint32_t *vals = ctx->arena.alloc<uint32_t>(m_bound), *vals2 = ctx->arena.alloc<uint32_t>(m_bound);
    int32_t *flag = ctx->arena.alloc<int32_t>(m_bound);
    int32_t *seg = ctx->arena.alloc<int32_t>(m_bound + 1);
    const unsigned g = dgrid(m_bound, 256);
    k_parent_keys<K><<<g, 256, 0, st>>>(coords, d_m, S, P, keys, vals);
    SFB_CHECK_LAUNCH();
    const int which = dsort_pairs<K>(ctx, keys, vals, keys2, vals2, d_m, m_bound, key_bits);
    K *ks = which ? keys2 : keys;
    uint32_t *vs = which ? vals2 : vals;
    k_flag_heads<K><<<g, 256, 0, st>>>(ks, d_m, flag);
    dscan(ctx, flag, flag, d_m, m_bound, nullptr, true);
    k_pool_segments<K><<<g, 256, 0, st>>>(ks, vs, flag, d_m, S, P, parent_coords, seg,
                                          child_to_parent, d_mp);
    SFB_CHECK_LAUNCH();
    if (feats && c > 0) {
        k_pool_means<T><<<dgrid(m_bound * c, 256), 256, 0, st>>>(feats, ld_in, c, vs, seg, d_mp,
                                                                  parent_feats, ld_out);
        SFB_CHECK_LAUNCH();
    }
}

template <class T>
static void pool_build_t(sfb_ctx *ctx, const int32_t *coords, const int64_t *d_m, int64_t m_bound,
                         int stride, const FrameParams &host, const FrameParams *P, const T *feats,
                         int c, int ld_in, int32_t *parent_coords, T *parent_feats, int ld_out,
                         int32_t *child_to_parent, int64_t *d_mp) {
    const int bits = host.total > 0 ? host.total : 1;
    if (host.total <= 32)
        pool_typed<uint32_t, T>(ctx, coords, d_m, m_bound, stride, P, bits, feats, c, ld_in,
                                parent_coords, parent_feats, ld_out, child_to_parent, d_mp);
    else
        pool_typed<unsigned long long, T>(ctx, coords, d_m, m_bound, stride, P, bits, feats, c, ld_in,
                                          parent_coords, parent_feats, ld_out, child_to_parent, d_mp);
}

void pool_build(sfb_ctx *ctx, const int32_t *coords, const int64_t *d_m, int64_t m_bound,
                int stride, const FrameParams &host, const FrameParams *P, const float *feats,
                int c, int ld_in, int32_t *parent_coords, float *parent_feats, int ld_out,
                int32_t *child_to_parent, int64_t *d_mp) {
    pool_build_t<float>(ctx, coords, d_m, m_bound, stride, host, P, feats, c, ld_in, parent_coords,
                        parent_feats, ld_out, child_to_parent, d_mp);
}

void pool_build(sfb_ctx *ctx, const int32_t *coords, const int64_t *d_m, int64_t m_bound,
                int stride, const FrameParams &host, const FrameParams *P, const double *feats,
                int c, int ld_in, int32_t *parent_coords, double *parent_feats, int ld_out,
                int32_t *child_to_parent, int64_t *d_mp) {
    pool_build_t<double>(ctx, coords, d_m, m_bound, stride, host, P, feats, c, ld_in, parent_coords,
                         parent_feats, ld_out, child_to_parent, d_mp);
}

// ---------------------------------------------------------------- lookup
// SparseVoxelGrid.lookup (voxelgrid.py:88-94): row of each query coordinate
// in the grid's canonical order, -1 where unoccupied (hash probe instead of
// searchsorted; identical result since rows are unique)
__global__ void k_lookup(const int32_t *__restrict__ q, int64_t nq, HashTable h,
                         int64_t *__restrict__ rows) {
    const uint32_t mask = *h.mask;
    SFB_FOR(i, nq) rows[i] = hash_find(h, mask, q[3 * i], q[3 * i + 1], q[3 * i + 2]);
}

void lookup_run(sfb_ctx *ctx, const int32_t *coords, int64_t m, const int32_t *query, int64_t nq,
                int64_t *rows) {
    if (nq == 0) return;
    if (m == 0) {
        SFB_CUDA(cudaMemsetAsync(rows, 0xff, sizeof(int64_t) * nq, ctx->stream));
        return;
    }
    HashTable h = hash_build(ctx, coords, nullptr, m);
    k_lookup<<<dgrid(nq, 256), 256, 0, ctx->stream>>>(query, nq, h, rows);
    SFB_CHECK_LAUNCH();
}

// ---------------------------------------------------------------- fast pooling
// Pooling inside the fused UNet does not need canonical parent order: every
// conv output row depends only on its own neighbourhood, so parents are
// numbered in order of their first child (deterministic, no sort). Each
// parent still averages its children in increasing child row, like
// np.add.at (the <= 8 children are sorted in-register before summing).
__global__ void k_pool_clear(unsigned long long *__restrict__ keys, int32_t *__restrict__ minrow,
                             int32_t *__restrict__ nkids, uint32_t *__restrict__ mask,
                             const int64_t *__restrict__ d_m) {
    const int64_t m = *d_m;
    uint64_t cap = 64;
    while (cap < (uint64_t)(2 * m)) cap <<= 1;
    if (blockIdx.x == 0 && threadIdx.x == 0) *mask = (uint32_t)(cap - 1);
    SFB_FOR(i, (int64_t)cap) {
        keys[i] = kEmpty;
        minrow[i] = INT_MAX;
    }
    SFB_FOR(i, m) nkids[i] = 0;
}

__global__ void k_pool_insert(const int32_t *__restrict__ coords, const int64_t *__restrict__ d_m,
                              int64_t S, unsigned long long *__restrict__ keys,
                              int32_t *__restrict__ minrow, const uint32_t *__restrict__ d_mask,
                              int32_t *__restrict__ slot_of) {
    const int64_t m = *d_m;
    const uint32_t mask = *d_mask;
    SFB_FOR(j, m) {
        const int64_t px = floor_div(coords[3 * j], S) * S, py = floor_div(coords[3 * j + 1], S) * S,
                      pz = floor_div(coords[3 * j + 2], S) * S;
        const unsigned long long key = (unsigned long long)pack_key(px, py, pz);
        uint32_t slot = hash64(key) & mask;
        while (true) {
            const unsigned long long prev = atomicCAS(&keys[slot], kEmpty, key);
            if (prev == kEmpty || prev == key) break;
            slot = (slot + 1) & mask;
        }
        atomicMin(&minrow[slot], (int32_t)j);
        slot_of[j] = (int32_t)slot;
    }
}

__global__ void k_pool_first(const int32_t *__restrict__ slot_of, const int32_t *__restrict__ minrow,
                             const int64_t *__restrict__ d_m, int32_t *__restrict__ flag) {
    const int64_t m = *d_m;
    SFB_FOR(j, m) flag[j] = minrow[slot_of[j]] == (int32_t)j;
}

// child -> parent row, parent coords, children lists; optionally the child's
// tap under its parent (dz*4+dy*2+dx, sparsenet.py:236) and the parent row in
// the table's value slots (the table then IS the parent level's voxel hash)
__global__ void k_pool_assign(const int32_t *__restrict__ coords, const int32_t *__restrict__ slot_of,
                              const int32_t *__restrict__ minrow, const int32_t *__restrict__ pid_of_first,
                              const int64_t *__restrict__ d_m, int64_t S, int32_t *__restrict__ pcoords,
                              int32_t *__restrict__ c2p, int32_t *__restrict__ nkids,
                              int32_t *__restrict__ kids, int32_t *__restrict__ tap,
                              int32_t *__restrict__ vals, int32_t *__restrict__ tmap, int64_t ld,
                              int32_t *__restrict__ tap_cnt) {
    const int64_t m = *d_m;
    const int64_t cs = S / 2;
    SFB_FOR(j, m) {
        const int32_t slot = slot_of[j];
        const int32_t first = minrow[slot];
        const int32_t pid = pid_of_first[first];
        c2p[j] = pid;
        int64_t d[3];
        for (int a = 0; a < 3; ++a) {
            const int64_t c = coords[3 * j + a], pc = floor_div(c, S) * S;
            d[a] = (c - pc) / cs;
            if (first == (int32_t)j) pcoords[3 * pid + a] = (int32_t)pc;
        }
        const int32_t tj = (int32_t)(d[2] * 4 + d[1] * 2 + d[0]);
        if (tap) tap[j] = tj;
        if (tap_cnt) atomicAdd(&tap_cnt[tj], 1);
        if (tmap)
#pragma unroll
            for (int k = 0; k < 8; ++k) tmap[k * ld + j] = (k == tj) ? pid : -1;
        if (vals && first == (int32_t)j) vals[slot] = pid;
        const int32_t k = atomicAdd(&nkids[pid], 1);
        if (k < 8) kids[8 * (int64_t)pid + k] = (int32_t)j;
    }
}

__global__ void k_pool_means_fast(const float *__restrict__ feats, int ld_in, int c,
                                  const int32_t *__restrict__ nkids, const int32_t *__restrict__ kids,
                                  const int64_t *__restrict__ d_mp, float *__restrict__ out,
                                  int ld_out) {
    const int64_t mp = *d_mp;
    SFB_FOR(idx, mp * c) {
        // channel counts are small: 32-bit quotient when the index fits
        const int64_t v = idx < (int64_t(1) << 31) ? (int64_t)((uint32_t)idx / (uint32_t)c) : idx / c;
        const int ch = (int)(idx - v * c);
        const int cnt = min(nkids[v], 8);
        // all 8 slots loaded at once (absent ones padded past any row), sorted
        // by a fixed compare-exchange network (registers, no local memory),
        // then every child's row gathered at once: one round trip per step
        // instead of one per child
        int32_t kk[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) kk[q] = q < cnt ? kids[8 * v + q] : INT32_MAX;
        auto cx = [&](int a, int b) {
            const int32_t lo = min(kk[a], kk[b]), hi = max(kk[a], kk[b]);
            kk[a] = lo;
            kk[b] = hi;
        };
        // Batcher's odd-even merge sort for 8 (19 exchanges): ascending child rows
        cx(0, 1); cx(2, 3); cx(4, 5); cx(6, 7);
        cx(0, 2); cx(1, 3); cx(4, 6); cx(5, 7);
        cx(1, 2); cx(5, 6);
        cx(0, 4); cx(1, 5); cx(2, 6); cx(3, 7);
        cx(2, 4); cx(3, 5);
        cx(1, 2); cx(3, 4); cx(5, 6);
        float f[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) f[q] = q < cnt ? feats[(int64_t)kk[q] * ld_in + ch] : 0.f;
        float acc = 0.f;
#pragma unroll
        for (int q = 0; q < 8; ++q)
            if (q < cnt) acc = __fadd_rn(acc, f[q]);
        out[v * ld_out + ch] = __fdiv_rn(acc, (float)cnt);
    }
}

void pool_fast(sfb_ctx *ctx, const int32_t *coords, const int64_t *d_m, int64_t m_bound,
               int64_t m_grid, int stride, const float *feats, int c, int ld_in,
               int32_t *parent_coords, float *parent_feats, int ld_out, int32_t *child_to_parent,
               int64_t *d_mp) {
    cudaStream_t st = ctx->stream;
    const int64_t S = 2 * (int64_t)stride;
    uint64_t cap = 64;
    while (cap < (uint64_t)(2 * m_bound)) cap <<= 1;
    uint64_t cap_grid = 64;
    while (cap_grid < (uint64_t)(2 * m_grid)) cap_grid <<= 1;
    auto *keys = ctx->arena.alloc<unsigned long long>(cap);
    int32_t *minrow = ctx->arena.alloc<int32_t>(cap);
    uint32_t *mask = ctx->arena.alloc<uint32_t>(1);
    int32_t *slot_of = ctx->arena.alloc<int32_t>(m_bound);
    int32_t *flag = ctx->arena.alloc<int32_t>(m_bound);
    int32_t *nkids = ctx->arena.alloc<int32_t>(m_bound);
    int32_t *kids = ctx->arena.alloc<int32_t>(8 * m_bound);
    const unsigned g = dgrid(m_grid, 256);
    k_pool_clear<<<dgrid((int64_t)cap_grid, 256), 256, 0, st>>>(keys, minrow, nkids, mask, d_m);
    k_pool_insert<<<g, 256, 0, st>>>(coords, d_m, S, keys, minrow, mask, slot_of);
    k_pool_first<<<g, 256, 0, st>>>(slot_of, minrow, d_m, flag);
    SFB_CHECK_LAUNCH();
    dscan(ctx, flag, flag, d_m, m_bound, d_mp, false);
    k_pool_assign<<<g, 256, 0, st>>>(coords, slot_of, minrow, flag, d_m, S, parent_coords,
                                     child_to_parent, nkids, kids, nullptr, nullptr, nullptr, 0,
                                     nullptr);
    k_pool_means_fast<<<dgrid(m_grid * c, 256), 256, 0, st>>>(feats, ld_in, c, nkids, kids, d_mp,
                                                              parent_feats, ld_out);
    SFB_CHECK_LAUNCH();
}

// children grouped by tap for the transposed conv (bucket order within a tap
// is arbitrary — each output row depends only on its own parent and tap)
// per-tap counts come from k_pool_assign; every thread forms the padded
// bucket offsets from the 8 counts, block 0 publishes them
__global__ void k_tap_scatter(const int32_t *__restrict__ tap, const int32_t *__restrict__ c2p,
                              const int64_t *__restrict__ d_m, const int32_t *__restrict__ cnt,
                              int32_t *__restrict__ cur, int32_t *__restrict__ off,
                              int64_t *__restrict__ d_rows, int32_t *__restrict__ perm,
                              int32_t *__restrict__ src) {
    const int64_t m = *d_m;
    int32_t o[9];
    o[0] = 0;
#pragma unroll
    for (int t = 0; t < 8; ++t) o[t + 1] = o[t] + (cnt[t] + 127) / 128 * 128;
    if (blockIdx.x == 0 && threadIdx.x < 9) {
        off[threadIdx.x] = o[threadIdx.x];
        if (threadIdx.x == 8) *d_rows = o[8];
    }
    const int lane = threadIdx.x & 31;
    SFB_FOR(j, m) {
        // one atomic per (warp, tap): the 8 bucket cursors are hot
        const int32_t t = tap[j];
        const unsigned act = __activemask();
        const unsigned peers = __match_any_sync(act, t);
        const int leader = __ffs(peers) - 1;
        int32_t b = 0;
        if (lane == leader) b = atomicAdd(&cur[t], __popc(peers));
        b = __shfl_sync(peers, b, leader);
        const int32_t pos = o[t] + b + __popc(peers & ((1u << lane) - 1u));
        perm[pos] = (int32_t)j;
        src[pos] = c2p[j];
    }
}

// The fused UNet splits pooling in two: the coordinate structure (parents,
// children lists, child taps, the parent level's hash table) depends only on
// coordinates and runs on a side stream ahead of the convolutions; the means
// need the level's conv output and stay on the critical path.
PoolStructure pool_structure(sfb_ctx *ctx, const int32_t *coords, const int64_t *d_m,
                             int64_t m_bound, int64_t m_grid, int stride, int32_t *parent_coords,
                             int64_t *d_mp) {
    cudaStream_t st = ctx->stream;
    PoolStructure P;
    const int64_t S = 2 * (int64_t)stride;
    uint64_t cap = 64;
    while (cap < (uint64_t)(2 * m_bound)) cap <<= 1;
    uint64_t cap_grid = 64;
    while (cap_grid < (uint64_t)(2 * m_grid)) cap_grid <<= 1;
    P.table.keys = ctx->arena.alloc<unsigned long long>(cap);
    P.table.vals = ctx->arena.alloc<int32_t>(cap);
    P.table.mask = ctx->arena.alloc<uint32_t>(1);
    int32_t *minrow = ctx->arena.alloc<int32_t>(cap);
    int32_t *slot_of = ctx->arena.alloc<int32_t>(m_bound);
    int32_t *flag = ctx->arena.alloc<int32_t>(m_bound);
    P.nkids = ctx->arena.alloc<int32_t>(m_bound);
    P.kids = ctx->arena.alloc<int32_t>(8 * m_bound);
    P.c2p = ctx->arena.alloc<int32_t>(m_bound);
    P.tap = ctx->arena.alloc<int32_t>(m_bound);
    P.tmap = nullptr;   // the fused UNet uses the tap buckets instead
    const unsigned g = dgrid(m_grid, 256);
    k_pool_clear<<<dgrid((int64_t)cap_grid, 256), 256, 0, st>>>(P.table.keys, minrow, P.nkids,
                                                                P.table.mask, d_m);
    k_pool_insert<<<g, 256, 0, st>>>(coords, d_m, S, P.table.keys, minrow, P.table.mask, slot_of);
    k_pool_first<<<g, 256, 0, st>>>(slot_of, minrow, d_m, flag);
    SFB_CHECK_LAUNCH();
    dscan(ctx, flag, flag, d_m, m_bound, d_mp, false);
    // tap buckets for the transposed conv of this level (counts by k_pool_assign)
    TapBuckets &B = P.buckets;
    int32_t *cnt = ctx->arena.alloc<int32_t>(32);   // counts, cursors, offsets
    SFB_CUDA(cudaMemsetAsync(cnt, 0, 16 * sizeof(int32_t), st));
    k_pool_assign<<<g, 256, 0, st>>>(coords, slot_of, minrow, flag, d_m, S, parent_coords, P.c2p,
                                     P.nkids, P.kids, P.tap, P.table.vals, P.tmap, m_bound, cnt);
    SFB_CHECK_LAUNCH();
    B.rows_bound = m_bound + 8 * 128;
    B.rows_grid = m_grid + 8 * 128;
    B.perm = ctx->arena.alloc<int32_t>(B.rows_bound);
    B.src = ctx->arena.alloc<int32_t>(B.rows_bound);
    B.off = cnt + 16;
    B.d_rows = ctx->arena.alloc<int64_t>(1);
    SFB_CUDA(cudaMemsetAsync(B.perm, 0xff, sizeof(int32_t) * B.rows_bound, st));
    SFB_CUDA(cudaMemsetAsync(B.src, 0xff, sizeof(int32_t) * B.rows_bound, st));
    k_tap_scatter<<<g, 256, 0, st>>>(P.tap, P.c2p, d_m, cnt, cnt + 8, B.off, B.d_rows, B.perm, B.src);
    SFB_CHECK_LAUNCH();
    return P;
}

void pool_means(sfb_ctx *ctx, const PoolStructure &P, const int64_t *d_mp, int64_t mp_grid,
                const float *feats, int c, int ld_in, float *parent_feats, int ld_out) {
    k_pool_means_fast<<<dgrid(mp_grid * c, 256), 256, 0, ctx->stream>>>(
        feats, ld_in, c, P.nkids, P.kids, d_mp, parent_feats, ld_out);
    SFB_CHECK_LAUNCH();
}

// Key layout of an arbitrary coordinate set (standalone pool API): one
// reduction + read-back, then the same layout type the frame uses.
__global__ void k_int_bbox_init(int *mm) {
    if (threadIdx.x < 3) mm[threadIdx.x] = INT_MAX;
    else if (threadIdx.x < 6) mm[threadIdx.x] = INT_MIN;
}
__global__ void k_int_bbox(const int32_t *__restrict__ c, int64_t m, int *mm) {
    int lo[3] = {INT_MAX, INT_MAX, INT_MAX}, hi[3] = {INT_MIN, INT_MIN, INT_MIN};
    SFB_FOR(i, m)
    for (int a = 0; a < 3; ++a) {
        lo[a] = min(lo[a], c[3 * i + a]);
        hi[a] = max(hi[a], c[3 * i + a]);
    }
    for (int a = 0; a < 3; ++a) {
        atomicMin(&mm[a], lo[a]);
        atomicMax(&mm[3 + a], hi[a]);
    }
}

void coords_layout(sfb_ctx *ctx, const int32_t *coords, int64_t m, FrameParams &P) {
    SFB_REQUIRE(m > 0, "cannot pool an empty grid");
    int *mm = ctx->arena.alloc<int>(6);
    k_int_bbox_init<<<1, 32, 0, ctx->stream>>>(mm);
    k_int_bbox<<<dgrid(m, 256, 2), 256, 0, ctx->stream>>>(coords, m, mm);
    SFB_CHECK_LAUNCH();
    ctx->read_back(mm, 6 * sizeof(int));
    const int *h = reinterpret_cast<const int *>(ctx->pinned);
    P = FrameParams{};
    P.total = 0;
    for (int a = 0; a < 3; ++a) {
        P.lo[a] = h[a];
        P.hi[a] = h[3 + a];
        P.bits[a] = bits_for((uint64_t)((int64_t)h[3 + a] - h[a]));
        P.total += P.bits[a];
    }
    P.total += 3;  // parent ranges may need one more bit per axis
}

}  // namespace sfb
