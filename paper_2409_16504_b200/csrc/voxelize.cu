// Density-1 voxelization on the device (reference: voxelgrid.py:125-168).
//
//   bbox reduce -> (host) s -> keygen: floor(p*s) packed into a compact
//   (z,y,x)-ordered key of only the bits the cloud needs -> stable LSD radix
//   sort of (key, point index) -> run-length segmentation -> per-voxel ordered
//   float64 sums (bit-identical to np.add.at, which walks points in increasing
//   index) -> 9 feature channels.
// HBM-bound integer/byte work; no tensor cores.
#include "common.cuh"
#include "scan.cuh"

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

// Flat, coalesced grid-stride pass over the (n,3) array; the total thread
// count is a multiple of 3 so each thread always sees the same axis. Shared
// atomics combine a block, then one global atomic per value per block.
constexpr int kBBoxThreads = 192;
__global__ void __launch_bounds__(kBBoxThreads) k_bbox(const double *__restrict__ pos, int64_t n,
                                                       unsigned long long *mm) {
    __shared__ unsigned long long s_mm[6];
    if (threadIdx.x < 3) s_mm[threadIdx.x] = ~0ull;
    else if (threadIdx.x < 6) s_mm[threadIdx.x] = 0ull;
    __syncthreads();
    const int64_t total = 3 * n;
    const int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int axis = (int)(g % 3);
    unsigned long long lo = ~0ull, hi = 0ull;
    for (int64_t j = g; j < total; j += stride) {
        unsigned long long u = ord_bits(pos[j]);
        lo = u < lo ? u : lo;
        hi = u > hi ? u : hi;
    }
    atomicMin(&s_mm[axis], lo);
    atomicMax(&s_mm[3 + axis], hi);
    __syncthreads();
    if (threadIdx.x < 3) atomicMin(&mm[threadIdx.x], s_mm[threadIdx.x]);
    else if (threadIdx.x < 6) atomicMax(&mm[threadIdx.x], s_mm[threadIdx.x]);
}

// 16-byte variant for an aligned array: element j of the double2 view holds
// doubles 2j, 2j+1, i.e. axes (2j) % 3 and (2j+1) % 3; with a thread stride
// that is a multiple of 3, each thread always sees the same axis pair.
// Four loads in flight per thread.
__global__ void __launch_bounds__(kBBoxThreads) k_bbox2(const double2 *__restrict__ pos2, int64_t n,
                                                        unsigned long long *mm) {
    __shared__ unsigned long long s_mm[6];
    if (threadIdx.x < 3) s_mm[threadIdx.x] = ~0ull;
    else if (threadIdx.x < 6) s_mm[threadIdx.x] = 0ull;
    __syncthreads();
    const int64_t total = 3 * n, total2 = total / 2;
    const int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int a0 = (int)((2 * g) % 3), a1 = (int)((2 * g + 1) % 3);
    unsigned long long lo0 = ~0ull, hi0 = 0ull, lo1 = ~0ull, hi1 = 0ull;
    int64_t j = g;
    for (; j + 3 * stride < total2; j += 4 * stride) {
        double2 v[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) v[q] = pos2[j + q * stride];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const unsigned long long u0 = ord_bits(v[q].x), u1 = ord_bits(v[q].y);
            lo0 = u0 < lo0 ? u0 : lo0;
            hi0 = u0 > hi0 ? u0 : hi0;
            lo1 = u1 < lo1 ? u1 : lo1;
            hi1 = u1 > hi1 ? u1 : hi1;
        }
    }
    for (; j < total2; j += stride) {
        const double2 v = pos2[j];
        const unsigned long long u0 = ord_bits(v.x), u1 = ord_bits(v.y);
        lo0 = u0 < lo0 ? u0 : lo0;
        hi0 = u0 > hi0 ? u0 : hi0;
        lo1 = u1 < lo1 ? u1 : lo1;
        hi1 = u1 > hi1 ? u1 : hi1;
    }
    if (g == 0 && (total & 1)) {   // the last double (axis 2) when 3n is odd
        const unsigned long long u = ord_bits(reinterpret_cast<const double *>(pos2)[total - 1]);
        atomicMin(&s_mm[2], u);
        atomicMax(&s_mm[5], u);
    }
    atomicMin(&s_mm[a0], lo0);
    atomicMax(&s_mm[3 + a0], hi0);
    atomicMin(&s_mm[a1], lo1);
    atomicMax(&s_mm[3 + a1], hi1);
    __syncthreads();
    if (threadIdx.x < 3) atomicMin(&mm[threadIdx.x], s_mm[threadIdx.x]);
    else if (threadIdx.x < 6) atomicMax(&mm[threadIdx.x], s_mm[threadIdx.x]);
}

static void bbox_launch(sfb_ctx *ctx, const double *pos, int64_t n, unsigned long long *mm) {
    k_bbox_init<<<1, 32, 0, ctx->stream>>>(mm);
    if ((reinterpret_cast<uintptr_t>(pos) & 15) == 0 && n >= 2) {
        k_bbox2<<<grid_for(3 * n / 2, kBBoxThreads * 4, ctx->num_sms * 2), kBBoxThreads, 0, ctx->stream>>>(
            reinterpret_cast<const double2 *>(pos), n, mm);
    } else {
        k_bbox<<<grid_for(3 * n, kBBoxThreads, ctx->num_sms * 4), kBBoxThreads, 0, ctx->stream>>>(pos, n, mm);
    }
    SFB_CHECK_LAUNCH();
}

void bbox_run(sfb_ctx *ctx, const double *pos, int64_t n, double *lo_hi_host) {
    SFB_REQUIRE(n > 0, "empty cloud has no bbox");
    auto *mm = ctx->arena.alloc<unsigned long long>(6);
    bbox_launch(ctx, pos, n, mm);
    ctx->read_back(mm, 6 * sizeof(unsigned long long));
    for (int a = 0; a < 6; ++a) lo_hi_host[a] = unord_bits((unsigned long long)ctx->pinned[a]);
}

// enqueue-only variant: the 6 order-preserving words land in caller pinned
// memory when the stream reaches them (no host synchronisation)
void bbox_async_run(sfb_ctx *ctx, const double *pos, int64_t n, uint64_t *ordered_host) {
    SFB_REQUIRE(n > 0, "empty cloud has no bbox");
    auto *mm = ctx->arena.alloc<unsigned long long>(6);
    bbox_launch(ctx, pos, n, mm);
    SFB_CUDA(cudaMemcpyAsync(ordered_host, mm, 6 * sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                             ctx->stream));
}

template <class K>
__global__ void k_keygen(const double *__restrict__ pos, int64_t n, const FrameParams *__restrict__ P,
                         K *__restrict__ keys, uint32_t *__restrict__ vals) {
    const double s = P->s;
    const int bx = P->bits[0], bxy = P->bits[0] + P->bits[1];
    const int64_t lx = P->lo[0], ly = P->lo[1], lz = P->lo[2];
    SFB_FOR(i, n) {
        int64_t ix = (int64_t)floor(__dmul_rn(pos[3 * i + 0], s)) - lx;
        int64_t iy = (int64_t)floor(__dmul_rn(pos[3 * i + 1], s)) - ly;
        int64_t iz = (int64_t)floor(__dmul_rn(pos[3 * i + 2], s)) - lz;
        keys[i] = (K)(((uint64_t)iz << bxy) | ((uint64_t)iy << bx) | (uint64_t)ix);
        vals[i] = (uint32_t)i;
    }
}

// keys of at most 32 bits: one 64-bit word per point, (index << 32) | key, so
// each radix pass scatters one 8-byte word instead of a key and a value
__global__ void k_keygen_packed(const double *__restrict__ pos, int64_t n,
                                const FrameParams *__restrict__ P, unsigned long long *__restrict__ kv) {
    const double s = P->s;
    const int bx = P->bits[0], bxy = P->bits[0] + P->bits[1];
    const int64_t lx = P->lo[0], ly = P->lo[1], lz = P->lo[2];
    SFB_FOR(i, n) {
        int64_t ix = (int64_t)floor(__dmul_rn(pos[3 * i + 0], s)) - lx;
        int64_t iy = (int64_t)floor(__dmul_rn(pos[3 * i + 1], s)) - ly;
        int64_t iz = (int64_t)floor(__dmul_rn(pos[3 * i + 2], s)) - lz;
        kv[i] = ((unsigned long long)i << 32) |
                (uint32_t)(((uint64_t)iz << bxy) | ((uint64_t)iy << bx) | (uint64_t)ix);
    }
}

// sorted (key, point) readers of k_vox_segments: split arrays or packed words
template <class K>
struct SplitKV {
    const K *k;
    const uint32_t *v;
    __device__ __forceinline__ K key(int64_t i) const { return k[i]; }
    __device__ __forceinline__ uint32_t val(int64_t i) const { return v[i]; }
};
struct PackedKV {
    const unsigned long long *p;
    __device__ __forceinline__ uint32_t key(int64_t i) const { return (uint32_t)p[i]; }
    __device__ __forceinline__ uint32_t val(int64_t i) const { return (uint32_t)(p[i] >> 32); }
};

// Segmentation of the sorted point keys in one pass (np.unique's sorted keys,
// inverse and CSR of voxelgrid.py:146, 165-168): head flags from adjacent
// keys, their inclusive scan by decoupled look-back (tiles in ticket order),
// then per element the point -> voxel map, the CSR order and, at each head,
// the voxel's coordinates, packed key and first offset. Replaces a flag
// kernel, a scan and a segment kernel (and the flag array's round trips).
constexpr int kSegThreads = 1024, kSegItems = 4, kSegTile = kSegThreads * kSegItems;

template <class K, class KV>
__global__ void __launch_bounds__(kSegThreads)
k_vox_segments(const KV kv, int64_t n,
               const FrameParams *__restrict__ P, int32_t *__restrict__ coords,
               int64_t *__restrict__ pkeys, int32_t *__restrict__ p2v, int32_t *__restrict__ order,
               int32_t *__restrict__ offsets, DevCounts *__restrict__ C,
               unsigned long long *__restrict__ status, unsigned int *__restrict__ ticket) {
    __shared__ int32_t s_val[kSegTile];
    __shared__ int32_t s_warp[32];
    __shared__ int s_tile;
    __shared__ int32_t s_excl;
    const int bx = P->bits[0], by = P->bits[1];
    const int64_t ntiles = (n + kSegTile - 1) / kSegTile;
    for (;;) {
        if (threadIdx.x == 0) s_tile = (int)atomicAdd(ticket, 1u);
        __syncthreads();
        const int64_t tile = s_tile;
        if (tile >= ntiles) break;
        const int64_t base = tile * kSegTile;
        K key[kSegItems];
        int32_t f[kSegItems];
#pragma unroll
        for (int k = 0; k < kSegItems; ++k) {   // coalesced: element base + k*1024 + tid
            const int64_t i = base + k * kSegThreads + threadIdx.x;
            f[k] = 0;
            if (i < n) {
                key[k] = kv.key(i);
                f[k] = (i == 0 || key[k] != kv.key(i - 1)) ? 1 : 0;
            }
            s_val[k * kSegThreads + threadIdx.x] = f[k];
        }
        __syncthreads();
        int32_t v[kSegItems], sum = 0;   // blocked: elements tid*4 .. tid*4+3 of the tile
#pragma unroll
        for (int k = 0; k < kSegItems; ++k) {
            v[k] = s_val[threadIdx.x * kSegItems + k];
            sum += v[k];
        }
        int32_t agg;
        const int32_t ex = block_excl_scan(sum, s_warp, &agg);
        if (threadIdx.x < 32) {
            const int32_t prefix = lb_prefix(status, tile, agg);
            if (threadIdx.x == 0) s_excl = prefix;
        }
        __syncthreads();
        int32_t run = s_excl + ex;
#pragma unroll
        for (int k = 0; k < kSegItems; ++k) {
            run += v[k];
            s_val[threadIdx.x * kSegItems + k] = run;   // inclusive head count
        }
        __syncthreads();
#pragma unroll
        for (int k = 0; k < kSegItems; ++k) {
            const int64_t j = base + k * kSegThreads + threadIdx.x;
            if (j >= n) continue;
            const int32_t vox = s_val[k * kSegThreads + threadIdx.x] - 1;
            const uint32_t i = kv.val(j);
            order[j] = (int32_t)i;
            p2v[i] = vox;
            if (j == n - 1) {
                offsets[vox + 1] = (int32_t)n;
                C->m[0] = vox + 1;
            }
            if (f[k]) {
                const uint64_t kk = (uint64_t)key[k];
                const int64_t x = (int64_t)(kk & ((1ull << bx) - 1)) + P->lo[0];
                const int64_t y = (int64_t)((kk >> bx) & ((1ull << by) - 1)) + P->lo[1];
                const int64_t z = (int64_t)(kk >> (bx + by)) + P->lo[2];
                coords[3 * vox + 0] = (int32_t)x;
                coords[3 * vox + 1] = (int32_t)y;
                coords[3 * vox + 2] = (int32_t)z;
                pkeys[vox] = pack_key(x, y, z);
                offsets[vox] = (int32_t)j;
            }
        }
        __syncthreads();
    }
}

// Six lanes per voxel, one per summed channel (scaled x, y, z, colour r, g,
// b; five voxels per warp): each lane walks the voxel's points in ascending
// point index (the CSR order) and adds its channel strictly in that order —
// bit-identical to np.add.at — with the point gathers of ~6 M voxels-lanes
// in flight instead of one serial walk per voxel.
__global__ void k_voxel_feats(const double *__restrict__ pos, const double *__restrict__ col,
                              const int32_t *__restrict__ order, const int32_t *__restrict__ offsets,
                              const int32_t *__restrict__ coords, const DevCounts *__restrict__ C,
                              const FrameParams *__restrict__ P, double *__restrict__ feats,
                              float *__restrict__ feats32) {
    const int64_t m = C->m[0];
    const double s = P->s;
    const int lane = threadIdx.x & 31;
    if (lane >= 30) return;
    const int slot = lane / 6, ch = lane % 6;
    const double *__restrict__ src = ch < 3 ? pos + ch : col + (ch - 3);
    const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t v = 5 * w0 + slot; v < m; v += 5 * nw) {
        const int32_t b = offsets[v], e = offsets[v + 1];
        double acc = 0.0;
#pragma unroll 8
        for (int32_t j = b; j < e; ++j) {
            const double x = src[3 * (size_t)order[j]];
            acc = __dadd_rn(acc, ch < 3 ? __dmul_rn(x, s) : x);
        }
        const double cnt = (double)(e - b);
        const double mean = __ddiv_rn(acc, cnt);
        double *f = feats + 9 * v;
        if (ch < 3) {
            double res = __dsub_rn(mean, __dadd_rn((double)coords[3 * v + ch], 0.5));
            const double a = __ddiv_rn(mean, s), r = fmin(fmax(res, -0.5), 0.5);
            f[ch] = a;
            f[6 + ch] = r;
            if (feats32) {   // the UNet's float32 input, same rounding as a separate cast
                feats32[9 * v + ch] = (float)a;
                feats32[9 * v + 6 + ch] = (float)r;
            }
        } else {
            f[ch] = mean;
            if (feats32) feats32[9 * v + ch] = (float)mean;
        }
    }
}

template <class K>
static void voxelize_typed(sfb_ctx *ctx, const double *pos, const double *col, int64_t n,
                           const FrameParams *P, int key_bits, VoxelOut &out, DevCounts *C,
                           bool feats_on_side) {
    cudaStream_t st = ctx->stream;
    const unsigned g = dgrid(n, 256);
    // the library's own stable LSD sort (devprims.cu: 8-bit digits, 1024-item
    // sub-tiles ranked with __match_any_sync, small shared memory so its CTAs
    // share SMs with the other lanes' kernels) on the key bits only: equal
    // keys keep ascending point order
    constexpr bool packed = sizeof(K) == 4;
    SplitKV<K> skv{};
    PackedKV pkv{};
    if (packed) {
        auto *w = ctx->arena.alloc<unsigned long long>(n), *w2 = ctx->arena.alloc<unsigned long long>(n);
        k_keygen_packed<<<g, 256, 0, st>>>(pos, n, P, w);
        SFB_CHECK_LAUNCH();
        pkv.p = dsort_pairs<unsigned long long>(ctx, w, nullptr, w2, nullptr, nullptr, n, key_bits) ? w2 : w;
    } else {
        K *keys = ctx->arena.alloc<K>(n), *keys2 = ctx->arena.alloc<K>(n);
        uint32_t *vals = ctx->arena.alloc<uint32_t>(n), *vals2 = ctx->arena.alloc<uint32_t>(n);
        k_keygen<K><<<g, 256, 0, st>>>(pos, n, P, keys, vals);
        SFB_CHECK_LAUNCH();
        const bool second = dsort_pairs<K>(ctx, keys, vals, keys2, vals2, nullptr, n, key_bits);
        skv.k = second ? keys2 : keys;
        skv.v = second ? vals2 : vals;
    }
    {
        const int64_t tiles = (n + kSegTile - 1) / kSegTile;
        const size_t bytes = sizeof(unsigned long long) * (size_t)(tiles + 1);
        auto *status = static_cast<unsigned long long *>(ctx->arena.alloc_bytes(bytes));
        SFB_CUDA(cudaMemsetAsync(status, 0, bytes, st));
        const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(tiles, 2 * 148));
        auto *ticket = reinterpret_cast<unsigned int *>(status + tiles);
        if (packed)
            k_vox_segments<uint32_t><<<grid, kSegThreads, 0, st>>>(pkv, n, P, out.coords, out.keys, out.p2v,
                                                               out.order, out.offsets, C, status, ticket);
        else
            k_vox_segments<K><<<grid, kSegThreads, 0, st>>>(skv, n, P, out.coords, out.keys, out.p2v,
                                                        out.order, out.offsets, C, status, ticket);
    }
    SFB_CHECK_LAUNCH();
    const int64_t vwarps = (ctx->grid_bound(n, ctx->hint_m[0]) + 4) / 5;
    cudaStream_t fs = st;
    if (feats_on_side) {   // fork: the sums need only the segmentation above
        cudaEvent_t fork = ctx->side_ev[sfb_ctx::kEvFeatsFork];
        SFB_CUDA(cudaEventRecord(fork, st));
        SFB_CUDA(cudaStreamWaitEvent(ctx->aux_stream, fork, 0));
        fs = ctx->aux_stream;
    }
    k_voxel_feats<<<dgrid(32 * vwarps, 256), 256, 0, fs>>>(pos, col, out.order, out.offsets,
                                                          out.coords, C, P, out.feats, out.feats32);
    SFB_CHECK_LAUNCH();
    if (feats_on_side) {
        SFB_CUDA(cudaEventRecord(ctx->side_ev[sfb_ctx::kEvFeatsJoin], fs));
        ctx->feats_pending = true;
    }
}

// Host half of voxelize_adaptive's key setup: s and the per-axis ranges are
// known from the bbox, so the compact key needs only the bits the cloud spans.
void voxel_layout(const double *lo_hi, double s, FrameParams &P) {
    SFB_REQUIRE(s > 0.0 && s == s, "voxel scale must be positive");
    P.s = s;
    P.inv_s = 1.0 / s;
    P.total = 0;
    for (int a = 0; a < 3; ++a) {
        // floor(lo*s) .. floor(hi*s) bounds floor(p*s) for every point (monotone rounding)
        int64_t lo = (int64_t)std::floor(lo_hi[a] * s);
        int64_t hi = (int64_t)std::floor(lo_hi[3 + a] * s);
        SFB_REQUIRE(lo > -(int64_t(1) << 20) && hi < (int64_t(1) << 20),
                    "voxel coordinates must satisfy |c| < 1048576");
        P.lo[a] = lo;
        P.hi[a] = hi;
        P.bits[a] = bits_for((uint64_t)(hi - lo));
        P.total += P.bits[a];
    }
}

void voxelize_run(sfb_ctx *ctx, const double *pos, const double *col, int64_t n,
                  const FrameParams &host, const FrameParams *P, VoxelOut &out, DevCounts *C,
                  bool feats_on_side) {
    SFB_REQUIRE(n >= 2, "voxelization needs at least 2 points");
    SFB_REQUIRE(n < (int64_t(1) << 31), "at most 2^31-1 points per cloud");
    const int bits = host.total > 0 ? host.total : 1;
    if (host.total <= 32) voxelize_typed<uint32_t>(ctx, pos, col, n, P, bits, out, C, feats_on_side);
    else voxelize_typed<unsigned long long>(ctx, pos, col, n, P, bits, out, C, feats_on_side);
}

}  // namespace sfb
