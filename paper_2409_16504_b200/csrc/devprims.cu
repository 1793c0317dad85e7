// Device-count primitives: scans and a stable LSD radix sort whose element
// count lives in DEVICE memory (written by an earlier kernel), with grids
// sized from a host capacity. They let the whole frame run without a single
// device->host size read after the bbox, which is what makes it capturable
// as one CUDA graph (the P2ENet level sizes, kept splats, runs and tile
// entries are all data-dependent).
#include <algorithm>
#include <mutex>
#include <set>
#include <tuple>

#include "common.cuh"
#include "scan.cuh"

namespace sfb {

constexpr int kScanBlocks = 148;
constexpr int kScanThreads = 1024;
constexpr int kScanGrid = 2 * 148;

// ------------------------------------------------------------------ scan
__device__ __forceinline__ int64_t chunk_of(int64_t n, int blocks) {
    return (n + blocks - 1) / blocks;
}

__global__ void __launch_bounds__(kScanThreads)
k_scan_partials(const int32_t *__restrict__ in, const int64_t *__restrict__ d_n, int64_t n_fixed,
                int32_t *__restrict__ part) {
    __shared__ int32_t s_warp[32];
    const int64_t n = d_n ? *d_n : n_fixed;
    const int64_t ch = chunk_of(n, gridDim.x);
    const int64_t b0 = blockIdx.x * ch, b1 = min(n, b0 + ch);
    int32_t s = 0;
    for (int64_t i = b0 + threadIdx.x; i < b1; i += blockDim.x) s += in[i];
    int32_t tot;
    block_excl_scan(s, s_warp, &tot);
    if (threadIdx.x == 0) part[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(kScanThreads)
k_scan_apply(const int32_t *__restrict__ in, const int64_t *__restrict__ d_n, int64_t n_fixed,
             const int32_t *__restrict__ part, int32_t *__restrict__ out,
             int64_t *__restrict__ total_out, int inclusive) {
    __shared__ int32_t s_warp[32];
    __shared__ int32_t s_base;
    const int64_t n = d_n ? *d_n : n_fixed;
    const int64_t ch = chunk_of(n, gridDim.x);
    const int64_t b0 = blockIdx.x * ch, b1 = min(n, b0 + ch);
    {   // base = sum of the partials of earlier blocks (parallel, <= 1024 blocks)
        const int32_t v = (int)threadIdx.x < (int)blockIdx.x ? part[threadIdx.x] : 0;
        int32_t tot;
        block_excl_scan(v, s_warp, &tot);
        if (threadIdx.x == 0) {
            s_base = tot;
            if (blockIdx.x == gridDim.x - 1 && total_out) *total_out = tot + part[blockIdx.x];
        }
        __syncthreads();
    }
    int32_t base = s_base;
    for (int64_t t0 = b0; t0 < b1; t0 += blockDim.x) {
        const int64_t i = t0 + threadIdx.x;
        const int32_t v = i < b1 ? in[i] : 0;
        int32_t tile_total;
        const int32_t ex = block_excl_scan(v, s_warp, &tile_total);
        if (i < b1) out[i] = base + ex + (inclusive ? v : 0);
        base += tile_total;
    }
}

// Single-pass scan with decoupled look-back: tiles of kLbItems*1024 values
// are taken in ticket order (so every tile a tile waits on is already
// running); a tile publishes its aggregate, warp 0 accumulates predecessor
// aggregates 32 at a time until it meets an inclusive prefix, then publishes
// its own inclusive prefix. One launch per scan instead of two.
constexpr int kLbItems = 4;
constexpr int kLbTile = kLbItems * kScanThreads;
__global__ void __launch_bounds__(kScanThreads)
k_scan_lb(const int32_t *__restrict__ in, int32_t *__restrict__ out, const int64_t *__restrict__ d_n,
          int64_t n_fixed, int64_t *__restrict__ total_out, int inclusive,
          unsigned long long *__restrict__ status, unsigned int *__restrict__ ticket) {
    __shared__ int32_t s_val[kLbTile];
    __shared__ int32_t s_warp[32];
    __shared__ int s_tile;
    __shared__ int32_t s_excl;
    const int64_t n = d_n ? *d_n : n_fixed;
    const int64_t ntiles = (n + kLbTile - 1) / kLbTile;
    const int lane = threadIdx.x & 31;
    for (;;) {
        if (threadIdx.x == 0) s_tile = (int)atomicAdd(ticket, 1u);
        __syncthreads();
        const int64_t tile = s_tile;
        if (tile >= ntiles) break;
        const int64_t base = tile * kLbTile;
#pragma unroll
        for (int k = 0; k < kLbItems; ++k) {
            const int64_t i = base + k * kScanThreads + threadIdx.x;
            s_val[k * kScanThreads + threadIdx.x] = i < n ? in[i] : 0;
        }
        __syncthreads();
        int32_t v[kLbItems], sum = 0;
#pragma unroll
        for (int k = 0; k < kLbItems; ++k) {
            v[k] = s_val[threadIdx.x * kLbItems + k];
            sum += v[k];
        }
        int32_t agg;
        const int32_t ex = block_excl_scan(sum, s_warp, &agg);
        if (threadIdx.x < 32) {
            int32_t prefix = 0;
            if (tile == 0) {
                if (lane == 0) atomicExch(&status[0], kLbInc | (uint32_t)agg);
            } else {
                if (lane == 0) atomicExch(&status[tile], kLbAgg | (uint32_t)agg);
                int64_t pred = tile - 1;
                for (;;) {   // window of 32 predecessors, nearest in lane 0
                    const int64_t q = pred - lane;
                    unsigned long long st = q >= 0 ? lb_load(&status[q]) : kLbInc;
                    while (__any_sync(0xffffffffu, (st >> 32) == 0)) {
                        if ((st >> 32) == 0) st = lb_load(&status[q]);
                    }
                    const unsigned inc = __ballot_sync(0xffffffffu, (st >> 32) == 2);
                    const int stop = inc ? __ffs(inc) - 1 : 31;   // lanes 0..stop count
                    int32_t val = lane <= stop ? (int32_t)(uint32_t)st : 0;
                    for (int o = 16; o; o >>= 1) val += __shfl_xor_sync(0xffffffffu, val, o);
                    prefix += val;
                    if (inc) break;
                    pred -= 32;
                }
                if (lane == 0) atomicExch(&status[tile], kLbInc | (uint32_t)(prefix + agg));
            }
            if (lane == 0) s_excl = prefix;
        }
        __syncthreads();
        int32_t run = s_excl + ex;
#pragma unroll
        for (int k = 0; k < kLbItems; ++k) {
            s_val[threadIdx.x * kLbItems + k] = run + (inclusive ? v[k] : 0);
            run += v[k];
        }
        __syncthreads();
#pragma unroll
        for (int k = 0; k < kLbItems; ++k) {
            const int64_t i = base + k * kScanThreads + threadIdx.x;
            if (i < n) out[i] = s_val[k * kScanThreads + threadIdx.x];
        }
        if (tile == ntiles - 1 && threadIdx.x == 0 && total_out) *total_out = s_excl + agg;
        __syncthreads();
    }
    if (ntiles == 0 && blockIdx.x == 0 && threadIdx.x == 0 && total_out) *total_out = 0;
}

// Three exclusive scans of one length in ONE launch (per-run fine / super /
// global entry counts): the same look-back with a status word per column.
constexpr int kScan3Items = 2;   // 3 x 2048 int32 staged per tile (24 KB)
struct Scan3 {
    const int32_t *in[3];
    int32_t *out[3];
    int64_t *tot[3];
};

__global__ void __launch_bounds__(kScanThreads)
k_scan3_lb(Scan3 S, const int64_t *__restrict__ d_n, int64_t n_fixed,
           unsigned long long *__restrict__ status /* [3][tiles] */, int64_t tiles_cap,
           unsigned int *__restrict__ ticket) {
    constexpr int IT = kScan3Items;
    constexpr int TILE = IT * kScanThreads;
    __shared__ int32_t s_val[3][TILE];
    __shared__ int32_t s_warp[32];
    __shared__ int s_tile;
    __shared__ int32_t s_excl[3];
    const int64_t n = d_n ? *d_n : n_fixed;
    const int64_t ntiles = (n + TILE - 1) / TILE;
    const int lane = threadIdx.x & 31;
    for (;;) {
        if (threadIdx.x == 0) s_tile = (int)atomicAdd(ticket, 1u);
        __syncthreads();
        const int64_t tile = s_tile;
        if (tile >= ntiles) break;
        const int64_t base = tile * TILE;
#pragma unroll
        for (int c = 0; c < 3; ++c)
#pragma unroll
            for (int k = 0; k < IT; ++k) {
                const int64_t i = base + k * kScanThreads + threadIdx.x;
                s_val[c][k * kScanThreads + threadIdx.x] = i < n ? S.in[c][i] : 0;
            }
        __syncthreads();
        int32_t v[3][IT], ex[3], agg[3];
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            int32_t sum = 0;
#pragma unroll
            for (int k = 0; k < IT; ++k) {
                v[c][k] = s_val[c][threadIdx.x * IT + k];
                sum += v[c][k];
            }
            ex[c] = block_excl_scan(sum, s_warp, &agg[c]);
        }
        if (threadIdx.x < 32) {
            for (int c = 0; c < 3; ++c) {
                unsigned long long *stc = status + c * tiles_cap;
                int32_t prefix = 0;
                if (tile == 0) {
                    if (lane == 0) atomicExch(&stc[0], kLbInc | (uint32_t)agg[c]);
                } else {
                    if (lane == 0) atomicExch(&stc[tile], kLbAgg | (uint32_t)agg[c]);
                    int64_t pred = tile - 1;
                    for (;;) {
                        const int64_t q = pred - lane;
                        unsigned long long st = q >= 0 ? lb_load(&stc[q]) : kLbInc;
                        while (__any_sync(0xffffffffu, (st >> 32) == 0)) {
                            if ((st >> 32) == 0) st = lb_load(&stc[q]);
                        }
                        const unsigned inc = __ballot_sync(0xffffffffu, (st >> 32) == 2);
                        const int stop = inc ? __ffs(inc) - 1 : 31;
                        int32_t val = lane <= stop ? (int32_t)(uint32_t)st : 0;
                        for (int o = 16; o; o >>= 1) val += __shfl_xor_sync(0xffffffffu, val, o);
                        prefix += val;
                        if (inc) break;
                        pred -= 32;
                    }
                    if (lane == 0) atomicExch(&stc[tile], kLbInc | (uint32_t)(prefix + agg[c]));
                }
                if (lane == 0) s_excl[c] = prefix;
            }
        }
        __syncthreads();
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            int32_t run = s_excl[c] + ex[c];
#pragma unroll
            for (int k = 0; k < IT; ++k) {
                s_val[c][threadIdx.x * IT + k] = run;
                run += v[c][k];
            }
        }
        __syncthreads();
#pragma unroll
        for (int c = 0; c < 3; ++c)
#pragma unroll
            for (int k = 0; k < IT; ++k) {
                const int64_t i = base + k * kScanThreads + threadIdx.x;
                if (i < n) S.out[c][i] = s_val[c][k * kScanThreads + threadIdx.x];
            }
        if (tile == ntiles - 1 && threadIdx.x < 3 && S.tot[threadIdx.x])
            *S.tot[threadIdx.x] = s_excl[threadIdx.x] + agg[threadIdx.x];
        __syncthreads();
    }
    if (ntiles == 0 && blockIdx.x == 0 && threadIdx.x < 3 && S.tot[threadIdx.x]) *S.tot[threadIdx.x] = 0;
}

void dscan3(sfb_ctx *ctx, const int32_t *in0, const int32_t *in1, const int32_t *in2, int32_t *out0,
            int32_t *out1, int32_t *out2, const int64_t *d_n, int64_t n_fixed, int64_t *tot0,
            int64_t *tot1, int64_t *tot2) {
    const int64_t tiles = (n_fixed + kScan3Items * kScanThreads - 1) / (kScan3Items * kScanThreads) + 1;
    const size_t bytes = sizeof(unsigned long long) * (size_t)(3 * tiles + 1);
    auto *status = static_cast<unsigned long long *>(ctx->arena.alloc_bytes(bytes));
    SFB_CUDA(cudaMemsetAsync(status, 0, bytes, ctx->stream));
    Scan3 S{{in0, in1, in2}, {out0, out1, out2}, {tot0, tot1, tot2}};
    const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(tiles, kScanGrid));
    k_scan3_lb<<<grid, kScanThreads, 0, ctx->stream>>>(S, d_n, n_fixed, status, tiles,
                                                       reinterpret_cast<unsigned int *>(status + 3 * tiles));
    SFB_CHECK_LAUNCH();
}

// exclusive (or inclusive) scan of n int32 (n from device if d_n, else n_fixed);
// in-place allowed; the grand total is written to *total_out when given.
void dscan(sfb_ctx *ctx, const int32_t *in, int32_t *out, const int64_t *d_n, int64_t n_fixed,
           int64_t *total_out, bool inclusive) {
    const int64_t tiles = (n_fixed + kLbTile - 1) / kLbTile;
    const size_t bytes = sizeof(unsigned long long) * (size_t)(tiles + 1);
    auto *status = static_cast<unsigned long long *>(ctx->arena.alloc_bytes(bytes));
    SFB_CUDA(cudaMemsetAsync(status, 0, bytes, ctx->stream));
    auto *ticket = reinterpret_cast<unsigned int *>(status + tiles);
    const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(tiles, kScanGrid));
    k_scan_lb<<<grid, kScanThreads, 0, ctx->stream>>>(in, out, d_n, n_fixed, total_out,
                                                      inclusive ? 1 : 0, status, ticket);
    SFB_CHECK_LAUNCH();
}

// ------------------------------------------------------------------ params
__global__ void k_write_params(FrameParams p, FrameParams *dst) { *dst = p; }

void write_params(sfb_ctx *ctx, const FrameParams &host, FrameParams *dev) {
    k_write_params<<<1, 1, 0, ctx->stream>>>(host, dev);
    SFB_CHECK_LAUNCH();
}

void set_max_dyn_smem(const void *func, int bytes) {
    static std::mutex mu;
    static std::set<std::tuple<int, const void *, int>> done;
    int dev = 0;
    SFB_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lock(mu);
    if (done.count({dev, func, bytes})) return;
    SFB_CUDA(cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    done.insert({dev, func, bytes});
}

const void *write_params_func() { return reinterpret_cast<const void *>(&k_write_params); }

Cam to_cam(const sfb_camera &c) {
    Cam k;
    for (int i = 0; i < 9; ++i) k.r[i] = c.rot[i];
    for (int i = 0; i < 3; ++i) k.t[i] = c.trans[i];
    k.fx = c.fx;
    k.fy = c.fy;
    k.cx = c.cx;
    k.cy = c.cy;
    k.w = c.width;
    k.h = c.height;
    return k;
}

// ------------------------------------------------------------------ radix sort
constexpr int kRsBlocks = 148;   // a multiple of 4 (the offset prologue reads kRsBlocks / 4 per round)
constexpr int kRsThreads = 256;
constexpr int kRsWarps = kRsThreads / 32;

// blocks that take part in a pass: at least one 256-item sub-tile each, at
// most kRsBlocks (small sorts spread thin: one sub-tile per block)
constexpr int kRsMinItems = 256;
__device__ __forceinline__ int rs_blocks(int64_t n) {
    int64_t b = (n + kRsMinItems - 1) / kRsMinItems;
    return (int)max((int64_t)1, min(b, (int64_t)kRsBlocks));
}

template <class K>
__global__ void __launch_bounds__(kRsThreads)
k_rs_upsweep(const K *__restrict__ keys, const int64_t *__restrict__ d_n, int64_t n_fixed, int shift,
             int32_t *__restrict__ hist) {
    __shared__ int32_t h[256];
    const int64_t n = d_n ? *d_n : n_fixed;
    const int nb = rs_blocks(n);
    if ((int)blockIdx.x >= nb) return;
    h[threadIdx.x] = 0;
    __syncthreads();
    const int64_t ch = chunk_of(n, nb);
    const int64_t b0 = blockIdx.x * ch, b1 = min(n, b0 + ch);
    for (int64_t i = b0 + threadIdx.x; i < b1; i += blockDim.x)
        atomicAdd(&h[(uint32_t)(keys[i] >> shift) & 255u], 1);
    __syncthreads();
    hist[blockIdx.x * 256 + threadIdx.x] = h[threadIdx.x];
}

// stable scatter: each block first forms its digit offsets from the
// block-major histogram (digit base = exclusive scan over digits of the
// totals, plus the counts of earlier blocks), then walks its chunk in order,
// kRsIpt * 256 items at a time: warp w owns items [w * 32 * kRsIpt, ...) of
// the sub-tile and ranks them in kRsIpt rounds of 32 (__match_any_sync peers
// + the warp's running per-digit count), then the warps' counts are prefixed
// per digit — 4 block barriers per 1024 items instead of 3 per 256
constexpr int kRsIpt = 4;
template <class K, bool HAS_VALS>
__global__ void __launch_bounds__(kRsThreads)
k_rs_downsweep(const K *__restrict__ kin, const uint32_t *__restrict__ vin, K *__restrict__ kout,
               uint32_t *__restrict__ vout, const int64_t *__restrict__ d_n, int64_t n_fixed,
               int shift, const int32_t *__restrict__ hist) {
    __shared__ int32_t run[256];
    __shared__ int32_t wcnt[kRsWarps][256];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t n = d_n ? *d_n : n_fixed;
    const int nb = rs_blocks(n);
    if ((int)blockIdx.x >= nb) return;
    const int64_t ch = chunk_of(n, nb);
    const int64_t b0 = blockIdx.x * ch, b1 = min(n, b0 + ch);
    constexpr int SUB = kRsThreads * kRsIpt;
    // sub-tile loads (warp w owns items [w * 32 * kRsIpt, ...)): the first
    // sub-tile's are issued before the offset prologue, each next one's
    // before the current one is ranked, so their latency hides
    auto load = [&](int64_t t0, K *key, uint32_t *val) {
        const int64_t wbase = t0 + (int64_t)warp * 32 * kRsIpt;
#pragma unroll
        for (int q = 0; q < kRsIpt; ++q) {
            const int64_t i = wbase + q * 32 + lane;
            const bool ok = i < b1;
            key[q] = ok ? kin[i] : K(0);
            val[q] = (HAS_VALS && ok) ? vin[i] : 0u;
        }
    };
    K key[kRsIpt];
    uint32_t val[kRsIpt];
    load(b0, key, val);
    {
        int32_t tot = 0, pre = 0;
        constexpr int R = kRsBlocks / 4;   // 37 loads in flight: <= 4 rounds
        for (int b = 0; b < nb; b += R) {
            int32_t c[R];
#pragma unroll
            for (int u = 0; u < R; ++u) c[u] = b + u < nb ? hist[(b + u) * 256 + threadIdx.x] : 0;
#pragma unroll
            for (int u = 0; u < R; ++u) {
                tot += c[u];
                pre += b + u < (int)blockIdx.x ? c[u] : 0;
            }
        }
        __shared__ int32_t s_warp[32];
        const int32_t base = block_excl_scan(tot, s_warp, nullptr);
        run[threadIdx.x] = base + pre;
    }
    for (int w = 0; w < kRsWarps; ++w) wcnt[w][threadIdx.x] = 0;
    __syncthreads();
    const uint32_t lt = (1u << lane) - 1u;
    for (int64_t t0 = b0; t0 < b1; t0 += SUB) {
        uint32_t dg[kRsIpt];
        int32_t lr[kRsIpt];
        const int64_t wbase = t0 + (int64_t)warp * 32 * kRsIpt;
#pragma unroll
        for (int q = 0; q < kRsIpt; ++q)
            dg[q] = wbase + q * 32 + lane < b1 ? ((uint32_t)(key[q] >> shift) & 255u) : 256u;
        K nkey[kRsIpt];
        uint32_t nval[kRsIpt];
        if (t0 + SUB < b1) load(t0 + SUB, nkey, nval);
#pragma unroll
        for (int q = 0; q < kRsIpt; ++q) {   // rounds in item order
            const uint32_t d = dg[q];
            const uint32_t peers = __match_any_sync(0xffffffffu, d);
            const int r = __popc(peers & lt);
            lr[q] = d < 256u ? wcnt[warp][d] + r : 0;
            __syncwarp();
            if (d < 256u && r == 0) wcnt[warp][d] += __popc(peers);
            __syncwarp();
        }
        __syncthreads();
        // per digit: exclusive prefix over warps (in place), digit total
        int32_t tot = 0;
#pragma unroll
        for (int w = 0; w < kRsWarps; ++w) {
            const int32_t c = wcnt[w][threadIdx.x];
            wcnt[w][threadIdx.x] = tot;
            tot += c;
        }
        __syncthreads();
#pragma unroll
        for (int q = 0; q < kRsIpt; ++q) {
            const uint32_t d = dg[q];
            if (d < 256u) {
                const int32_t pos = run[d] + wcnt[warp][d] + lr[q];
                kout[pos] = key[q];
                if (HAS_VALS) vout[pos] = val[q];
            }
        }
        __syncthreads();
        run[threadIdx.x] += tot;
#pragma unroll
        for (int w = 0; w < kRsWarps; ++w) wcnt[w][threadIdx.x] = 0;
#pragma unroll
        for (int q = 0; q < kRsIpt; ++q) {
            key[q] = nkey[q];
            val[q] = nval[q];
        }
        __syncthreads();
    }
}

// Stable LSD sort of (key, val) over bits [0, bits). Result ends in (k0, v0)
// if the pass count is even, else in (k1, v1); returns which (0/1).
template <class K>
int dsort_pairs(sfb_ctx *ctx, K *k0, uint32_t *v0, K *k1, uint32_t *v1, const int64_t *d_n,
                int64_t n_fixed, int bits) {
    const int passes = (bits + 7) / 8;
    int32_t *hist = ctx->arena.alloc<int32_t>(256 * kRsBlocks);
    for (int p = 0; p < passes; ++p) {
        K *ki = (p & 1) ? k1 : k0, *ko = (p & 1) ? k0 : k1;
        uint32_t *vi = (p & 1) ? v1 : v0, *vo = (p & 1) ? v0 : v1;
        k_rs_upsweep<K><<<kRsBlocks, kRsThreads, 0, ctx->stream>>>(ki, d_n, n_fixed, 8 * p, hist);
        if (v0)
            k_rs_downsweep<K, true><<<kRsBlocks, kRsThreads, 0, ctx->stream>>>(ki, vi, ko, vo, d_n,
                                                                               n_fixed, 8 * p, hist);
        else
            k_rs_downsweep<K, false><<<kRsBlocks, kRsThreads, 0, ctx->stream>>>(
                ki, nullptr, ko, nullptr, d_n, n_fixed, 8 * p, hist);
        SFB_CHECK_LAUNCH();
    }
    return passes & 1;
}

template int dsort_pairs<uint32_t>(sfb_ctx *, uint32_t *, uint32_t *, uint32_t *, uint32_t *,
                                   const int64_t *, int64_t, int);
template int dsort_pairs<unsigned long long>(sfb_ctx *, unsigned long long *, uint32_t *,
                                             unsigned long long *, uint32_t *, const int64_t *,
                                             int64_t, int);

}  // namespace sfb
