// Block scan and decoupled look-back pieces shared by the device-count scans
// (devprims.cu) and the fused voxel segmentation (voxelize.cu).
#pragma once
#include "common.cuh"

namespace sfb {

// exclusive scan of one int32 per thread over the block (any multiple of 32
// threads up to 1024); *total gets the block sum when non-null
__device__ __forceinline__ int32_t block_excl_scan(int32_t v, int32_t *s_warp, int32_t *total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) s_warp[warp] = x;
    __syncthreads();
    if (warp == 0) {
        int32_t w = lane < (int)(blockDim.x >> 5) ? s_warp[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            int32_t y = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= o) w += y;
        }
        s_warp[lane] = w;
    }
    __syncthreads();
    int32_t incl = x + (warp ? s_warp[warp - 1] : 0);
    if (total) *total = s_warp[(blockDim.x >> 5) - 1];
    __syncthreads();
    return incl - v;
}

// decoupled look-back status words: aggregate / inclusive prefix flags in the
// high half, the value in the low half
constexpr unsigned long long kLbAgg = 1ull << 32, kLbInc = 2ull << 32;

__device__ __forceinline__ unsigned long long lb_load(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

// warp 0 of a tile: publish the tile's aggregate, accumulate predecessor
// aggregates 32 at a time until an inclusive prefix is met, publish the
// inclusive prefix; returns the tile's exclusive prefix (all lanes)
__device__ __forceinline__ int32_t lb_prefix(unsigned long long *status, int64_t tile, int32_t agg) {
    const int lane = threadIdx.x & 31;
    if (tile == 0) {
        if (lane == 0) atomicExch(&status[0], kLbInc | (uint32_t)agg);
        return 0;
    }
    if (lane == 0) atomicExch(&status[tile], kLbAgg | (uint32_t)agg);
    int32_t prefix = 0;
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
    return prefix;
}

}  // namespace sfb
