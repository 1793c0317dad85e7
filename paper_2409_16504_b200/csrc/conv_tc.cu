// tcgen05 gather-GEMM-scatter for the P2ENet sparse convolutions (sm_100a).
//
// Reference semantics: sparse_conv (sparsenet.py:187-214)
//   out[v] = b + sum_{taps t} in[nbr(v,t)] @ W[t]   (ReLU)
// as an implicit GEMM: M = output voxels, N = Cout, K = taps x Cin.
//
// B200 mapping:
//  * CTA = 128 output rows (UMMA M=128, cta_group::1) x all Cout (UMMA N),
//    accumulator in TMEM (fp32, N columns), one elected thread issues
//    tcgen05.mma.kind::tf32 for the whole CTA.
//  * fp32 accuracy with tf32 tensor cores: every operand x is split into
//    hi = rn_tf32(x) and lo = rn_tf32(x - hi); D += Alo*Blo + Alo*Bhi +
//    Ahi*Blo + Ahi*Bhi (all four products, small terms first).
//    This keeps the conv at ~1e-6 relative error (bf16 inputs would break the
//    1e-3 Gaussian-parameter tolerance).
//  * per tap: the weight tile W[t] (pre-split, pre-laid-out in the UMMA
//    K-major canonical layout at load time) is staged by a TMA bulk copy
//    (cp.async.bulk, mbarrier complete_tx); the 128 neighbour rows are
//    gathered by the 128 threads (one row each, kernel map read coalesced),
//    split hi/lo in registers and written in the same canonical layout.
//    Two smem stages: the gather of tap t+1 overlaps the MMAs of tap t.
//  * coarse levels have few 128-row tiles (e.g. 4 at the bottleneck), so the
//    27 taps are split across CTAs (split-K) to fill the 148 SMs; partial
//    tiles go to a workspace and a deterministic reduce kernel sums them in
//    split order, adds the bias and applies ReLU (bitwise run-to-run stable).
#include <cooperative_groups.h>
#include <cuda.h>   // CUtensorMap (the encode entry point comes through the runtime)
#include <cuda_bf16.h>

#include <mutex>

#include "common.cuh"

namespace sfb {

namespace cg = cooperative_groups;

namespace {

constexpr int kM = 128;        // UMMA M / rows per CTA
constexpr int kThreadsTC = 128;

// canonical K-major SWIZZLE_NONE offset (floats) of element (row, k) in a
// [rows x KP] tile: 8-row groups of KP*8 floats, 4-wide k chunks of 32 floats
__host__ __device__ inline int core_off(int row, int k, int KP) {
    return (row >> 3) * (KP * 8) + (k >> 2) * 32 + (row & 7) * 4 + (k & 3);
}

// round-to-nearest (ties away) to tf32, as cvt.rna.tf32.f32 but in two
// integer ops (add half an ulp of tf32, clear the 13 dropped bits): the hi
// part of the split carries |x - hi| <= 2^-11 |x|, and lo = x - hi is exact
// in fp32 before its own rounding, so hi + lo keeps ~22 bits
__device__ __forceinline__ float tf32_round(float x) {
    return __uint_as_float((__float_as_uint(x) + 0x1000u) & 0xffffe000u);
}

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ uint64_t smem_desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= (uint64_t)((addr >> 4) & 0x3fff);
    d |= (uint64_t)((lbo >> 4) & 0x3fff) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3fff) << 32;
    d |= (uint64_t)1 << 46;  // descriptor version (sm_100)
    return d;                // base offset 0, lbo mode 0, SWIZZLE_NONE
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

// wait for the phase of `parity` to complete; a wait that never completes
// (a pipeline bug) traps after ~2^28 polls instead of hanging the GPU
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    const uint32_t addr = smem_u32(bar);
    for (uint32_t n = 0;; ++n) {
        uint32_t done;
        asm volatile(
            "{\n\t.reg .pred P;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, P;\n\t}"
            : "=r"(done)
            : "r"(addr), "r"(parity)
            : "memory");
        if (done) return;
        if (n > (1u << 28)) __trap();
    }
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void tma_bulk_g2s(void *dst, const void *src, uint32_t bytes,
                                             uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
            "r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

// TMA row gather (sm_100 tile::gather4): rows r0..r3 of the 2D feature
// tensor behind `tm` (box = KP columns x 1 row), columns from `col`, land as
// four consecutive KP-float rows at `dst`; rows past the tensor read as zeros
__device__ __forceinline__ void tma_gather4(void *dst, const CUtensorMap *tm, int col, int r0, int r1,
                                           int r2, int r3, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes "
        "[%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(tm)), "r"(col), "r"(r0), "r"(r1), "r"(r2), "r"(r3),
        "r"(smem_u32(bar))
        : "memory");
}

// 16-byte asynchronous global -> shared copy (LDGSTS); src_bytes = 0 zero-fills
__device__ __forceinline__ void cp_async16(void *dst, const void *src, uint32_t src_bytes) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(dst)), "l"(src),
                 "r"(src_bytes)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc,
                                         uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void mma_bf16(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc,
                                         uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void mma_commit(uint64_t *bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                     smem_u32(bar))
                 : "memory");
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float *v) {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
        "%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
          "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

// canonical K-major SWIZZLE_NONE offset (bf16 elements): 8-row groups of
// KP*8 elements, 8-wide k chunks of 64 elements (16-byte core rows)
__host__ __device__ inline int core_off_bf16(int row, int k, int KP) {
    return (row >> 3) * (KP * 8) + (k >> 3) * 64 + (row & 7) * 8 + (k & 7);
}

// BF = false: tf32 operands split hi + lo (fp32-accurate, 4 MMAs per k-step);
// BF = true: single bf16 operands (the north star's fast mode, 1 MMA)
template <int KP, int NP, bool BF = false>
struct TcShape {
    static constexpr int TERMS = BF ? 1 : 2;
    // taps per MMA batch: narrow inputs (Cin <= 16) take two taps per round of
    // gather / barrier / drain, halving the per-tap latency cost
    static constexpr int TAPB = KP == 16 ? 2 : 1;
    static constexpr int A_FLOATS = BF ? kM * KP / 2 : kM * KP;   // one term of one tap, 4-byte words
    static constexpr int B_FLOATS = BF ? NP * KP / 2 : NP * KP;
    static constexpr int A_TAP = TERMS * A_FLOATS, B_TAP = TERMS * B_FLOATS;   // per tap
    static constexpr int STAGE_FLOATS = TAPB * (A_TAP + B_TAP);
    // one stage: measured on config 2, a second stage buys no overlap the
    // co-resident CTAs of other items do not already give, and halving the
    // shared memory raises residency (0.379 vs 0.403 ms/frame with 8 lanes)
    static constexpr int STAGES = 1;
    // single stage with small weight tiles: the weights alone get a second
    // buffer, so batch k+1's tiles (TMA) are in flight while batch k is staged
    // and multiplied
    static constexpr bool BDB = STAGES == 1 && TAPB * B_TAP * 4 <= 32 * 1024;
    static constexpr int B_EXTRA = BDB ? TAPB * B_TAP : 0;
    // the stage buffers double as the cluster split-K reduction tile [kM][NP]
    static constexpr int BUF_FLOATS = STAGES * STAGE_FLOATS + B_EXTRA > kM * NP ? STAGES * STAGE_FLOATS + B_EXTRA
                                                                                 : kM * NP;
    // TMA-staged A rows (fp32 tf32x3 path, KP <= 64): a ring of RS raw stages
    // of TAPB x 128 gathered rows, filled RS-1 batches ahead by gather4
    static constexpr bool TMA_OK = !BF && KP <= 64;
    static constexpr int RS = KP <= 32 ? 3 : 2;
    static constexpr int RAW_FLOATS = TMA_OK ? RS * TAPB * kM * KP : 0;
    static constexpr int RAW_OFF = (BUF_FLOATS * 4 + 1023) / 1024 * 1024 / 4;   // floats, 1 KB aligned
    static constexpr int BAR_OFF = RAW_OFF + RAW_FLOATS;
    // + the kernel-map rows of one item's taps, sized per launch (src_rows)
    static constexpr int SMEM = BAR_OFF * 4 + 1024 + 128;
    // the ring is only laid out for the ring staging modes: register-prefetch
    // CTAs (the default) take the buffers + barriers + kernel-map rows only,
    // so more of them (and other lanes' kernels) fit on an SM
    static constexpr int smem_bytes(int src_rows, bool ring = true) {
        return (ring ? SMEM : RAW_OFF * 4 + 1024 + 128) + src_rows * kM * 4;
    }
    // two accumulators (tap t in buffer t % 2): the epilogue of tap t-1 reads
    // one while the MMAs of tap t write the other
    static constexpr uint32_t TMEM_COLS = 2 * NP <= 32 ? 32 : (2 * NP <= 64 ? 64 : (2 * NP <= 128 ? 128 : 256));
    // c_format F32; a/b_format TF32 (2) or BF16 (1); N >> 3; M >> 4
    static constexpr uint32_t IDESC = (1u << 4) | ((BF ? 1u : 2u) << 7) | ((BF ? 1u : 2u) << 10) |
                                      ((uint32_t)(NP >> 3) << 17) | ((uint32_t)(kM >> 4) << 24);
};

// split-K factor for a level: the smallest divisor c (<= 32) of the tap count
// with at most 32 taps per split and tiles*c >= target work items (else the
// largest such divisor); 0 when no divisor keeps a split within 32 taps
__host__ __device__ inline int choose_splits(int64_t tiles, int taps, int target) {
    int best = 0;
    for (int c = 1; c <= taps && c <= 32; ++c) {
        if (taps % c || taps / c > 32) continue;
        best = c;
        if (tiles * c >= target) break;
    }
    return best;
}
constexpr int kSplitTarget = 2 * 148;
constexpr int64_t kMaxPartialRows = 1480 * 128;

template <int KP, int NP, bool BF>
__global__ void __launch_bounds__(kThreadsTC)
k_conv_tc(const float *__restrict__ in, int ld_in, int cin, const int32_t *__restrict__ nbr,
          int64_t nbr_ld, const int64_t *__restrict__ d_m, int64_t m_fixed, int taps,
          const float *__restrict__ wtc, const float *__restrict__ bias, int cout, int relu,
          float *__restrict__ out, int ld_out, float *__restrict__ partial,
          const int32_t *__restrict__ row_map, const int32_t *__restrict__ tap_off,
          int cluster_splits, int src_rows, int vec4, const __grid_constant__ CUtensorMap tmA,
          int tma, int oob_row, int khalf) {
    // cluster mode (cluster_splits > 1): the splits of a tile are the CTAs of
    // one thread-block cluster; partial tiles meet in distributed shared
    // memory and each CTA reduces a slice of the tile's rows in split order —
    // no partial workspace in HBM, no reduce launch
    // tap-bucketed mode (transposed conv, tap_off != null): rows arrive grouped
    // by tap, each bucket padded to whole 128-row tiles (tap_off = 9 padded
    // offsets), nbr[row] is the row's parent (-1 pad), row_map[row] its output
    // row; every tile is ONE tap (K = Cin), so no split-K is needed
    using S = TcShape<KP, NP, BF>;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    float *stage_base = reinterpret_cast<float *>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    // A-row staging: 0 = register prefetch one batch ahead; 1 = TMA gather4
    // into the shared ring, RS batches ahead; 2 = each thread's own row by
    // cp.async (LDGSTS) into the ring, RS batches ahead (no barrier: a thread
    // only reads the row it copied)
    const bool use_tma = S::TMA_OK && tma == 1;
    const bool use_cpa = S::TMA_OK && tma == 2;
    const bool use_ring = use_tma || use_cpa;
    float *raw = stage_base + S::RAW_OFF;   // TMA ring [RS][TAPB][kM][KP] (ring modes only)
    const int bar_off = use_ring ? S::BAR_OFF : S::RAW_OFF;
    uint64_t *bar_full = reinterpret_cast<uint64_t *>(stage_base + bar_off);
    uint64_t *bar_done = bar_full + 2;   // indexed by batch parity (i & 1), phase i >> 1
    uint64_t *raw_full = bar_done + 2;   // [RS]: stage s's rows landed
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(raw_full + 4);
    // kernel-map rows of this item's taps: s_src[t - t0][tid]
    int32_t (*s_src)[kM] = reinterpret_cast<int32_t (*)[kM]>(stage_base + bar_off + 32);

    const int tid = threadIdx.x, warp = tid >> 5;
    const int64_t m = d_m ? *d_m : m_fixed;
    const int64_t tiles = (m + kM - 1) / kM;
    const int splits = tap_off ? 1 : (cluster_splits > 0 ? cluster_splits
                                                         : choose_splits(tiles, taps, kSplitTarget));
    const int tps = (taps + splits - 1) / splits;
    const int64_t work = tiles * splits;
    if ((int64_t)blockIdx.x >= work) return;   // uniform per CTA, before any collective
    if (!tap_off && tps > src_rows) __trap();  // the host sizes src_rows to the split

    if (tid == 0) {
        for (int s = 0; s < 2; ++s) {
            mbar_init(&bar_full[s], 1);
            mbar_init(&bar_done[s], 1);
        }
        for (int s = 0; s < 4; ++s) mbar_init(&raw_full[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(tmem_slot)),
                     "r"(S::TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = *tmem_slot;

    // Per-tap accumulation: each tap's MMAs start a fresh TMEM accumulator
    // and the threads add it into fp32 registers with IEEE adds. (Summing all
    // taps inside the tensor core loses ~20x more to its accumulator rounding
    // than FFMA does; per tap the K is only Cin.)
    const uint32_t lane_base = (uint32_t)(warp * 32) << 16;
    int issued = 0;  // MMA batches issued by this CTA so far (drives stage/phase)
    float acc[NP];
    auto drain = [&](int i) {   // add the accumulator of batch i into acc
        mbar_wait(&bar_done[i & 1], (i >> 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;");
        const uint32_t buf = tmem + lane_base + (uint32_t)((i & 1) * NP);
#pragma unroll
        for (int c = 0; c < NP; c += 16) {
            float v[16];
            tmem_ld16(buf + c, v);
#pragma unroll
            for (int q = 0; q < 16; ++q) acc[c + q] = __fadd_rn(acc[c + q], v[q]);
        }
        asm volatile("tcgen05.fence::before_thread_sync;");
    };
    __shared__ uint32_t s_mask[kThreadsTC / 32];
    for (int64_t wi = blockIdx.x; wi < work; wi += gridDim.x) {
        const int64_t row0 = (wi / splits) * kM;
        const int split = (int)(wi % splits);
        int t0 = split * tps, t1 = min(taps, t0 + tps);
        if (tap_off) {   // the bucket of this tile (khalf: its two K halves)
            int tb = 0;
            while (tb < 7 && row0 >= tap_off[tb + 1]) ++tb;
            t0 = khalf ? 2 * tb : tb;
            t1 = t0 + (khalf ? 2 : 1);
        }
        const int64_t row = row0 + tid;
#pragma unroll
        for (int c = 0; c < NP; ++c) acc[c] = 0.f;
        // prefetch the kernel map of every tap of the item (independent
        // coalesced loads) and OR the per-tap occupancy over the tile
        uint32_t mymask = 0;
        for (int t = t0; t < t1; ++t) {
            const int tr = khalf ? t >> 1 : t;   // the real tap of a K-half pseudo-tap
            const int32_t src = row < m ? nbr[(tap_off ? 0 : (int64_t)tr * nbr_ld) + row] : -1;
            s_src[t - t0][tid] = src;
            mymask |= (src >= 0 ? 1u : 0u) << (t - t0);
        }
        mymask = __reduce_or_sync(0xffffffffu, mymask);
        if ((tid & 31) == 0) s_mask[warp] = mymask;
        __syncthreads();
        uint32_t mask = 0;
#pragma unroll
        for (int w = 0; w < kThreadsTC / 32; ++w) mask |= s_mask[w];
        // register-prefetched gather: the rows of the next batch (up to TAPB
        // non-empty taps) are in flight while the current one is split,
        // staged and multiplied
        constexpr int TB = S::TAPB;
        float v[TB][KP];
        int nxt_t[TB], nxt_n = 0;
        auto take = [&]() {   // pop the next batch of taps off the mask
            nxt_n = 0;
            while (mask && nxt_n < TB) {
                nxt_t[nxt_n++] = t0 + __ffs(mask) - 1;
                mask &= mask - 1;
            }
        };
        auto fetch = [&]() {
#pragma unroll
            for (int q = 0; q < TB; ++q) {
                const int32_t src = q < nxt_n ? s_src[nxt_t[q] - t0][tid] : -1;
                // khalf: pseudo-tap t reads channels [KP (t & 1), +KP) of the row
                const int koff = khalf && q < nxt_n ? KP * (nxt_t[q] & 1) : 0;
                const int cin_q = cin - koff;
                const float *x = src >= 0 ? in + (int64_t)src * ld_in + koff : nullptr;
                if (vec4) {   // 16-byte rows (cin, ld_in multiples of 4, aligned base)
#pragma unroll
                    for (int k = 0; k < KP; k += 4) {
                        const float4 f = (x && k < cin_q) ? __ldg(reinterpret_cast<const float4 *>(x + k))
                                                          : make_float4(0.f, 0.f, 0.f, 0.f);
                        v[q][k] = f.x;
                        v[q][k + 1] = f.y;
                        v[q][k + 2] = f.z;
                        v[q][k + 3] = f.w;
                    }
                } else {
#pragma unroll
                    for (int k = 0; k < KP; ++k) v[q][k] = (x && k < cin_q) ? __ldg(x + k) : 0.f;
                }
            }
        };
        // TMA mode: warp 0 gathers the rows of the item's batches RS ahead into
        // the raw ring (all threads track the batch sequence, only warp 0
        // issues); the threads then read their rows from shared memory instead
        // of holding a register prefetch
        uint32_t pmask = mask;
        const int g0 = issued;   // global batch index of this item's first batch
        int npref = 0;
        auto prefetch = [&]() {
            int pt[TB], pn = 0;
            while (pmask && pn < TB) {
                pt[pn++] = t0 + __ffs(pmask) - 1;
                pmask &= pmask - 1;
            }
            if (use_cpa) {   // my row of each tap of the batch; an empty group past the last batch
                if (pn > 0) {
                    const int stg = (g0 + npref++) % S::RS;
                    float *dst = raw + (size_t)stg * TB * kM * KP + (size_t)tid * KP;
                    for (int q = 0; q < pn; ++q) {
                        const int32_t r = s_src[pt[q] - t0][tid];
                        const float *src = r >= 0 ? in + (int64_t)r * ld_in : in;
#pragma unroll
                        for (int k = 0; k < KP; k += 4)
                            cp_async16(dst + (size_t)q * kM * KP + k, src + k, r >= 0 ? 16u : 0u);
                    }
                }
                cp_async_commit();
                return;
            }
            if (pn == 0) return;
            const int stg = (g0 + npref++) % S::RS;
            if (warp == 0) {
                if (tid == 0) mbar_expect_tx(&raw_full[stg], (uint32_t)(pn * kM * KP * 4));
                __syncwarp();
                float *dst = raw + (size_t)stg * TB * kM * KP;
                for (int q = 0; q < pn; ++q) {
                    const int32_t *sr = s_src[pt[q] - t0] + 4 * tid;
                    const int r0 = sr[0] >= 0 ? sr[0] : oob_row, r1 = sr[1] >= 0 ? sr[1] : oob_row,
                              r2 = sr[2] >= 0 ? sr[2] : oob_row, r3 = sr[3] >= 0 ? sr[3] : oob_row;
                    tma_gather4(dst + (size_t)q * kM * KP + (size_t)4 * tid * KP, &tmA, 0, r0, r1, r2, r3,
                                &raw_full[stg]);
                }
            }
        };
        take();
        if (use_ring) {
            for (int k = 0; k < S::RS; ++k) prefetch();
        } else if (nxt_n) {
            fetch();
        }
        // weights: with two stages, batch k+1's tiles are fetched (TMA) as soon
        // as batch k-1 has drained, so their latency hides behind batch k
        auto b_slot = [&](int slot) {   // weight buffer of a slot
            return S::BDB ? (slot ? stage_base + S::STAGE_FLOATS : stage_base + TB * S::A_TAP)
                          : stage_base + slot * S::STAGE_FLOATS + TB * S::A_TAP;
        };
        auto load_w = [&](const int *tt, int nt, int slot) {
            const uint32_t bytes = (uint32_t)(nt * S::B_TAP * 4);
            float *B = b_slot(slot);
            mbar_expect_tx(&bar_full[slot], bytes);
            for (int q = 0; q < nt; ++q)
                tma_bulk_g2s(B + q * S::B_TAP, wtc + (size_t)tt[q] * S::B_TAP, S::B_TAP * 4, &bar_full[slot]);
        };
        int item_issued = 0;
        while (nxt_n) {
            int cur_t[TB];
            const int cur_n = nxt_n;
#pragma unroll
            for (int q = 0; q < TB; ++q) cur_t[q] = nxt_t[q];
            const int s = issued % S::STAGES;
            // weight slot and its barrier phase: per stage, or per batch parity (BDB)
            const int ws = S::BDB ? (issued & 1) : s;
            const int use = S::BDB ? (issued >> 1) : issued / S::STAGES;
            float *A_base = stage_base + s * S::STAGE_FLOATS;
            float *B_base = b_slot(ws);
            // stage free again: the batch that last used it (i - STAGES) has
            // completed. Batch barriers alternate by batch parity, so no wait
            // below can alias a later phase: the next commit to the barrier
            // of batch j is batch j+2, issued only after j is drained.
            if (issued >= S::STAGES) {
                const int j = issued - S::STAGES;
                mbar_wait(&bar_done[j & 1], (j >> 1) & 1);
            }
            if (tid == 0 && ((S::STAGES == 1 && !S::BDB) || item_issued == 0)) load_w(cur_t, cur_n, ws);
            if (use_ring) {   // this batch's rows, fetched RS batches ago
                const int stg = issued % S::RS;
                if (use_tma) mbar_wait(&raw_full[stg], (uint32_t)(issued / S::RS) & 1u);
                else cp_async_wait<S::RS - 1>();   // my oldest group: this batch
                const float *src = raw + (size_t)stg * TB * kM * KP + (size_t)tid * KP;
#pragma unroll
                for (int q = 0; q < TB; ++q) {
                    if (q >= cur_n) break;
#pragma unroll
                    for (int k = 0; k < KP; k += 4) {
                        const float4 f = *reinterpret_cast<const float4 *>(src + (size_t)q * kM * KP + k);
                        v[q][k] = f.x;
                        v[q][k + 1] = f.y;
                        v[q][k + 2] = f.z;
                        v[q][k + 3] = f.w;
                    }
                }
            }
            // my row of each tap of the batch in the canonical layout: bf16, or tf32 hi/lo
#pragma unroll
            for (int q = 0; q < TB; ++q) {
                if (q >= cur_n) break;
                float *A_hi = A_base + q * S::A_TAP;
                float *A_lo = A_hi + S::A_FLOATS;   // tf32 only
                if constexpr (BF) {
                    uint16_t *A16 = reinterpret_cast<uint16_t *>(A_hi);
#pragma unroll
                    for (int c = 0; c < KP / 8; ++c) {
                        uint32_t w[4];
#pragma unroll
                        for (int h = 0; h < 4; ++h) {
                            const __nv_bfloat162 b2 =
                                __floats2bfloat162_rn(v[q][8 * c + 2 * h], v[q][8 * c + 2 * h + 1]);
                            w[h] = *reinterpret_cast<const uint32_t *>(&b2);
                        }
                        *reinterpret_cast<uint4 *>(A16 + core_off_bf16(tid, 8 * c, KP)) =
                            make_uint4(w[0], w[1], w[2], w[3]);
                    }
                } else {
#pragma unroll
                    for (int c = 0; c < KP / 4; ++c) {
                        float4 hi, lo;
                        hi.x = tf32_round(v[q][4 * c]);
                        hi.y = tf32_round(v[q][4 * c + 1]);
                        hi.z = tf32_round(v[q][4 * c + 2]);
                        hi.w = tf32_round(v[q][4 * c + 3]);
                        lo.x = tf32_round(v[q][4 * c] - hi.x);
                        lo.y = tf32_round(v[q][4 * c + 1] - hi.y);
                        lo.z = tf32_round(v[q][4 * c + 2] - hi.z);
                        lo.w = tf32_round(v[q][4 * c + 3] - hi.w);
                        const int off = core_off(tid, 4 * c, KP);
                        *reinterpret_cast<float4 *>(A_hi + off) = hi;
                        *reinterpret_cast<float4 *>(A_lo + off) = lo;
                    }
                }
            }
            take();
            if (nxt_n && !use_ring) fetch();   // next batch's rows, in flight from here
            // next batch's weights: its slot was last read by batch issued-1,
            // complete since the wait above
            if (S::BDB && tid == 0 && nxt_n) load_w(nxt_t, nxt_n, (issued + 1) & 1);
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncthreads();   // also orders the last drain's TMEM reads before these MMAs
            if (use_ring) prefetch();   // batch issued + RS into the stage just read
            if (tid == 0) {
                mbar_wait(&bar_full[ws], use & 1);
                asm volatile("tcgen05.fence::after_thread_sync;");
                const uint32_t lbo = 128, sbo = BF ? KP * 16 : KP * 32;
                const uint32_t dst = tmem + (uint32_t)((issued & 1) * NP);
                for (int q = 0; q < cur_n; ++q) {
                    const float *A_hi = A_base + q * S::A_TAP, *A_lo = A_hi + S::A_FLOATS;
                    const float *B_hi = B_base + q * S::B_TAP, *B_lo = B_hi + S::B_FLOATS;
                    if constexpr (BF) {
#pragma unroll
                        for (int ks = 0; ks < KP / 16; ++ks)
                            mma_bf16(dst, smem_desc(smem_u32(A_hi) + ks * 256, lbo, sbo),
                                     smem_desc(smem_u32(B_hi) + ks * 256, lbo, sbo), S::IDESC,
                                     (q > 0 || ks > 0) ? 1u : 0u);
                    } else {
#pragma unroll
                        for (int ks = 0; ks < KP / 8; ++ks) {
                            const uint64_t ahi = smem_desc(smem_u32(A_hi) + ks * 256, lbo, sbo);
                            const uint64_t alo = smem_desc(smem_u32(A_lo) + ks * 256, lbo, sbo);
                            const uint64_t bhi = smem_desc(smem_u32(B_hi) + ks * 256, lbo, sbo);
                            const uint64_t blo = smem_desc(smem_u32(B_lo) + ks * 256, lbo, sbo);
                            // small terms first: lo*lo, lo*hi, hi*lo, then hi*hi
                            mma_tf32(dst, alo, blo, S::IDESC, (q > 0 || ks > 0) ? 1u : 0u);
                            mma_tf32(dst, alo, bhi, S::IDESC, 1u);
                            mma_tf32(dst, ahi, blo, S::IDESC, 1u);
                            mma_tf32(dst, ahi, bhi, S::IDESC, 1u);
                        }
                    }
                }
                mma_commit(&bar_done[issued & 1]);
            }
            if (item_issued > 0) drain(issued - 1);   // previous batch, overlapping this one's MMAs
            if (S::STAGES == 2 && tid == 0 && nxt_n)   // slot of batch issued-1 is free now
                load_w(nxt_t, nxt_n, (issued + 1) & 1);
            ++issued;
            ++item_issued;
        }
        if (item_issued > 0) drain(issued - 1);
        if (cluster_splits > 1) {
            // my partial tile into my shared memory (the stage buffers are idle
            // now), cluster barrier, then rows [r0, r1) of the tile summed over
            // the cluster's CTAs in split (= rank) order
            float *red = stage_base;   // [kM][NP]
#pragma unroll
            for (int c = 0; c < NP; c += 4)
                *reinterpret_cast<float4 *>(red + tid * NP + c) =
                    make_float4(acc[c], acc[c + 1], acc[c + 2], acc[c + 3]);
            cg::cluster_group cl = cg::this_cluster();
            cl.sync();
            const int rank = (int)cl.block_rank();
            const int per = (kM + splits - 1) / splits;
            const int r0 = rank * per, r1 = min(kM, r0 + per);
            for (int e = tid; e < (r1 - r0) * NP; e += kThreadsTC) {
                const int rr = r0 + e / NP, c = e % NP;
                const int64_t grow = row0 + rr;
                if (c >= cout || grow >= m) continue;
                float sum = 0.f;
                for (int k = 0; k < splits; ++k) sum += cl.map_shared_rank(red, k)[rr * NP + c];
                const float v = sum + bias[c];
                out[grow * (int64_t)ld_out + c] = relu ? fmaxf(v, 0.f) : v;
            }
            cl.sync();   // peers keep their shared memory until every slice is read
        } else if (row < m) {
            if (splits > 1) {
                float *p = partial + ((size_t)split * m + row) * NP;
#pragma unroll
                for (int c = 0; c < NP; c += 4)
                    *reinterpret_cast<float4 *>(p + c) = make_float4(acc[c], acc[c + 1], acc[c + 2], acc[c + 3]);
            } else {
                const int64_t orow = row_map ? (int64_t)row_map[row] : row;
                if (orow >= 0) {
                    float *o = out + orow * (int64_t)ld_out;
#pragma unroll
                    for (int c = 0; c < NP; ++c)
                        if (c < cout) {
                            float v = acc[c] + bias[c];
                            o[c] = relu ? fmaxf(v, 0.f) : v;
                        }
                }
            }
        }
        // all TMEM reads done before the next item's MMAs overwrite the accumulators
        __syncthreads();
        asm volatile("tcgen05.fence::after_thread_sync;");
    }
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                     "r"(S::TMEM_COLS));
}

// deterministic split-K reduction: out = act(b + sum_s partial[s]) in split order
__global__ void k_splitk_reduce(const float *__restrict__ partial, const int64_t *__restrict__ d_m,
                                int64_t m_fixed, int taps, int np, const float *__restrict__ bias,
                                int cout, int relu, float *__restrict__ out, int ld_out) {
    const int64_t m = d_m ? *d_m : m_fixed;
    const int splits = choose_splits((m + kM - 1) / kM, taps, kSplitTarget);
    if (splits == 1) return;
    SFB_FOR(i, m * cout) {
        const int64_t r = i / cout;
        const int c = (int)(i % cout);
        float s = 0.f;
        for (int k = 0; k < splits; ++k) s += partial[((size_t)k * m + r) * np + c];
        const float v = s + bias[c];
        out[r * ld_out + c] = relu ? fmaxf(v, 0.f) : v;
    }
}

// W[t][ci][co] -> per tap [hi | lo] tiles of [NP x KP] in the canonical layout
__global__ void k_prep_weights(const float *__restrict__ w, int taps, int cin, int cout, int KP,
                               int NP, float *__restrict__ wtc) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    int64_t per = (int64_t)NP * KP;
    if (i >= taps * per) return;
    int t = (int)(i / per);
    int rem = (int)(i % per);
    int n = rem / KP, k = rem % KP;
    float x = (n < cout && k < cin) ? w[((size_t)t * cin + k) * cout + n] : 0.f;
    float hi = tf32_round(x), lo = tf32_round(x - hi);
    float *base = wtc + (size_t)t * 2 * per;
    int off = core_off(n, k, KP);
    base[off] = hi;
    base[per + off] = lo;
}

__global__ void k_prep_weights_bf16(const float *__restrict__ w, int taps, int cin, int cout, int KP,
                                    int NP, uint16_t *__restrict__ wbf) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    int64_t per = (int64_t)NP * KP;
    if (i >= taps * per) return;
    int t = (int)(i / per);
    int rem = (int)(i % per);
    int n = rem / KP, k = rem % KP;
    float x = (n < cout && k < cin) ? w[((size_t)t * cin + k) * cout + n] : 0.f;
    const __nv_bfloat16 b = __float2bfloat16_rn(x);
    wbf[(size_t)t * per + core_off_bf16(n, k, KP)] = *reinterpret_cast<const uint16_t *>(&b);
}

int pad_k(int c) { return c <= 16 ? 16 : (c <= 32 ? 32 : (c <= 64 ? 64 : 128)); }
int pad_n(int c) { return c <= 16 ? 16 : (c <= 32 ? 32 : (c <= 64 ? 64 : (c <= 128 ? 128 : 256))); }

// cuTensorMapEncodeTiled through the runtime's driver entry point (the
// library links only the static cudart)
using EncodeTiled = CUresult (*)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *,
                                 const cuuint64_t *, const cuuint64_t *, const cuuint32_t *,
                                 const cuuint32_t *, CUtensorMapInterleave, CUtensorMapSwizzle,
                                 CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiled encode_tiled() {
    static EncodeTiled fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiled>(p);
    });
    return fn;
}

// Row-gather tensor map of a feature matrix [rows x ld] fp32: box = KP columns
// x 1 row (tile::gather4 takes 4 row indices); false when not expressible
bool feature_map(CUtensorMap *tm, const float *base, int ld, int64_t rows, int KP) {
    EncodeTiled enc = encode_tiled();
    if (!enc || rows < 1 || rows >= (int64_t(1) << 31) || (ld % 4) != 0 || ld < KP ||
        (reinterpret_cast<uintptr_t>(base) & 15) != 0)
        return false;
    const cuuint64_t dims[2] = {(cuuint64_t)ld, (cuuint64_t)rows};
    const cuuint64_t strides[1] = {(cuuint64_t)ld * 4};
    const cuuint32_t box[2] = {(cuuint32_t)KP, 1u};
    const cuuint32_t es[2] = {1u, 1u};
    return enc(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float *>(base), dims, strides, box, es,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
               CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int KP, int NP, bool BF>
void launch_tc(sfb_ctx *ctx, const NetLayer &L, const float *in, int ld_in, const int32_t *nbr,
               int64_t nbr_ld, const int64_t *d_m, int64_t m_bound, int relu, float *out,
               int ld_out, int64_t m_grid, const int32_t *row_map, const int32_t *tap_off,
               int csplit_req, int khalf = 0) {
    using S = TcShape<KP, NP, BF>;
    set_max_dyn_smem(reinterpret_cast<const void *>(k_conv_tc<KP, NP, BF>), S::smem_bytes(32));
    const int64_t tiles_bound = (m_grid + kM - 1) / kM;
    // Split-K. csplit_req > 1: the splits of a tile form a thread-block
    // cluster (size fixed by the caller from the layer's place in the
    // network, never from size hints, so the summation order — hence the
    // result — does not depend on launch-time bounds); 1: no split; < 0:
    // splits chosen on the device from the actual row count, partials
    // reduced by k_splitk_reduce.
    const int csplit = tap_off ? 1 : (csplit_req > 8 ? 8 : csplit_req);
    // taps one work item can cover: one per bucket tile; taps/csplit in a
    // cluster; with device-chosen splits the split may be 1, so all taps
    const int taps_eff = khalf ? 2 * L.taps : L.taps;   // khalf: pseudo-taps of 64 channels
    const int src_rows = tap_off ? (khalf ? 2 : 1)
                                 : (csplit >= 1 ? (taps_eff + csplit - 1) / csplit : std::min(taps_eff, 32));
    const int vec4 = (L.cin % 4 == 0 && ld_in % 4 == 0 && (reinterpret_cast<uintptr_t>(in) & 15) == 0) ? 1 : 0;
    // A rows by TMA gather (tcgen05 tf32x3 path, full-width rows, multi-tap items)
    CUtensorMap tm{};
    int tma = 0;
    if (S::TMA_OK && !tap_off && !khalf && L.cin == KP && vec4) {
        if (ctx->conv_stage == 1 && feature_map(&tm, in, ld_in, m_bound, KP)) tma = 1;
        else if (ctx->conv_stage == 2) tma = 2;
    }
    const int oob_row = (int)std::min<int64_t>(m_bound, INT32_MAX);
    if (csplit > 1) {
        const int64_t m_tiles = (m_bound + kM - 1) / kM;   // grid covers the device count's bound
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3((unsigned)(std::max<int64_t>(1, std::min(tiles_bound, m_tiles)) * csplit));
        cfg.blockDim = dim3(kThreadsTC);
        cfg.dynamicSmemBytes = S::smem_bytes(src_rows, tma != 0);
        cfg.stream = ctx->stream;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = (unsigned)csplit;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        const float *wts = BF ? reinterpret_cast<const float *>(L.w_bf16) : khalf ? L.w_tc_k2 : L.w_tc;
        SFB_CUDA(cudaLaunchKernelEx(&cfg, k_conv_tc<KP, NP, BF>, in, ld_in, L.cin, nbr, nbr_ld, d_m,
                                    m_bound, taps_eff, wts, L.b, L.cout, relu, out, ld_out,
                                    static_cast<float *>(nullptr), row_map, tap_off, csplit, src_rows, vec4,
                                    tm, tma, oob_row, khalf));
        return;
    }
    const int64_t work_bound = (tap_off || csplit == 1)
                                   ? tiles_bound
                                   : tiles_bound * choose_splits(tiles_bound, taps_eff, kSplitTarget);
    const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(work_bound, kSplitTarget));
    float *partial = ctx->arena.alloc<float>((size_t)std::min<int64_t>(kMaxPartialRows,
                                                                       32 * m_bound) * NP);
    const float *wts = BF ? reinterpret_cast<const float *>(L.w_bf16) : khalf ? L.w_tc_k2 : L.w_tc;
    k_conv_tc<KP, NP, BF><<<grid, kThreadsTC, S::smem_bytes(src_rows, tma != 0), ctx->stream>>>(
        in, ld_in, L.cin, nbr, nbr_ld, d_m, m_bound, taps_eff, wts, L.b, L.cout, relu, out, ld_out,
        partial, row_map, tap_off, csplit == 1 ? 1 : 0, src_rows, vec4, tm, tma, oob_row, khalf);
    SFB_CHECK_LAUNCH();
    if (tap_off || csplit == 1) return;   // no split-K partials
    k_splitk_reduce<<<dgrid(std::min<int64_t>(m_grid, kMaxPartialRows) * L.cout, 256), 256, 0,
                      ctx->stream>>>(partial, d_m, m_bound, taps_eff, NP, L.b, L.cout, relu, out,
                                     ld_out);
    SFB_CHECK_LAUNCH();
}

}  // namespace

bool conv_tc_supported(const NetLayer &L) {
    if (L.kind != 0 && L.kind != 1) return false;   // conv, or transposed conv as an 8-tap map
    if (choose_splits(1, L.taps, kSplitTarget) == 0) return false;   // > 32 taps per split
    int kp = pad_k(L.cin), np = pad_n(L.cout);
    if (L.cin > 128 || L.cout > 128) return false;
    const int tapb = kp == 16 ? 2 : 1;
    size_t stage = (size_t)tapb * (2 * kM * kp + 2 * np * kp) * 4;
    return stage + 2048 <= 200 * 1024;
}

// W[t][ci][co] -> per pseudo-tap p = 2t + h the [hi | lo] tiles of [NP x H]
// covering input channels [H h, H h + H) (K-split transposed convs, H = half
// the padded input width)
__global__ void k_prep_weights_k2(const float *__restrict__ w, int taps, int cin, int cout, int H,
                                  int NP, float *__restrict__ wtc) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t per = (int64_t)NP * H;
    if (i >= 2 * taps * per) return;
    const int pt = (int)(i / per), t = pt >> 1, h = pt & 1;
    const int rem = (int)(i % per);
    const int n = rem / H, k = rem % H, ci = H * h + k;
    const float x = (n < cout && ci < cin) ? w[((size_t)t * cin + ci) * cout + n] : 0.f;
    const float hi = tf32_round(x), lo = tf32_round(x - hi);
    float *base = wtc + (size_t)pt * 2 * per;
    const int off = core_off(n, k, H);
    base[off] = hi;
    base[per + off] = lo;
}

void prepare_tc_weights(sfb_ctx *ctx, NetLayer &L) {
    L.cin_pad = pad_k(L.cin);
    L.cout_pad = pad_n(L.cout);
    size_t n = (size_t)L.taps * 2 * L.cin_pad * L.cout_pad;
    SFB_CUDA(cudaMalloc(&L.w_tc, n * sizeof(float)));
    int64_t total = (int64_t)L.taps * L.cin_pad * L.cout_pad;
    k_prep_weights<<<grid_for(total, 256), 256, 0, ctx->stream>>>(L.w, L.taps, L.cin, L.cout,
                                                                  L.cin_pad, L.cout_pad, L.w_tc);
    if (L.kind == 1 && L.cin_pad >= 64) {
        SFB_CUDA(cudaMalloc(&L.w_tc_k2, n * sizeof(float)));
        k_prep_weights_k2<<<grid_for(total, 256), 256, 0, ctx->stream>>>(
            L.w, L.taps, L.cin, L.cout, L.cin_pad / 2, L.cout_pad, L.w_tc_k2);
    }
    SFB_CUDA(cudaMalloc(&L.w_bf16, (size_t)total * sizeof(uint16_t)));
    k_prep_weights_bf16<<<grid_for(total, 256), 256, 0, ctx->stream>>>(L.w, L.taps, L.cin, L.cout,
                                                                       L.cin_pad, L.cout_pad, L.w_bf16);
    SFB_CHECK_LAUNCH();
}

void conv_layer_tc(sfb_ctx *ctx, const NetLayer &L, const float *in, int ld_in, const int32_t *nbr,
                   int64_t nbr_ld, const int64_t *d_m, int64_t m_bound, int relu, float *out,
                   int ld_out, int64_t m_grid, const int32_t *row_map, const int32_t *tap_off,
                   int csplit) {
    const bool bf = ctx->net_mode == SFB_NET_TC_BF16;
    // 64- and 128-wide transposed convs as two K halves (both the bucketed
    // and the 8-tap map path, so they stay bitwise equal): half the staged
    // tile per CTA, the halves summed in fp32 registers
    if (!bf && L.kind == 1 && L.cin_pad >= 64 && L.w_tc_k2) {
#define SFB_TC_K2(K, N)                                                                         \
        if (L.cin_pad == 2 * K && L.cout_pad == N)                                              \
            return launch_tc<K, N, false>(ctx, L, in, ld_in, nbr, nbr_ld, d_m, m_bound, relu, out, \
                                          ld_out, m_grid, row_map, tap_off, csplit, 1);
        SFB_TC_K2(64, 16) SFB_TC_K2(64, 32) SFB_TC_K2(64, 64)
        SFB_TC_K2(32, 16) SFB_TC_K2(32, 32) SFB_TC_K2(32, 64)
#undef SFB_TC_K2
    }
#define SFB_TC_CASE(K, N)                                                                 \
    if (L.cin_pad == K && L.cout_pad == N) {                                              \
        if (bf)                                                                           \
            launch_tc<K, N, true>(ctx, L, in, ld_in, nbr, nbr_ld, d_m, m_bound, relu, out, ld_out, \
                                  m_grid, row_map, tap_off, csplit);                      \
        else                                                                              \
            launch_tc<K, N, false>(ctx, L, in, ld_in, nbr, nbr_ld, d_m, m_bound, relu, out, ld_out, \
                                   m_grid, row_map, tap_off, csplit);                     \
        return;                                                                           \
    }
    SFB_TC_CASE(16, 16) SFB_TC_CASE(16, 32) SFB_TC_CASE(16, 64) SFB_TC_CASE(16, 128)
    SFB_TC_CASE(32, 16) SFB_TC_CASE(32, 32) SFB_TC_CASE(32, 64) SFB_TC_CASE(32, 128)
    SFB_TC_CASE(64, 16) SFB_TC_CASE(64, 32) SFB_TC_CASE(64, 64) SFB_TC_CASE(64, 128)
    SFB_TC_CASE(128, 16) SFB_TC_CASE(128, 32) SFB_TC_CASE(128, 64)
#undef SFB_TC_CASE
    throw Error(SFB_ERR_STATE, "tcgen05 conv: unsupported channel padding");
}

}  // namespace sfb
