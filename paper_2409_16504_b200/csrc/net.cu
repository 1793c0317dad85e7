// P2ENet on the device: P2EN weight loading, gather-GEMM-scatter sparse
// convolutions, pruned transposed convolutions, the fused 2-layer MLP head and
// the head activations (reference: sparsenet.py:187-341, 390-434).
//
// Data layout in HBM, per level l (stride 2^l): canonical voxel coords
// (M_l,3) int32, a tap-major kernel map (27, M_l) int32, and float32
// row-major features. The decoder's skip concatenation [up, skip]
// (sparsenet.py:278-282) is never materialised by a copy: the encoder conv of
// level l writes its output straight into columns [C_up, C_up+C_skip) of the
// level-l concat buffer, and the transposed conv later fills columns
// [0, C_up) of the same rows.
//
// Arithmetic modes: SFB_NET_SIMT_F32 (fp32 FFMA gather-GEMM, the parity
// anchor) and SFB_NET_TC_TF32X3 (tcgen05 tensor cores, tf32 hi/lo split
// giving fp32-level accuracy; conv_tc.cu).
#include <cmath>

#include "common.cuh"

namespace sfb {

void conv_layer_tc(sfb_ctx *ctx, const NetLayer &L, const float *in, int ld_in, const int32_t *nbr,
                   int64_t nbr_ld, const int64_t *d_m, int64_t m_bound, int relu, float *out,
                   int ld_out, int64_t m_grid, const int32_t *row_map = nullptr,
                   const int32_t *tap_off = nullptr, int csplit = -1);
bool conv_tc_supported(const NetLayer &L);
void prepare_tc_weights(sfb_ctx *ctx, NetLayer &L);

// ------------------------------------------------------------ weight loading
namespace {
struct Cursor {
    const uint8_t *p;
    size_t n, pos = 0;
    const uint8_t *take(size_t k) {
        if (pos + k > n) throw Error(SFB_ERR_ARG, "weights: file ends inside a field");
        const uint8_t *r = p + pos;
        pos += k;
        return r;
    }
    uint32_t u32() {
        uint32_t v;
        std::memcpy(&v, take(4), 4);
        return v;
    }
    uint8_t u8() { return *take(1); }
};
}  // namespace

void net_load(sfb_ctx *ctx, const void *blob, size_t nbytes) {
    Cursor c{static_cast<const uint8_t *>(blob), nbytes};
    if (std::memcmp(c.take(4), "P2EN", 4) != 0)
        throw Error(SFB_ERR_ARG, "weights: not a weight file (bad magic)");
    uint32_t version = c.u32();
    if (version != 1) throw Error(SFB_ERR_ARG, "weights: unsupported version " + std::to_string(version));
    uint32_t levels = c.u32();
    std::vector<int> enc(c.u32()), dec;
    for (auto &e : enc) e = (int)c.u32();
    dec.resize(c.u32());
    for (auto &d : dec) d = (int)c.u32();
    int head_hidden = (int)c.u32();
    uint32_t count = c.u32();
    SFB_REQUIRE(enc.size() >= 3 && dec.size() == enc.size() - 2 && levels == dec.size(),
                "weights: topology does not match its plan");
    // expected layer chain (sparsenet.py:108-118)
    struct Want { int kind, cin, cout; };
    std::vector<Want> want;
    for (size_t i = 0; i + 1 < enc.size(); ++i) want.push_back({0, enc[i], enc[i + 1]});
    int width = enc.back();
    for (size_t j = 0; j < dec.size(); ++j) {
        want.push_back({1, width, dec[j]});
        width = dec[j] + enc[enc.size() - 2 - j];
    }
    want.push_back({2, width, head_hidden});
    want.push_back({2, head_hidden, 14});
    SFB_REQUIRE(count == want.size(), "weights: layer count does not match the plan");

    Net fresh;
    try {
        for (uint32_t i = 0; i < count; ++i) {
            NetLayer L;
            L.kind = c.u8();
            L.kernel = c.u8();
            L.cin = (int)c.u32();
            L.cout = (int)c.u32();
            SFB_REQUIRE(L.kind == want[i].kind && L.cin == want[i].cin && L.cout == want[i].cout,
                        "weights: layer " + std::to_string(i) + " disagrees with the plan");
            if (L.kind == 0) SFB_REQUIRE(L.kernel >= 1 && (L.kernel & 1), "weights: conv kernels must be odd");
            if (L.kind == 1) SFB_REQUIRE(L.kernel == 2, "weights: transposed_conv kernel is fixed at 2");
            if (L.kind == 2) SFB_REQUIRE(L.kernel == 1, "weights: mlp kernel is fixed at 1");
            L.taps = L.kind == 2 ? 1 : L.kernel * L.kernel * L.kernel;
            size_t nw = (size_t)L.taps * L.cin * L.cout;
            const uint8_t *w = c.take(4 * nw);
            const uint8_t *b = c.take(4 * (size_t)L.cout);
            SFB_CUDA(cudaMalloc(&L.w, 4 * nw));
            fresh.allocations.push_back(L.w);
            SFB_CUDA(cudaMalloc(&L.b, 4 * (size_t)L.cout));
            fresh.allocations.push_back(L.b);
            SFB_CUDA(cudaMemcpyAsync(L.w, w, 4 * nw, cudaMemcpyHostToDevice, ctx->stream));
            SFB_CUDA(cudaMemcpyAsync(L.b, b, 4 * (size_t)L.cout, cudaMemcpyHostToDevice, ctx->stream));
            fresh.layers.push_back(L);
        }
        SFB_REQUIRE(c.pos == c.n, "weights: trailing bytes after last layer");
        for (auto &L : fresh.layers)
            if (conv_tc_supported(L)) {
                prepare_tc_weights(ctx, L);
                fresh.allocations.push_back(L.w_tc);
                fresh.allocations.push_back(L.w_bf16);
                if (L.w_tc_k2) fresh.allocations.push_back(L.w_tc_k2);
            }
        SFB_CUDA(cudaStreamSynchronize(ctx->stream));
    } catch (...) {
        fresh.release();
        throw;
    }
    ctx->net.release();
    ctx->net = fresh;
    ctx->net.enc = enc;
    ctx->net.dec = dec;
    ctx->net.head_hidden = head_hidden;
    ctx->net.levels = (int)levels;
    ctx->net.loaded = true;
}

// A standalone layer (sparse_conv / transposed_conv_pruned called with their
// own weights, sparsenet.py:187, 217) kept in ctx->adhoc.
void layer_set(sfb_ctx *ctx, int kind, int kernel, int cin, int cout, const float *w_host,
               const float *b_host) {
    SFB_REQUIRE(kind == 0 || kind == 1, "only conv / transposed_conv layers can be set");
    SFB_REQUIRE(cin > 0 && cout > 0, "channel counts must be positive");
    if (kind == 0) SFB_REQUIRE(kernel >= 1 && (kernel & 1), "conv kernels must be odd");
    if (kind == 1) SFB_REQUIRE(kernel == 2, "transposed_conv kernel is fixed at 2");
    NetLayer &L = ctx->adhoc;
    for (void *p : {(void *)L.w, (void *)L.b, (void *)L.w_tc, (void *)L.w_bf16, (void *)L.w_tc_k2})
        if (p) cudaFree(p);
    L = NetLayer{};
    L.kind = kind;
    L.kernel = kernel;
    L.cin = cin;
    L.cout = cout;
    L.taps = kernel * kernel * kernel;
    size_t nw = (size_t)L.taps * cin * cout;
    SFB_CUDA(cudaMalloc(&L.w, 4 * nw));
    SFB_CUDA(cudaMalloc(&L.b, 4 * (size_t)cout));
    SFB_CUDA(cudaMemcpyAsync(L.w, w_host, 4 * nw, cudaMemcpyHostToDevice, ctx->stream));
    SFB_CUDA(cudaMemcpyAsync(L.b, b_host, 4 * (size_t)cout, cudaMemcpyHostToDevice, ctx->stream));
    if (conv_tc_supported(L)) prepare_tc_weights(ctx, L);
    SFB_CUDA(cudaStreamSynchronize(ctx->stream));
}

// ------------------------------------------------------------ SIMT gather-GEMM
// CTA = 32 output rows x all output channels. Per tap: gather the 32
// neighbour rows (zeros where empty) and W[tap] into shared memory, then
// every thread accumulates its outputs over the tap's input channels.
constexpr int kRows = 32;
constexpr int kThreads = 256;
constexpr int kMaxOut = 16;  // kRows * cout / kThreads for cout <= 128
// transposed convs are tap-bucketed (one weight tap per 128-row tile) from 16
// tiles up (A/B on config 2, 8 frames in flight: 0.316 vs 0.336 ms/frame for a
// 64-tile threshold, same latency); tinier levels split the taps over a cluster
constexpr int64_t kTconvBucketRows = 16 * 128;

__global__ void __launch_bounds__(kThreads)
k_conv_simt(const float *__restrict__ in, int ld_in, const int32_t *__restrict__ nbr, int64_t nbr_ld,
            const int64_t *__restrict__ d_m, int64_t m_fixed, int taps, int cin, int cout,
            const float *__restrict__ w, const float *__restrict__ b, int relu,
            float *__restrict__ out, int ld_out) {
    extern __shared__ float sm[];
    float *A = sm;                  // [kRows][cin]
    float *W = sm + kRows * cin;    // [cin][cout]
    const int64_t m = d_m ? *d_m : m_fixed;
    const int nout = kRows * cout;
    for (int64_t r0 = (int64_t)blockIdx.x * kRows; r0 < m; r0 += (int64_t)gridDim.x * kRows) {
        float acc[kMaxOut];
#pragma unroll
        for (int k = 0; k < kMaxOut; ++k) acc[k] = 0.f;
        for (int t = 0; t < taps; ++t) {
            int any = 0;
            for (int i = threadIdx.x; i < kRows * cin; i += kThreads) {
                int r = i / cin, ci = i % cin;
                int64_t row = r0 + r;
                int32_t src = row < m ? nbr[(int64_t)t * nbr_ld + row] : -1;
                any |= src >= 0;
                A[i] = src >= 0 ? in[(int64_t)src * ld_in + ci] : 0.f;
            }
            if (!__syncthreads_or(any)) continue;
            const float *wt = w + (size_t)t * cin * cout;
            for (int i = threadIdx.x; i < cin * cout; i += kThreads) W[i] = wt[i];
            __syncthreads();
#pragma unroll
            for (int k = 0; k < kMaxOut; ++k) {
                int o = threadIdx.x + k * kThreads;
                if (o < nout) {
                    int r = o / cout, co = o % cout;
                    float sacc = acc[k];
                    for (int ci = 0; ci < cin; ++ci) sacc = fmaf(A[r * cin + ci], W[ci * cout + co], sacc);
                    acc[k] = sacc;
                }
            }
            __syncthreads();
        }
#pragma unroll
        for (int k = 0; k < kMaxOut; ++k) {
            int o = threadIdx.x + k * kThreads;
            if (o < nout) {
                int r = o / cout, co = o % cout;
                int64_t row = r0 + r;
                if (row < m) {
                    float v = acc[k] + b[co];
                    out[row * ld_out + co] = relu ? fmaxf(v, 0.f) : v;
                }
            }
        }
        __syncthreads();
    }
}

// Narrow first layer (Cin = 9, Cout = 16 at level 0): PARTS threads per output
// row (2: 8 accumulators each, twice the warps on the ~31 k rows — 0.746 vs
// 0.750 ms latency, same throughput), the whole weight tensor in
// shared memory (read as 16-byte broadcasts), the row's kernel-map entries
// loaded up front and the next tap's input row in flight while the current
// one is multiplied. Its K = 9 per tap would use a quarter of a 16-wide
// tensor-core step and its 27-tap chain of MMA round trips is longer than
// the FFMA work itself. Sums in tap order, then input channel (fp32 FFMA).
// A/B on config 2 with 8 frames in flight: 0.297 vs 0.308 ms/frame for the
// tcgen05 path on this layer, same latency.
template <int CIN, int COUT, int TAPS, int PARTS>
__global__ void __launch_bounds__(128)
k_conv_narrow(const float *__restrict__ in, int ld_in, const int32_t *__restrict__ nbr, int64_t nbr_ld,
              const int64_t *__restrict__ d_m, int64_t m_fixed, const float *__restrict__ w,
              const float *__restrict__ b, int relu, float *__restrict__ out, int ld_out) {
    // PARTS threads per row, each with COUT / PARTS of the outputs
    constexpr int CO = COUT / PARTS;
    static_assert(CO % 4 == 0, "outputs per thread must be a multiple of 4");
    extern __shared__ __align__(16) float sW[];   // [TAPS][CIN][COUT]
    static_assert((TAPS * CIN * COUT) % 4 == 0, "16-byte weight staging");
    // weights staged with 16-byte loads, 8 in flight per thread (a rolled
    // scalar loop waits ~30 round trips before the first FMA)
#pragma unroll 8
    for (int i = threadIdx.x; i < TAPS * CIN * COUT / 4; i += blockDim.x)
        reinterpret_cast<float4 *>(sW)[i] = __ldg(reinterpret_cast<const float4 *>(w) + i);
    __syncthreads();
    const int64_t m = d_m ? *d_m : m_fixed;
    SFB_FOR(item, m * PARTS) {
        const int64_t row = item / PARTS;
        const int c0 = (int)(item % PARTS) * CO;
        int32_t src[TAPS];
#pragma unroll
        for (int t = 0; t < TAPS; ++t) src[t] = nbr[(int64_t)t * nbr_ld + row];
        float acc[CO];
#pragma unroll
        for (int c = 0; c < CO; ++c) acc[c] = 0.f;
        float x[CIN];
#pragma unroll
        for (int c = 0; c < CIN; ++c) x[c] = src[0] >= 0 ? __ldg(in + (int64_t)src[0] * ld_in + c) : 0.f;
#pragma unroll
        for (int t = 0; t < TAPS; ++t) {
            float xn[CIN];
            if (t + 1 < TAPS) {
#pragma unroll
                for (int c = 0; c < CIN; ++c)
                    xn[c] = src[t + 1] >= 0 ? __ldg(in + (int64_t)src[t + 1] * ld_in + c) : 0.f;
            }
            if (src[t] >= 0) {
#pragma unroll
                for (int ci = 0; ci < CIN; ++ci) {
                    const float4 *wr = reinterpret_cast<const float4 *>(sW + (t * CIN + ci) * COUT + c0);
#pragma unroll
                    for (int q = 0; q < CO / 4; ++q) {
                        const float4 wv = wr[q];
                        acc[4 * q] = fmaf(x[ci], wv.x, acc[4 * q]);
                        acc[4 * q + 1] = fmaf(x[ci], wv.y, acc[4 * q + 1]);
                        acc[4 * q + 2] = fmaf(x[ci], wv.z, acc[4 * q + 2]);
                        acc[4 * q + 3] = fmaf(x[ci], wv.w, acc[4 * q + 3]);
                    }
                }
            }
            if (t + 1 < TAPS) {
#pragma unroll
                for (int c = 0; c < CIN; ++c) x[c] = xn[c];
            }
        }
        float *o = out + row * (int64_t)ld_out + c0;
#pragma unroll
        for (int c = 0; c < CO; ++c) {
            const float v = acc[c] + b[c0 + c];
            o[c] = relu ? fmaxf(v, 0.f) : v;
        }
    }
}

template <int CIN, int COUT, int TAPS, int PARTS>
static void launch_narrow(sfb_ctx *ctx, const NetLayer &L, const float *in, int ld_in, const int32_t *nbr,
                          int64_t nbr_ld, const int64_t *d_m, int64_t m_bound, int relu, float *out,
                          int ld_out, int64_t m_grid) {
    constexpr size_t smem = sizeof(float) * TAPS * CIN * COUT;
    set_max_dyn_smem(reinterpret_cast<const void *>(k_conv_narrow<CIN, COUT, TAPS, PARTS>), (int)smem);
    k_conv_narrow<CIN, COUT, TAPS, PARTS><<<dgrid(m_grid * PARTS, 128, 8), 128, smem, ctx->stream>>>(
        in, ld_in, nbr, nbr_ld, d_m, m_bound, L.w, L.b, relu, out, ld_out);
    SFB_CHECK_LAUNCH();
}

void conv_layer(sfb_ctx *ctx, const NetLayer &L, const float *in, int ld_in, const int32_t *nbr,
                int64_t nbr_ld, const int64_t *d_m, int64_t m_bound, int relu, float *out,
                int ld_out, int64_t m_grid, int csplit) {
    if (m_bound == 0) return;
    if (m_grid < 0) m_grid = m_bound;
    if (ctx->net_mode != SFB_NET_TC_BF16 && L.cin == 9 && L.cout == 16 && L.taps == 27) {
        launch_narrow<9, 16, 27, 2>(ctx, L, in, ld_in, nbr, nbr_ld, d_m, m_bound, relu, out, ld_out, m_grid);
        return;
    }
    if (ctx->net_mode != SFB_NET_SIMT_F32 && L.w_tc) {
        conv_layer_tc(ctx, L, in, ld_in, nbr, nbr_ld, d_m, m_bound, relu, out, ld_out, m_grid,
                      nullptr, nullptr, csplit);
        return;
    }
    SFB_REQUIRE(kRows * L.cout <= kMaxOut * kThreads, "conv: cout > 128 unsupported");
    size_t smem = sizeof(float) * ((size_t)kRows * L.cin + (size_t)L.cin * L.cout);
    SFB_REQUIRE(smem <= 200 * 1024, "conv: channels too wide for one CTA");
    set_max_dyn_smem(reinterpret_cast<const void *>(k_conv_simt), 200 * 1024);
    k_conv_simt<<<dgrid(m_grid, kRows, 4), kThreads, smem, ctx->stream>>>(
        in, ld_in, nbr, nbr_ld, d_m, m_bound, L.taps, L.cin, L.cout, L.w, L.b, relu, out, ld_out);
    SFB_CHECK_LAUNCH();
}

// transposed conv: out[r] = b + in[parent[r]] @ W[tap[r]]  (orphans: bias only)
__global__ void k_tconv(const float *__restrict__ in, int ld_in, const int32_t *__restrict__ parent,
                        const int32_t *__restrict__ tap, const int64_t *__restrict__ d_m,
                        int64_t m_fixed, int cin, int cout, const float *__restrict__ w,
                        const float *__restrict__ b, int relu, float *__restrict__ out, int ld_out) {
    const int64_t m = d_m ? *d_m : m_fixed;
    SFB_FOR(idx, m * cout) {
        const int64_t r = idx / cout;
        const int co = (int)(idx % cout);
        const int32_t p = parent[r];
        float s = 0.f;
        if (p >= 0) {
            const float *x = in + (int64_t)p * ld_in;
            const float *wt = w + (size_t)tap[r] * cin * cout + co;
            for (int ci = 0; ci < cin; ++ci) s = fmaf(x[ci], wt[(size_t)ci * cout], s);
        }
        const float v = s + b[co];
        out[r * ld_out + co] = relu ? fmaxf(v, 0.f) : v;
    }
}

// 8-tap "kernel map" of a transposed conv: row r gathers its parent under
// tap[r] only, so sum_t in[map[t][r]] @ W[t] = in[parent[r]] @ W[tap[r]]
// (orphans: no tap, bias only) — the tcgen05 gather-GEMM then runs it as-is
__global__ void k_tmap(const int32_t *__restrict__ parent, const int32_t *__restrict__ tap,
                       const int64_t *__restrict__ d_m, int64_t m_fixed, int64_t ld,
                       int32_t *__restrict__ tmap) {
    const int64_t m = d_m ? *d_m : m_fixed;
    SFB_FOR(r, m) {
        const int32_t p = parent[r], t = tap[r];
#pragma unroll
        for (int k = 0; k < 8; ++k) tmap[k * ld + r] = (k == t) ? p : -1;
    }
}

void tconv_layer(sfb_ctx *ctx, const NetLayer &L, const float *in, int ld_in,
                 const int32_t *parent, const int32_t *tap, const int64_t *d_m, int64_t m_bound,
                 int relu, float *out, int ld_out, int64_t m_grid, const int32_t *tmap,
                 const TapBuckets *tb, int csplit) {
    if (m_bound == 0) return;
    if (m_grid < 0) m_grid = m_bound;
    if (ctx->net_mode != SFB_NET_SIMT_F32 && L.w_tc) {
        // the 8-tap map's scratch is taken on both paths so the arena layout
        // does not depend on which one the size hints select
        int32_t *tbuf = tmap ? nullptr : ctx->arena.alloc<int32_t>(8 * (size_t)m_bound);
        // rows bucketed by tap (one tap per 128-row tile) from 16 tiles up;
        // only tiny levels split the 8 taps over a cluster instead (A/B on
        // config 2 with 8 frames in flight: 0.316 vs 0.336 ms/frame for a
        // 64-tile threshold, same latency)
        if (tb && m_grid >= kTconvBucketRows) {
            conv_layer_tc(ctx, L, in, ld_in, tb->src, 0, tb->d_rows, tb->rows_bound, relu, out,
                          ld_out, tb->rows_grid, tb->perm, tb->off);
            return;
        }
        if (!tmap) {
            k_tmap<<<dgrid(m_grid, 256), 256, 0, ctx->stream>>>(parent, tap, d_m, m_bound, m_bound, tbuf);
            SFB_CHECK_LAUNCH();
            tmap = tbuf;
        }
        conv_layer_tc(ctx, L, in, ld_in, tmap, m_bound, d_m, m_bound, relu, out, ld_out, m_grid,
                      nullptr, nullptr, csplit);
        return;
    }
    k_tconv<<<dgrid(m_grid * L.cout, 256), 256, 0, ctx->stream>>>(
        in, ld_in, parent, tap, d_m, m_bound, L.cin, L.cout, L.w, L.b, relu, out, ld_out);
    SFB_CHECK_LAUNCH();
}

// child tap from coordinates (child stride cs, parent stride 2cs)
__global__ void k_child_tap(const int32_t *__restrict__ coords, const int64_t *__restrict__ d_m,
                            int cs, int32_t *__restrict__ tap) {
    const int64_t m = *d_m;
    const int64_t ps = 2 * (int64_t)cs;
    SFB_FOR(r, m) {
        int64_t d[3];
        for (int a = 0; a < 3; ++a) {
            int64_t c = coords[3 * r + a];
            d[a] = floor_div(c - floor_div(c, ps) * ps, cs);
        }
        tap[r] = (int32_t)(d[2] * 4 + d[1] * 2 + d[0]);
    }
}

// ------------------------------------------------------------ MLP head
constexpr int kHeadRows = 32;

__global__ void k_head_mlp(const float *__restrict__ f, int ld, const int64_t *__restrict__ d_m,
                           int cin, int hid, const float *__restrict__ w1,
                           const float *__restrict__ b1, const float *__restrict__ w2,
                           const float *__restrict__ b2, float *__restrict__ raw) {
    extern __shared__ float sm[];
    float *F = sm;                         // [rows][cin]
    float *H = F + kHeadRows * cin;        // [rows][hid]
    float *W1 = H + kHeadRows * hid;       // [cin][hid]
    float *W2 = W1 + cin * hid;            // [hid][14]
    const int64_t m = *d_m;
    for (int i = threadIdx.x; i < cin * hid; i += blockDim.x) W1[i] = w1[i];
    for (int i = threadIdx.x; i < hid * 14; i += blockDim.x) W2[i] = w2[i];
    for (int64_t r0 = (int64_t)blockIdx.x * kHeadRows; r0 < m; r0 += (int64_t)gridDim.x * kHeadRows) {
    __syncthreads();
    for (int i = threadIdx.x; i < kHeadRows * cin; i += blockDim.x) {
        int64_t row = r0 + i / cin;
        F[i] = row < m ? f[row * ld + i % cin] : 0.f;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < kHeadRows * hid; i += blockDim.x) {
        int r = i / hid, j = i % hid;
        float s = 0.f;
        for (int c = 0; c < cin; ++c) s = fmaf(F[r * cin + c], W1[c * hid + j], s);
        H[i] = fmaxf(s + b1[j], 0.f);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < kHeadRows * 14; i += blockDim.x) {
        int r = i / 14, k = i % 14;
        int64_t row = r0 + r;
        if (row >= m) continue;
        float s = 0.f;
        for (int c = 0; c < hid; ++c) s = fmaf(H[r * hid + c], W2[c * 14 + k], s);
        raw[row * 14 + k] = s + b2[k];
    }
    }
}

// thread-per-row head for the default widths: the row's features live in
// registers, weights are broadcast from shared memory (every lane reads the
// same W element in the same step), hidden units are consumed as produced
template <int CIN, int HID>
__global__ void __launch_bounds__(128)
k_head_row(const float *__restrict__ f, int ld, const int64_t *__restrict__ d_m,
           const float *__restrict__ w1, const float *__restrict__ b1, const float *__restrict__ w2,
           const float *__restrict__ b2, float *__restrict__ raw) {
    __shared__ __align__(16) float W1[CIN * HID], B1[HID], W2[HID * 14], B2[14];
    // 16-byte weight staging, all loads in flight (see k_conv_narrow)
    static_assert((CIN * HID) % 4 == 0 && (HID * 14) % 4 == 0, "16-byte weight staging");
#pragma unroll
    for (int i = threadIdx.x; i < CIN * HID / 4; i += 128)
        reinterpret_cast<float4 *>(W1)[i] = __ldg(reinterpret_cast<const float4 *>(w1) + i);
#pragma unroll
    for (int i = threadIdx.x; i < HID * 14 / 4; i += 128)
        reinterpret_cast<float4 *>(W2)[i] = __ldg(reinterpret_cast<const float4 *>(w2) + i);
    for (int i = threadIdx.x; i < HID; i += blockDim.x) B1[i] = b1[i];
    if (threadIdx.x < 14) B2[threadIdx.x] = b2[threadIdx.x];
    __syncthreads();
    const int64_t m = *d_m;
    SFB_FOR(row, m) {
        float x[CIN];
#pragma unroll
        for (int c = 0; c < CIN; c += 4) {
            const float4 v = *reinterpret_cast<const float4 *>(f + row * ld + c);
            x[c] = v.x;
            x[c + 1] = v.y;
            x[c + 2] = v.z;
            x[c + 3] = v.w;
        }
        float o[14];
#pragma unroll
        for (int k = 0; k < 14; ++k) o[k] = 0.f;
#pragma unroll 4
        for (int j = 0; j < HID; ++j) {
            float h = 0.f;
#pragma unroll
            for (int c = 0; c < CIN; ++c) h = fmaf(x[c], W1[c * HID + j], h);
            h = fmaxf(h + B1[j], 0.f);
#pragma unroll
            for (int k = 0; k < 14; ++k) o[k] = fmaf(h, W2[j * 14 + k], o[k]);
        }
#pragma unroll
        for (int k = 0; k < 14; ++k) raw[row * 14 + k] = o[k] + B2[k];
    }
}

// ------------------------------------------------------------ activations
__device__ __forceinline__ double logaddexp0(double x) {
    // numpy npy_logaddexp(0, x): larger + log1p(exp(-|difference|))
    double tmp = 0.0 - x;
    if (tmp > 0) return 0.0 + log1p(exp(-tmp));
    if (tmp <= 0) return x + log1p(exp(tmp));
    return tmp;  // NaN
}

template <class R>
__device__ __forceinline__ void activate_row(const R *r, double scale, double *delta,
                                             double *sigma, double *q, double *opac,
                                             double *normal) {
    double x[14];
#pragma unroll
    for (int k = 0; k < 14; ++k) x[k] = (double)r[k];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        delta[a] = tanh(x[a]) * scale;
        sigma[a] = fmax(logaddexp0(x[3 + a]), 1e-12) * scale;
    }
    double qq[4] = {x[6] + 1.0, x[7], x[8], x[9]};
    double qn = sqrt(qq[0] * qq[0] + qq[1] * qq[1] + qq[2] * qq[2] + qq[3] * qq[3]);
    if (qn < 1e-12) {
        q[0] = 1.0;
        q[1] = q[2] = q[3] = 0.0;
    } else {
        double d = fmax(qn, 1e-300);
        for (int a = 0; a < 4; ++a) q[a] = qq[a] / d;
    }
    double o = x[10];
    if (o >= 0) *opac = 1.0 / (1.0 + exp(-o));
    else {
        double e = exp(o);
        *opac = e / (1.0 + e);
    }
    double nn = sqrt(x[11] * x[11] + x[12] * x[12] + x[13] * x[13]);
    if (nn < 1e-8) {
        normal[0] = normal[1] = 0.0;
        normal[2] = 1.0;
    } else {
        double d = fmax(nn, 1e-300);
        for (int a = 0; a < 3; ++a) normal[a] = x[11 + a] / d;
    }
}

__global__ void k_activate(const double *__restrict__ raw, int64_t m, double scale, double *delta,
                           double *sigma, double *quat, double *opac, double *normal) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= m) return;
    activate_row(raw + 14 * i, scale, delta + 3 * i, sigma + 3 * i, quat + 4 * i, opac + i,
                 normal + 3 * i);
}

void activate_run(sfb_ctx *ctx, const double *raw, int64_t m, double scale, double *delta,
                  double *sigma, double *quat, double *opac, double *normal) {
    SFB_REQUIRE(scale > 0, "voxel_scale must be positive");
    if (m == 0) return;
    k_activate<<<grid_for(m, 128), 128, 0, ctx->stream>>>(raw, m, scale, delta, sigma, quat, opac,
                                                          normal);
    SFB_CHECK_LAUNCH();
}

// Per-voxel Gaussian: centre = (coord + 0.5 + residual) * scale + delta
// (voxelgrid.py:119-122 + estimators.py:223), then the activated fields.
template <class R>
__global__ void k_voxel_splats(const R *__restrict__ raw, const int32_t *__restrict__ coords,
                               const double *__restrict__ feats9, const int64_t *__restrict__ d_m,
                               const FrameParams *__restrict__ P, double *centers, double *sigma,
                               double *quat, double *opac, double *normal) {
    const int64_t m = *d_m;
    const double scale = P->inv_s;
    SFB_FOR(v, m) {
    double delta[3];
    activate_row(raw + 14 * v, scale, delta, sigma + 3 * v, quat + 4 * v, opac + v, normal + 3 * v);
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        double rec = __dmul_rn(__dadd_rn(__dadd_rn((double)coords[3 * v + a], 0.5), feats9[9 * v + 6 + a]),
                               scale);
        centers[3 * v + a] = __dadd_rn(rec, delta[a]);
    }
    }
}

void head_to_voxel_splats(sfb_ctx *ctx, const void *raw, const int32_t *coords,
                          const double *feats9, const int64_t *d_m, int64_t m_bound,
                          const FrameParams *P, double *centers, double *sigma, double *quat,
                          double *opac, double *normal) {
    if (ctx->net_mode == SFB_NET_SIMT_F64)
        k_voxel_splats<double><<<dgrid(m_bound, 128), 128, 0, ctx->stream>>>(
            static_cast<const double *>(raw), coords, feats9, d_m, P, centers, sigma, quat, opac, normal);
    else
        k_voxel_splats<float><<<dgrid(m_bound, 128), 128, 0, ctx->stream>>>(
            static_cast<const float *>(raw), coords, feats9, d_m, P, centers, sigma, quat, opac, normal);
    SFB_CHECK_LAUNCH();
}

// ------------------------------------------------------------ float64 network
// SFB_NET_SIMT_F64: the reference network's own arithmetic — float64
// features, float32 weights upcast (sparsenet.py:207-210, 245, 285-286) — on
// the FP64 pipe. The parity mode of the end-to-end image check: the Gaussian
// parameters then agree with the reference to ~1e-13 instead of the ~1e-6 of
// the fp32-accurate tensor-core path, so no (splat, pixel) alpha or
// transmittance lands on the other side of a 1/255 cutoff. Same structure
// (kernel maps, pooling, buckets) as the fp32 path; only the feature kernels
// differ.
constexpr int kRowsD = 32;

// CTA = 32 output rows x all output channels; per tap the 32 gathered input
// rows (float64) and the tap's weights (float32) sit in shared memory, every
// thread accumulates its outputs over the tap's input channels
__global__ void __launch_bounds__(kThreads)
k_conv_f64(const double *__restrict__ in, int ld_in, const int32_t *__restrict__ nbr, int64_t nbr_ld,
           const int64_t *__restrict__ d_m, int taps, int cin, int cout, const float *__restrict__ w,
           const float *__restrict__ b, int relu, double *__restrict__ out, int ld_out) {
    extern __shared__ __align__(16) unsigned char sm_raw[];
    double *A = reinterpret_cast<double *>(sm_raw);            // [kRowsD][cin]
    float *W = reinterpret_cast<float *>(A + kRowsD * cin);    // [cin][cout]
    const int64_t m = *d_m;
    const int nout = kRowsD * cout;
    for (int64_t r0 = (int64_t)blockIdx.x * kRowsD; r0 < m; r0 += (int64_t)gridDim.x * kRowsD) {
        double acc[kMaxOut];
#pragma unroll
        for (int k = 0; k < kMaxOut; ++k) acc[k] = 0.0;
        for (int t = 0; t < taps; ++t) {
            int any = 0;
            for (int i = threadIdx.x; i < kRowsD * cin; i += kThreads) {
                const int r = i / cin, ci = i % cin;
                const int64_t row = r0 + r;
                const int32_t src = row < m ? nbr[(int64_t)t * nbr_ld + row] : -1;
                any |= src >= 0;
                A[i] = src >= 0 ? in[(int64_t)src * ld_in + ci] : 0.0;
            }
            if (!__syncthreads_or(any)) continue;
            const float *wt = w + (size_t)t * cin * cout;
            for (int i = threadIdx.x; i < cin * cout; i += kThreads) W[i] = wt[i];
            __syncthreads();
#pragma unroll
            for (int k = 0; k < kMaxOut; ++k) {
                const int o = threadIdx.x + k * kThreads;
                if (o < nout) {
                    const int r = o / cout, co = o % cout;
                    double sacc = 0.0;
                    for (int ci = 0; ci < cin; ++ci) sacc = fma(A[r * cin + ci], (double)W[ci * cout + co], sacc);
                    acc[k] += sacc;   // x_t @ W_t, then accumulated in tap order
                }
            }
            __syncthreads();
        }
#pragma unroll
        for (int k = 0; k < kMaxOut; ++k) {
            const int o = threadIdx.x + k * kThreads;
            if (o < nout) {
                const int r = o / cout, co = o % cout;
                const int64_t row = r0 + r;
                if (row < m) {
                    const double v = (double)b[co] + acc[k];
                    out[row * ld_out + co] = relu ? fmax(v, 0.0) : v;
                }
            }
        }
        __syncthreads();
    }
}

// transposed conv: out[r] = b + in[parent[r]] @ W[tap[r]] (orphans: bias only)
__global__ void k_tconv_f64(const double *__restrict__ in, int ld_in, const int32_t *__restrict__ parent,
                            const int32_t *__restrict__ tap, const int64_t *__restrict__ d_m, int cin,
                            int cout, const float *__restrict__ w, const float *__restrict__ b, int relu,
                            double *__restrict__ out, int ld_out) {
    const int64_t m = *d_m;
    SFB_FOR(idx, m * cout) {
        const int64_t r = idx / cout;
        const int co = (int)(idx % cout);
        const int32_t p = parent[r];
        double s = 0.0;
        if (p >= 0) {
            const double *x = in + (int64_t)p * ld_in;
            const float *wt = w + (size_t)tap[r] * cin * cout + co;
            for (int ci = 0; ci < cin; ++ci) s = fma(x[ci], (double)wt[(size_t)ci * cout], s);
        }
        const double v = (double)b[co] + s;
        out[r * ld_out + co] = relu ? fmax(v, 0.0) : v;
    }
}

// pool_2x2x2 means: children summed in child-row order (np.add.at)
__global__ void k_pool_means_f64(const double *__restrict__ feats, int ld_in, int c,
                                 const int32_t *__restrict__ nkids, const int32_t *__restrict__ kids,
                                 const int64_t *__restrict__ d_mp, double *__restrict__ out, int ld_out) {
    const int64_t mp = *d_mp;
    SFB_FOR(idx, mp * c) {
        const int64_t v = idx / c;
        const int ch = (int)(idx % c);
        const int cnt = min(nkids[v], 8);
        int32_t kk[8];
        for (int q = 0; q < cnt; ++q) kk[q] = kids[8 * v + q];
        for (int q = 1; q < cnt; ++q) {   // ascending child rows
            const int32_t x = kk[q];
            int r = q - 1;
            while (r >= 0 && kk[r] > x) {
                kk[r + 1] = kk[r];
                --r;
            }
            kk[r + 1] = x;
        }
        double acc = 0.0;
        for (int q = 0; q < cnt; ++q) acc += feats[(int64_t)kk[q] * ld_in + ch];
        out[v * ld_out + ch] = acc / (double)cnt;
    }
}

// head MLP relu(f @ W1 + b1) @ W2 + b2 (sparsenet.py:284-286), 32 rows per CTA
__global__ void k_head_f64(const double *__restrict__ f, int ld, const int64_t *__restrict__ d_m,
                           int cin, int hid, const float *__restrict__ w1, const float *__restrict__ b1,
                           const float *__restrict__ w2, const float *__restrict__ b2,
                           double *__restrict__ raw) {
    extern __shared__ __align__(16) unsigned char sm_raw[];
    double *F = reinterpret_cast<double *>(sm_raw);   // [rows][cin]
    double *H = F + kHeadRows * cin;                   // [rows][hid]
    const int64_t m = *d_m;
    for (int64_t r0 = (int64_t)blockIdx.x * kHeadRows; r0 < m; r0 += (int64_t)gridDim.x * kHeadRows) {
        __syncthreads();
        for (int i = threadIdx.x; i < kHeadRows * cin; i += blockDim.x) {
            const int64_t row = r0 + i / cin;
            F[i] = row < m ? f[row * ld + i % cin] : 0.0;
        }
        __syncthreads();
        for (int i = threadIdx.x; i < kHeadRows * hid; i += blockDim.x) {
            const int r = i / hid, j = i % hid;
            double sacc = 0.0;
            for (int c = 0; c < cin; ++c) sacc = fma(F[r * cin + c], (double)w1[c * hid + j], sacc);
            H[i] = fmax(sacc + (double)b1[j], 0.0);
        }
        __syncthreads();
        for (int i = threadIdx.x; i < kHeadRows * 14; i += blockDim.x) {
            const int r = i / 14, k = i % 14;
            const int64_t row = r0 + r;
            if (row >= m) continue;
            double sacc = 0.0;
            for (int c = 0; c < hid; ++c) sacc = fma(H[r * hid + c], (double)w2[c * 14 + k], sacc);
            raw[row * 14 + k] = sacc + (double)b2[k];
        }
    }
}

static void conv_f64(sfb_ctx *ctx, const NetLayer &L, const double *in, int ld_in,
                     const int32_t *nbr, int64_t nbr_ld, const int64_t *d_m, int64_t m_grid,
                     double *out, int ld_out) {
    SFB_REQUIRE(kRowsD * L.cout <= kMaxOut * kThreads, "conv: cout > 128 unsupported");
    const size_t smem = sizeof(double) * kRowsD * L.cin + sizeof(float) * L.cin * L.cout;
    SFB_REQUIRE(smem <= 200 * 1024, "conv: channels too wide for one CTA");
    set_max_dyn_smem(reinterpret_cast<const void *>(k_conv_f64), 200 * 1024);
    k_conv_f64<<<dgrid(m_grid, kRowsD, 4), kThreads, smem, ctx->stream>>>(
        in, ld_in, nbr, nbr_ld, d_m, L.taps, L.cin, L.cout, L.w, L.b, 1, out, ld_out);
    SFB_CHECK_LAUNCH();
}

// ------------------------------------------------------------ UNet
__global__ void k_feats_to_f32(const double *__restrict__ f, const int64_t *__restrict__ d_m, int c,
                               float *__restrict__ o) {
    const int64_t n = *d_m * c;
    SFB_FOR(i, n) o[i] = (float)f[i];
}

// Whole UNet + head with every level size kept on the device: buffers are
// sized by the host bound (the point count bounds every level), kernels loop
// over the device counts, so the sequence has no host synchronisation.
// split-K of the encoder / bottleneck convs by level (fixed per level, never
// from size hints, so results are independent of launch-time bounds): the
// splits of a tile form a thread-block cluster (DSMEM reduction); 1 = no
// split, -1 = split on the device from the actual row count. Level 0 has
// ~M0/128 tiles, every level ~4x fewer. Chosen by A/B on config 2 with 8
// frames in flight: {1, 1, 4, 8} gives 0.337 ms/frame vs 0.364 for {2, 4, 8,
// device} at the same single-frame latency — with concurrent frames the extra
// CTAs and the partial-sum reduction cost more than the parallelism they buy.
constexpr int kLevelSplit[4] = {1, 1, 4, 8};

void unet_level_bounds(const FrameParams &host, int64_t n, int levels, int64_t *bound) {
    auto round3 = [](int64_t x) {   // up to 3 significant bits
        int64_t step = 1;
        while ((x >> 3) >= step * 2) step <<= 1;
        return (x + step - 1) / step * step;
    };
    int64_t prev = n;
    for (int l = 0; l <= levels; ++l) {
        const int64_t S = int64_t(1) << l;
        double cells = 1.0;
        for (int a = 0; a < 3; ++a)
            cells *= (double)(floor_div(host.hi[a], S) - floor_div(host.lo[a], S) + 1);
        int64_t b = cells < (double)prev ? round3((int64_t)cells) : prev;
        b = std::min(std::max<int64_t>(b, 1), prev);
        bound[l] = prev = b;
    }
}
constexpr int kTconvSplit = 8;

void unet_run(sfb_ctx *ctx, const int32_t *coords0, const double *feats9, int64_t mb,
              const FrameParams &host, const FrameParams *P, DevCounts *C, void *raw_out,
              const float *feats32) {
    Net &net = ctx->net;
    SFB_REQUIRE(net.loaded, "network weights are not loaded");
    const int L = net.levels;
    SFB_REQUIRE(L + 1 <= 9, "at most 8 UNet levels");
    SFB_REQUIRE(L < sfb_ctx::kEvFeatsFork, "too many UNet levels for the side branch");
    const auto &enc = net.enc;
    const auto &dec = net.dec;
    cudaStream_t st = ctx->stream;
    std::vector<const int32_t *> coords(L + 1);
    std::vector<int32_t *> nbr(L + 1);
    std::vector<PoolStructure> ps(L);
    std::vector<float *> cat(L), pin(L + 1);
    std::vector<int> width(L);
    coords[0] = coords0;
    for (int l = 0; l < L; ++l) width[l] = dec[L - 1 - l] + enc[l + 1];
    // per-level row bounds (buffers, kernel-map leading dimensions, grids)
    std::vector<int64_t> mbl(L + 1), mg(L + 1);
    unet_level_bounds(host, mb, L, mbl.data());
    for (int l = 0; l <= L; ++l) mg[l] = ctx->grid_bound(mbl[l], ctx->hint_m[l]);
    std::vector<int> kern(L + 1);
    {
        int layer = 0;
        for (int l = 0; l <= L; ++l) kern[l] = net.layers[layer++].kernel;
    }
    // side branch fork point: the coordinate structure of the coarser levels
    // needs only the level-0 coordinates, so it starts with the level-0 hash
    SFB_CUDA(cudaEventRecord(ctx->side_ev[L], st));
    // level 0: hash + kernel map on the critical path
    HashTable h0;
    nbr[0] = ctx->arena.alloc<int32_t>((size_t)kern[0] * kern[0] * kern[0] * mbl[0]);
    h0 = hash_build(ctx, coords[0], &C->m[0], mbl[0], mg[0]);
    kernel_map_build(ctx, h0, coords[0], &C->m[0], mbl[0], 1, kern[0], nbr[0], mg[0]);
    if (ctx->feats_pending) {   // join the voxel-feature sums (voxelize_run on the aux stream)
        SFB_CUDA(cudaStreamWaitEvent(st, ctx->side_ev[sfb_ctx::kEvFeatsJoin], 0));
        ctx->feats_pending = false;
    }
    // side branch: the coordinate structure of every coarser level (parents,
    // children, taps, hash = the pooling table, kernel map) depends only on
    // coordinates, so it runs concurrently with the level-0 kernel map and
    // the convolutions; event l marks "level l+1 structure and kernel map ready"
    SFB_CUDA(cudaStreamWaitEvent(ctx->side_stream, ctx->side_ev[L], 0));
    ctx->stream = ctx->side_stream;
    try {
        for (int l = 0; l < L; ++l) {
            int32_t *pc = ctx->arena.alloc<int32_t>((size_t)mbl[l + 1] * 3);
            const int k = kern[l + 1];
            nbr[l + 1] = ctx->arena.alloc<int32_t>((size_t)k * k * k * mbl[l + 1]);
            ps[l] = pool_structure(ctx, coords[l], &C->m[l], mbl[l], mg[l], 1 << l, pc, &C->m[l + 1]);
            kernel_map_build(ctx, ps[l].table, pc, &C->m[l + 1], mbl[l + 1], 2 << l, k, nbr[l + 1],
                             mg[l + 1]);
            coords[l + 1] = pc;
            SFB_CUDA(cudaEventRecord(ctx->side_ev[l], ctx->stream));
        }
    } catch (...) {
        ctx->stream = st;
        throw;
    }
    ctx->stream = st;
    auto export_debug = [&]() {   // parity export (eager frames only)
        const FrameDebug &D = ctx->frame_debug;
        if (!(D.cap > 0 && D.level_coords && D.level_maps)) return;
        SFB_REQUIRE(mb <= D.cap, "frame debug buffers are smaller than the cloud");
        for (int l = 0; l <= L && l < D.levels; ++l) {
            const int taps = kern[l] * kern[l] * kern[l];
            SFB_REQUIRE(taps <= 27, "frame debug export holds up to 27 taps per level");
            SFB_CUDA(cudaMemcpyAsync(D.level_coords + (size_t)l * 3 * D.cap, coords[l],
                                     sizeof(int32_t) * 3 * mbl[l], cudaMemcpyDeviceToDevice, st));
            for (int t = 0; t < taps; ++t)
                SFB_CUDA(cudaMemcpyAsync(D.level_maps + ((size_t)l * 27 + t) * D.cap,
                                         nbr[l] + (size_t)t * mbl[l], sizeof(int32_t) * mbl[l],
                                         cudaMemcpyDeviceToDevice, st));
        }
    };
    if (ctx->net_mode == SFB_NET_SIMT_F64) {   // float64 features end to end
        double *raw = static_cast<double *>(raw_out);
        std::vector<double *> catd(L), pind(L + 1);
        int layer = 0;
        for (int l = 0; l < L; ++l) {
            catd[l] = ctx->arena.alloc<double>((size_t)mbl[l] * width[l]);
            const int up = dec[L - 1 - l];
            conv_f64(ctx, net.layers[layer++], l ? pind[l] : feats9, l ? enc[l] : 9, nbr[l], mbl[l],
                     &C->m[l], mg[l], catd[l] + up, width[l]);
            pind[l + 1] = ctx->arena.alloc<double>((size_t)mbl[l + 1] * enc[l + 1]);
            SFB_CUDA(cudaStreamWaitEvent(st, ctx->side_ev[l], 0));   // level l+1 structure ready
            k_pool_means_f64<<<dgrid(mg[l + 1] * enc[l + 1], 256), 256, 0, st>>>(
                catd[l] + up, width[l], enc[l + 1], ps[l].nkids, ps[l].kids, &C->m[l + 1], pind[l + 1],
                enc[l + 1]);
            SFB_CHECK_LAUNCH();
        }
        double *bott = ctx->arena.alloc<double>((size_t)mbl[L] * enc[L + 1]);
        conv_f64(ctx, net.layers[layer++], pind[L], enc[L], nbr[L], mbl[L], &C->m[L], mg[L], bott,
                 enc[L + 1]);
        const double *coarse = bott;
        int ld_coarse = enc[L + 1];
        for (int l = L - 1; l >= 0; --l) {
            const NetLayer &T = net.layers[layer++];
            k_tconv_f64<<<dgrid(mg[l] * T.cout, 256), 256, 0, st>>>(
                coarse, ld_coarse, ps[l].c2p, ps[l].tap, &C->m[l], T.cin, T.cout, T.w, T.b, 1, catd[l],
                width[l]);
            SFB_CHECK_LAUNCH();
            coarse = catd[l];
            ld_coarse = width[l];
        }
        export_debug();
        const NetLayer &h1 = net.layers[layer], &h2 = net.layers[layer + 1];
        const size_t smem = sizeof(double) * kHeadRows * (h1.cin + h1.cout);
        SFB_REQUIRE(smem <= 200 * 1024, "head MLP too wide");
        set_max_dyn_smem(reinterpret_cast<const void *>(k_head_f64), 200 * 1024);
        k_head_f64<<<dgrid(mg[0], kHeadRows, 4), 128, smem, st>>>(
            catd[0], width[0], &C->m[0], h1.cin, h1.cout, h1.w, h1.b, h2.w, h2.b, raw);
        SFB_CHECK_LAUNCH();
        return;
    }
    float *raw = static_cast<float *>(raw_out);
    if (feats32 && enc[0] == 9) {
        pin[0] = const_cast<float *>(feats32);
    } else {
        pin[0] = ctx->arena.alloc<float>((size_t)mbl[0] * enc[0]);
        k_feats_to_f32<<<dgrid(mg[0] * enc[0], 256), 256, 0, st>>>(feats9, &C->m[0], enc[0], pin[0]);
        SFB_CHECK_LAUNCH();
    }
    int layer = 0;
    for (int l = 0; l < L; ++l) {
        cat[l] = ctx->arena.alloc<float>((size_t)mbl[l] * width[l]);
        const int up = dec[L - 1 - l];
        conv_layer(ctx, net.layers[layer], pin[l], enc[l], nbr[l], mbl[l], &C->m[l], mbl[l], 1,
                   cat[l] + up, width[l], mg[l], kLevelSplit[std::min(l, 3)]);
        ++layer;
        pin[l + 1] = ctx->arena.alloc<float>((size_t)mbl[l + 1] * enc[l + 1]);
        SFB_CUDA(cudaStreamWaitEvent(st, ctx->side_ev[l], 0));   // level l+1 structure ready
        pool_means(ctx, ps[l], &C->m[l + 1], mg[l + 1], cat[l] + up, enc[l + 1], width[l],
                   pin[l + 1], enc[l + 1]);
    }
    float *bott = ctx->arena.alloc<float>((size_t)mbl[L] * enc[L + 1]);
    conv_layer(ctx, net.layers[layer], pin[L], enc[L], nbr[L], mbl[L], &C->m[L], mbl[L], 1, bott,
               enc[L + 1], mg[L], kLevelSplit[std::min(L, 3)]);
    ++layer;
    const float *coarse = bott;
    int ld_coarse = enc[L + 1];
    for (int l = L - 1; l >= 0; --l) {
        tconv_layer(ctx, net.layers[layer], coarse, ld_coarse, ps[l].c2p, ps[l].tap, &C->m[l],
                    mbl[l], 1, cat[l], width[l], mg[l], ps[l].tmap, &ps[l].buckets, kTconvSplit);
        ++layer;
        coarse = cat[l];
        ld_coarse = width[l];
    }
    export_debug();
    const NetLayer &h1 = net.layers[layer], &h2 = net.layers[layer + 1];
    size_t smem = sizeof(float) * ((size_t)kHeadRows * (h1.cin + h1.cout) + (size_t)h1.cin * h1.cout +
                                   (size_t)h1.cout * 14);
    set_max_dyn_smem(reinterpret_cast<const void *>(k_head_mlp), 200 * 1024);
    SFB_REQUIRE(smem <= 200 * 1024, "head MLP too wide");
    if (h1.cin == 32 && h1.cout == 64 && width[0] % 4 == 0) {
        k_head_row<32, 64><<<dgrid(mg[0], 128, 4), 128, 0, st>>>(cat[0], width[0], &C->m[0], h1.w,
                                                                 h1.b, h2.w, h2.b, raw);
        SFB_CHECK_LAUNCH();
        return;
    }
    k_head_mlp<<<dgrid(mg[0], kHeadRows, 4), 128, smem, st>>>(cat[0], width[0], &C->m[0], h1.cin,
                                                           h1.cout, h1.w, h1.b, h2.w, h2.b, raw);
    SFB_CHECK_LAUNCH();
}

}  // namespace sfb
