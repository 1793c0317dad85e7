// C ABI of libsfb200 (declared in include/sfb200.h): argument checks, error
// codes, arena reset per call, and the fused pipelines built from the stages
// in voxelize.cu / hashmap.cu / net.cu / conv_tc.cu / render.cu.
//
// Every stage keeps its data-dependent sizes in a DevCounts block on the
// device, so a call is a pure stream of kernels. sfb_frame replays the whole
// cloud -> P2ENet -> planes sequence as one CUDA graph: the first call with a
// new shape runs eagerly (growing the arena), the second captures, later
// calls update the parameter kernel node (lattice scale, key layout, camera,
// background) and launch the graph.
#include <algorithm>
#include <cmath>

#include "common.cuh"

using namespace sfb;

namespace sfb {
const void *write_params_func();
}

namespace {

void record_done(sfb_ctx *ctx) {
    if (cudaEventRecord(ctx->done_event, ctx->stream) == cudaSuccess) {
        ctx->done_stream = ctx->stream;
        ctx->done_valid = true;
    } else {
        cudaGetLastError();
    }
}

// Join whatever the side / aux streams still hold into ctx->stream (error
// paths: an abandoned capture must not end with unjoined streams, and the next
// call's arena reuse must be ordered after forked work). Errors are ignored.
void join_forked(sfb_ctx *ctx) {
    for (cudaStream_t s : {ctx->side_stream, ctx->aux_stream}) {
        if (s && cudaEventRecord(ctx->side_ev[sfb_ctx::kEvFeatsJoin], s) == cudaSuccess)
            cudaStreamWaitEvent(ctx->stream, ctx->side_ev[sfb_ctx::kEvFeatsJoin], 0);
    }
    cudaGetLastError();
}

template <class F>
int guard(sfb_ctx *ctx, F &&f) {
    if (!ctx) return SFB_ERR_ARG;
    try {
        SFB_CUDA(cudaSetDevice(ctx->device));
        // the arena is reset and reused below: order this call after the
        // previous call's kernels when they went to another stream
        if (ctx->done_valid && ctx->done_stream != ctx->stream)
            SFB_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->done_event, 0));
        ctx->arena.reset();
        ctx->feats_pending = false;
        ctx->n_marks = 0;
        ctx->mark(ST_BEGIN);
        try {
            f();
        } catch (...) {
            join_forked(ctx);   // whatever was enqueued before the error
            record_done(ctx);
            throw;
        }
        record_done(ctx);
        ctx->last_error.clear();
        return SFB_OK;
    } catch (const Error &e) {
        ctx->last_error = e.what();
        return e.code;
    } catch (const std::exception &e) {
        ctx->last_error = e.what();
        return SFB_ERR_STATE;
    }
}

DevCounts *new_counts(sfb_ctx *ctx) {
    DevCounts *C = ctx->arena.alloc<DevCounts>(1);
    SFB_CUDA(cudaMemsetAsync(C, 0, sizeof(DevCounts), ctx->stream));
    ctx->last_counts = C;
    return C;
}

FrameParams *params(sfb_ctx *ctx, const FrameParams &host) {
    FrameParams *P = ctx->arena.alloc<FrameParams>(1);
    write_params(ctx, host, P);
    return P;
}

FrameParams camera_params(const sfb_camera *cam, const double *bg) {
    FrameParams P{};
    if (cam) P.cam = to_cam(*cam);
    for (int a = 0; a < 3; ++a) P.bg[a] = bg ? bg[a] : 0.0;
    return P;
}

__global__ void k_expand_splats(const int32_t *__restrict__ p2v, int64_t n,
                                const double *__restrict__ vc, const double *__restrict__ vs,
                                const double *__restrict__ vq, const double *__restrict__ vo,
                                const double *__restrict__ vn, const double *__restrict__ col,
                                double *centers, double *scales, double *quats, double *opac,
                                double *colors, double *normals) {
    SFB_FOR(i, n) {
        const int64_t v = p2v[i];
        for (int a = 0; a < 3; ++a) {
            centers[3 * i + a] = vc[3 * v + a];
            scales[3 * i + a] = vs[3 * v + a];
            normals[3 * i + a] = vn[3 * v + a];
            if (colors) colors[3 * i + a] = col[3 * i + a];
        }
        for (int a = 0; a < 4; ++a) quats[4 * i + a] = vq[4 * v + a];
        opac[i] = vo[v];
    }
}

__global__ void k_tap_transpose(const int32_t *__restrict__ tm, int64_t m, int taps,
                                int32_t *__restrict__ out) {
    SFB_FOR(i, m * taps) {
        const int64_t r = i / taps;
        const int t = (int)(i % taps);
        out[i] = tm[(int64_t)t * m + r];
    }
}

struct VoxelSplats {
    VoxelOut vox;
    double *c, *s, *q, *o, *n;
};

// voxelize -> UNet -> head -> per-voxel Gaussians, all device-sized (bound n)
VoxelSplats neural_voxels(sfb_ctx *ctx, const double *pos, const double *col, int64_t n,
                          const FrameParams &host, const FrameParams *P, DevCounts *C) {
    SFB_REQUIRE(ctx->net.loaded, "network weights are not loaded");
    SFB_REQUIRE(ctx->net.enc[0] == 9, "input grid has 9 channels, plan expects " +
                                          std::to_string(ctx->net.enc[0]));
    VoxelSplats V;
    VoxelOut &o = V.vox;
    o.coords = ctx->arena.alloc<int32_t>(3 * n);
    o.feats = ctx->arena.alloc<double>(9 * n);
    o.keys = ctx->arena.alloc<int64_t>(n);
    o.p2v = ctx->arena.alloc<int32_t>(n);
    o.order = ctx->arena.alloc<int32_t>(n);
    o.offsets = ctx->arena.alloc<int32_t>(n + 1);
    if (ctx->net_mode != SFB_NET_SIMT_F64) o.feats32 = ctx->arena.alloc<float>(9 * n);
    voxelize_run(ctx, pos, col, n, host, P, o, C, true);
    ctx->mark(ST_VOXELIZE);
    void *raw = ctx->arena.alloc<double>(14 * n);   // float32 rows, or float64 (SIMT_F64)
    unet_run(ctx, o.coords, o.feats, n, host, P, C, raw, o.feats32);
    ctx->mark(ST_UNET);
    double *blk = ctx->arena.alloc<double>(14 * n);
    V.c = blk;
    V.s = blk + 3 * n;
    V.q = blk + 6 * n;
    V.o = blk + 10 * n;
    V.n = blk + 11 * n;
    head_to_voxel_splats(ctx, raw, o.coords, o.feats, &C->m[0], n, P, V.c, V.s, V.q, V.o, V.n);
    ctx->mark(ST_HEAD);
    return V;
}

RenderInputs splat_inputs(const sfb_splats *s) {
    RenderInputs in{};
    in.centers = s->centers;
    in.scales = s->scales;
    in.quats = s->quaternions;
    in.opac = s->opacities;
    in.n_geom = s->n;
    in.d_n_geom = nullptr;
    in.colors = s->colors;
    in.normals = s->normals;
    in.n_points = s->n;
    return in;
}

// enqueue the fused frame (eager or under capture)
void enqueue_frame(sfb_ctx *ctx, const double *pos, const double *col, int64_t n,
                   const FrameParams &host, FrameParams *P, const sfb_camera *cam,
                   const sfb_render_options *opts, int mask, float *rgb, float *normal,
                   float *depth, float *trans, uint8_t *rgba) {
    write_params(ctx, host, P);
    DevCounts *C = new_counts(ctx);
    VoxelSplats V = neural_voxels(ctx, pos, col, n, host, P, C);
    RenderInputs in{};
    in.centers = V.c;
    in.scales = V.s;
    in.quats = V.q;
    in.opac = V.o;
    in.n_geom = n;
    in.d_n_geom = &C->m[0];
    in.point_to_geom = V.vox.p2v;
    in.geom_offsets = V.vox.offsets;
    in.geom_order = V.vox.order;
    in.colors = col;
    in.normals = V.n;
    in.n_points = n;
    render_run(ctx, in, P, cam->width, cam->height, *opts, mask, C, rgb, normal, depth, trans, rgba);
}

// render_pose shading into the frame parameters; returns the plane mask the
// compositor must accumulate for the mode
int apply_shading(FrameParams &P, const sfb_shading *sh) {
    SFB_REQUIRE(sh, "null shading");
    SFB_REQUIRE(sh->mode == SFB_MODE_RGB || sh->mode == SFB_MODE_NORMAL || sh->mode == SFB_MODE_RELIT,
                "unknown render_pose mode");
    P.shade_mode = sh->mode;
    for (int a = 0; a < 3; ++a) P.light[a] = sh->light[a];
    P.ambient = sh->ambient;
    P.diffuse = sh->diffuse;
    if (sh->mode == SFB_MODE_RELIT) {
        const double l2 = sh->light[0] * sh->light[0] + sh->light[1] * sh->light[1] +
                          sh->light[2] * sh->light[2];
        SFB_REQUIRE(std::fabs(std::sqrt(l2) - 1.0) <= 1e-6, "light_dir must be unit length");
    }
    return sh->mode == SFB_MODE_RGB ? SFB_PLANE_RGB
           : sh->mode == SFB_MODE_NORMAL ? SFB_PLANE_NORMAL : (SFB_PLANE_RGB | SFB_PLANE_NORMAL);
}

}  // namespace

struct sfb_frame_graph {
    // shape key: everything baked into the kernels' launch configuration
    int64_t n;
    int32_t width, height, tile, terminate, mask, key_bits;
    double alpha_max;
    const void *ptrs[7];
    int64_t level_bound[9];   // UNet buffer bounds (unet_level_bounds) baked into the graph
    int net_mode;
    uint64_t net_epoch;
    int seen = 0;                     // eager runs with this key
    cudaGraphExec_t exec = nullptr;
    cudaGraph_t graph = nullptr;
    cudaGraphNode_t param_node = nullptr;
    FrameParams *dev_params = nullptr;
    ~sfb_frame_graph() {
        if (exec) cudaGraphExecDestroy(exec);
        if (graph) cudaGraphDestroy(graph);
    }
};

extern "C" {

int sfb_version(void) { return 2; }

int sfb_ctx_create(int device, sfb_ctx **out) {
    if (!out) return SFB_ERR_ARG;
    *out = nullptr;
    auto *ctx = new (std::nothrow) sfb_ctx();
    if (!ctx) return SFB_ERR_OOM;
    ctx->device = device;
    if (cudaSetDevice(device) != cudaSuccess ||
        cudaDeviceGetAttribute(&ctx->num_sms, cudaDevAttrMultiProcessorCount, device) != cudaSuccess ||
        cudaMallocHost(&ctx->pinned, 4096) != cudaSuccess ||
        cudaStreamCreateWithFlags(&ctx->capture_stream, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&ctx->fork_event, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&ctx->done_event, cudaEventDisableTiming) != cudaSuccess ||
        cudaStreamCreateWithFlags(&ctx->side_stream, cudaStreamNonBlocking) != cudaSuccess ||
        cudaStreamCreateWithFlags(&ctx->aux_stream, cudaStreamNonBlocking) != cudaSuccess) {
        delete ctx;
        return SFB_ERR_CUDA;
    }
    for (auto &e : ctx->side_ev)
        if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) {
            delete ctx;
            return SFB_ERR_CUDA;
        }
    *out = ctx;
    return SFB_OK;
}

int sfb_ctx_destroy(sfb_ctx *ctx) {
    if (!ctx) return SFB_ERR_ARG;
    cudaSetDevice(ctx->device);
    cudaDeviceSynchronize();
    for (auto *g : ctx->graphs) delete g;
    ctx->graphs.clear();
    delete ctx;
    return SFB_OK;
}

const char *sfb_last_error(sfb_ctx *ctx) { return ctx ? ctx->last_error.c_str() : "null context"; }

int sfb_set_stream(sfb_ctx *ctx, void *stream) {
    if (!ctx) return SFB_ERR_ARG;
    ctx->stream = static_cast<cudaStream_t>(stream);
    return SFB_OK;
}

int sfb_set_timing(sfb_ctx *ctx, int on) {
    if (!ctx) return SFB_ERR_ARG;
    ctx->timing = on != 0;
    return SFB_OK;
}

int sfb_set_debug_counters(sfb_ctx *ctx, int64_t *dev_counters) {
    if (!ctx) return SFB_ERR_ARG;
    ctx->debug_counters = dev_counters;
    return SFB_OK;
}

int sfb_set_frame_debug(sfb_ctx *ctx, int64_t capacity, int64_t *source, int32_t *run_start,
                        int32_t *run_count, int32_t *run_rect, int32_t levels,
                        int32_t *level_coords, int32_t *level_maps) {
    if (!ctx || capacity < 0 || levels < 0) return SFB_ERR_ARG;
    FrameDebug D;
    if (capacity > 0) {
        D.cap = capacity;
        D.source = source;
        D.run_start = run_start;
        D.run_count = run_count;
        D.run_rect = run_rect;
        D.levels = levels;
        D.level_coords = level_coords;
        D.level_maps = level_maps;
    }
    ctx->frame_debug = D;
    return SFB_OK;
}

int sfb_set_conv_staging(sfb_ctx *ctx, int mode) {
    if (!ctx || mode < 0 || mode > 2) return SFB_ERR_ARG;
    ctx->conv_stage = mode;
    ++ctx->net_epoch;   // frame graphs captured with another staging are stale
    return SFB_OK;
}

int sfb_set_entry_capacity(sfb_ctx *ctx, int64_t capacity) {
    if (!ctx || capacity < 0) return SFB_ERR_ARG;
    ctx->entry_cap_override = capacity;
    return SFB_OK;
}

int sfb_set_graphs(sfb_ctx *ctx, int on) {
    if (!ctx) return SFB_ERR_ARG;
    ctx->use_graphs = on != 0;
    return SFB_OK;
}

int sfb_stage_times(sfb_ctx *ctx, int32_t *stage_ids, float *ms, int32_t cap, int32_t *n_out) {
    if (!ctx || !n_out) return SFB_ERR_ARG;
    int n = 0;
    for (int i = 1; i < ctx->n_marks && n < cap; ++i) {
        float t = 0.f;
        if (cudaEventSynchronize(ctx->ev[i]) != cudaSuccess ||
            cudaEventElapsedTime(&t, ctx->ev[i - 1], ctx->ev[i]) != cudaSuccess)
            return SFB_ERR_CUDA;
        stage_ids[n] = ctx->stage_id[i];
        ms[n++] = t;
    }
    *n_out = n;
    return SFB_OK;
}

int sfb_get_stats(sfb_ctx *ctx, sfb_stats *out) {
    if (!ctx || !out) return SFB_ERR_ARG;
    if (ctx->last_counts) {
        DevCounts c{};
        if (cudaMemcpy(&c, ctx->last_counts, sizeof(c), cudaMemcpyDeviceToHost) != cudaSuccess)
            return SFB_ERR_CUDA;
        ctx->stats.kept = c.kept;
        ctx->stats.runs = c.runs;
        ctx->stats.fine_entries = c.ef;
        ctx->stats.super_entries = c.es;
        ctx->stats.global_entries = c.g;
        for (int l = 0; l < 8; ++l) ctx->stats.voxels[l] = c.m[l];
    }
    *out = ctx->stats;
    return SFB_OK;
}

int sfb_bbox(sfb_ctx *ctx, const double *positions, int64_t n, double *lo_hi_host) {
    return guard(ctx, [&] { bbox_run(ctx, positions, n, lo_hi_host); });
}

int sfb_bbox_async(sfb_ctx *ctx, const double *positions, int64_t n, uint64_t *ordered) {
    return guard(ctx, [&] {
        SFB_REQUIRE(positions && ordered, "null argument");
        bbox_async_run(ctx, positions, n, ordered);
    });
}

int sfb_voxelize(sfb_ctx *ctx, const double *positions, const double *colors, int64_t n, double s,
                 const double *lo_hi_host, int32_t *coords, double *feats, int64_t *keys,
                 int32_t *p2v, int32_t *order, int32_t *offsets, int64_t *m_host) {
    return guard(ctx, [&] {
        FrameParams host{};
        voxel_layout(lo_hi_host, s, host);
        FrameParams *P = params(ctx, host);
        DevCounts *C = new_counts(ctx);
        VoxelOut o{coords, feats, keys, p2v, order, offsets};
        voxelize_run(ctx, positions, colors, n, host, P, o, C);
        ctx->read_back(&C->m[0], sizeof(int64_t));
        *m_host = ctx->pinned[0];
    });
}

int sfb_kernel_map(sfb_ctx *ctx, const int32_t *coords, int64_t m, int32_t stride, int32_t kernel,
                   int32_t *map_out) {
    return guard(ctx, [&] {
        SFB_REQUIRE(kernel >= 1 && (kernel & 1), "conv kernels must be odd");
        SFB_REQUIRE(stride >= 1, "stride must be positive");
        if (m == 0) return;
        HashTable h = hash_build(ctx, coords, nullptr, m);
        const int taps = kernel * kernel * kernel;
        int32_t *tm = ctx->arena.alloc<int32_t>((size_t)taps * m);
        kernel_map_build(ctx, h, coords, nullptr, m, stride, kernel, tm);
        k_tap_transpose<<<dgrid(m * taps, 256), 256, 0, ctx->stream>>>(tm, m, taps, map_out);
        SFB_CHECK_LAUNCH();
    });
}

int sfb_transposed_map(sfb_ctx *ctx, const int32_t *parent_coords, int64_t m_parent,
                       int32_t parent_stride, const int32_t *targets, int64_t m_targets,
                       int32_t *parent_out, int32_t *tap_out) {
    return guard(ctx, [&] {
        SFB_REQUIRE(parent_stride >= 2 && (parent_stride & (parent_stride - 1)) == 0,
                    "transposed conv needs a stride >= 2 grid to subdivide");
        if (m_targets == 0) return;
        HashTable h = hash_build(ctx, parent_coords, nullptr, m_parent);
        transposed_lookup(ctx, h, parent_stride, targets, nullptr, m_targets, parent_out, tap_out);
    });
}

int sfb_pool(sfb_ctx *ctx, const int32_t *coords, const float *feats, int64_t m, int32_t c,
             int32_t stride, int32_t *parent_coords, float *parent_feats, int32_t *c2p,
             int64_t *m_parent_host) {
    return guard(ctx, [&] {
        FrameParams host{};
        coords_layout(ctx, coords, m, host);
        FrameParams *P = params(ctx, host);
        DevCounts *C = new_counts(ctx);
        *reinterpret_cast<int64_t *>(ctx->pinned) = m;
        SFB_CUDA(cudaMemcpyAsync(&C->m[0], ctx->pinned, sizeof(int64_t), cudaMemcpyHostToDevice,
                                 ctx->stream));
        pool_build(ctx, coords, &C->m[0], m, stride, host, P, feats, c, c, parent_coords,
                   parent_feats, c, c2p, &C->m[1]);
        ctx->read_back(&C->m[1], sizeof(int64_t));
        *m_parent_host = ctx->pinned[0];
    });
}

int sfb_pool_f64(sfb_ctx *ctx, const int32_t *coords, const double *feats, int64_t m, int32_t c,
                 int32_t stride, int32_t *parent_coords, double *parent_feats, int32_t *c2p,
                 int64_t *m_parent_host) {
    return guard(ctx, [&] {
        FrameParams host{};
        coords_layout(ctx, coords, m, host);
        FrameParams *P = params(ctx, host);
        DevCounts *C = new_counts(ctx);
        *reinterpret_cast<int64_t *>(ctx->pinned) = m;
        SFB_CUDA(cudaMemcpyAsync(&C->m[0], ctx->pinned, sizeof(int64_t), cudaMemcpyHostToDevice,
                                 ctx->stream));
        pool_build(ctx, coords, &C->m[0], m, stride, host, P, feats, c, c, parent_coords,
                   parent_feats, c, c2p, &C->m[1]);
        ctx->read_back(&C->m[1], sizeof(int64_t));
        *m_parent_host = ctx->pinned[0];
    });
}

int sfb_lookup(sfb_ctx *ctx, const int32_t *coords, int64_t m, const int32_t *query, int64_t nq,
               int64_t *rows) {
    return guard(ctx, [&] {
        SFB_REQUIRE((coords || m == 0) && (query || nq == 0) && (rows || nq == 0), "null argument");
        lookup_run(ctx, coords, m, query, nq, rows);
    });
}

int sfb_net_load(sfb_ctx *ctx, const void *blob, size_t nbytes) {
    return guard(ctx, [&] {
        net_load(ctx, blob, nbytes);
        ++ctx->net_epoch;
    });
}

int sfb_net_set_mode(sfb_ctx *ctx, int mode) {
    if (!ctx || (mode != SFB_NET_SIMT_F32 && mode != SFB_NET_TC_TF32X3 && mode != SFB_NET_TC_BF16 &&
                 mode != SFB_NET_SIMT_F64))
        return SFB_ERR_ARG;
    ctx->net_mode = mode;
    return SFB_OK;
}

static const NetLayer &pick_layer(sfb_ctx *ctx, int layer) {
    if (layer < 0) {
        SFB_REQUIRE(ctx->adhoc.w, "no standalone layer set (sfb_layer_set)");
        return ctx->adhoc;
    }
    SFB_REQUIRE(ctx->net.loaded, "network weights are not loaded");
    SFB_REQUIRE(layer < (int)ctx->net.layers.size(), "layer index out of range");
    return ctx->net.layers[layer];
}

int sfb_layer_set(sfb_ctx *ctx, int kind, int kernel, int cin, int cout, const float *w_host,
                  const float *b_host) {
    return guard(ctx, [&] { layer_set(ctx, kind, kernel, cin, cout, w_host, b_host); });
}

int sfb_sparse_conv(sfb_ctx *ctx, int layer, const int32_t *coords, const float *feats, int64_t m,
                    int32_t stride, int relu, float *out) {
    return guard(ctx, [&] {
        const NetLayer &L = pick_layer(ctx, layer);
        SFB_REQUIRE(L.kind == 0, "expected a conv spec");
        if (m == 0) return;
        HashTable h = hash_build(ctx, coords, nullptr, m);
        int32_t *nbr = ctx->arena.alloc<int32_t>((size_t)L.taps * m);
        kernel_map_build(ctx, h, coords, nullptr, m, stride, L.kernel, nbr);
        conv_layer(ctx, L, feats, L.cin, nbr, m, nullptr, m, relu, out, L.cout);
    });
}

int sfb_transposed_conv(sfb_ctx *ctx, int layer, const int32_t *parent_coords,
                        const float *parent_feats, int64_t m_parent, int32_t parent_stride,
                        const int32_t *targets, int64_t m_targets, int relu, float *out) {
    return guard(ctx, [&] {
        const NetLayer &L = pick_layer(ctx, layer);
        SFB_REQUIRE(L.kind == 1, "expected a transposed_conv spec");
        if (m_targets == 0) return;
        HashTable h = hash_build(ctx, parent_coords, nullptr, m_parent);
        int32_t *parent = ctx->arena.alloc<int32_t>(m_targets);
        int32_t *tap = ctx->arena.alloc<int32_t>(m_targets);
        transposed_lookup(ctx, h, parent_stride, targets, nullptr, m_targets, parent, tap);
        tconv_layer(ctx, L, parent_feats, L.cin, parent, tap, nullptr, m_targets, relu, out, L.cout);
    });
}

int sfb_unet_forward(sfb_ctx *ctx, const int32_t *coords, const double *feats9, int64_t m0,
                     void *raw_out) {
    return guard(ctx, [&] {
        SFB_REQUIRE(m0 > 0, "empty voxel grid");
        FrameParams host{};
        coords_layout(ctx, coords, m0, host);
        FrameParams *P = params(ctx, host);
        DevCounts *C = new_counts(ctx);
        *reinterpret_cast<int64_t *>(ctx->pinned) = m0;
        SFB_CUDA(cudaMemcpyAsync(&C->m[0], ctx->pinned, sizeof(int64_t), cudaMemcpyHostToDevice,
                                 ctx->stream));
        unet_run(ctx, coords, feats9, m0, host, P, C, raw_out);
        SFB_CUDA(cudaStreamSynchronize(ctx->stream));   // pinned staging reused next call
    });
}

int sfb_activate_head(sfb_ctx *ctx, const double *raw, int64_t m, double scale, double *delta,
                      double *sigma, double *quat, double *opacity, double *normal) {
    return guard(ctx, [&] { activate_run(ctx, raw, m, scale, delta, sigma, quat, opacity, normal); });
}

int sfb_estimate_neural(sfb_ctx *ctx, const double *positions, const double *colors, int64_t n,
                        double s, const double *lo_hi_host, double *centers, double *scales,
                        double *quaternions, double *opacities, double *colors_out,
                        double *normals) {
    return guard(ctx, [&] {
        FrameParams host{};
        voxel_layout(lo_hi_host, s, host);
        FrameParams *P = params(ctx, host);
        DevCounts *C = new_counts(ctx);
        VoxelSplats V = neural_voxels(ctx, positions, colors, n, host, P, C);
        k_expand_splats<<<dgrid(n, 256), 256, 0, ctx->stream>>>(
            V.vox.p2v, n, V.c, V.s, V.q, V.o, V.n, colors, centers, scales, quaternions, opacities,
            colors_out, normals);
        SFB_CHECK_LAUNCH();
    });
}

int sfb_render(sfb_ctx *ctx, const sfb_splats *splats, const sfb_camera *cam,
               const sfb_render_options *opts, int32_t plane_mask, const double *bg, float *rgb,
               float *normal, float *depth, float *trans) {
    return guard(ctx, [&] {
        SFB_REQUIRE(splats && cam && opts, "null argument");
        FrameParams *P = params(ctx, camera_params(cam, bg));
        DevCounts *C = new_counts(ctx);
        render_run(ctx, splat_inputs(splats), P, cam->width, cam->height, *opts, plane_mask, C, rgb,
                   normal, depth, trans);
    });
}

int sfb_knn(sfb_ctx *ctx, const double *positions, int64_t n, int32_t k, double *d2, int64_t *idx) {
    return guard(ctx, [&] {
        SFB_REQUIRE(positions && d2 && idx, "null argument");
        knn_run(ctx, positions, n, k, d2, idx);
    });
}

int sfb_nn_distance(sfb_ctx *ctx, const double *d2, int64_t n, int32_t k, double *dist) {
    return guard(ctx, [&] {
        SFB_REQUIRE(d2 && dist && k >= 1, "null argument");
        if (n > 0) nn_dist_run(ctx, d2, n, k, dist);
    });
}

int sfb_local_pca(sfb_ctx *ctx, const double *positions, int64_t n, int32_t k, const int64_t *idx,
                  double sigma_mult, double dbar, const double *centroid, double *scales,
                  double *quats, double *normals) {
    return guard(ctx, [&] {
        SFB_REQUIRE(positions && idx && centroid && scales && quats && normals, "null argument");
        double *mc = ctx->arena.alloc<double>(3);
        SFB_CUDA(cudaMemcpyAsync(mc, centroid, 3 * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
        if (n > 0) local_pca_run(ctx, positions, n, k, sigma_mult, idx, dbar, mc, scales, quats, normals);
        SFB_CUDA(cudaStreamSynchronize(ctx->stream));   // centroid_host is the caller's stack
    });
}

int sfb_ply_decode(sfb_ctx *ctx, const uint8_t *body, int64_t n, int32_t stride,
                   const int32_t *offsets, double *positions, double *colors, double *normals) {
    return guard(ctx, [&] {
        SFB_REQUIRE(offsets && positions && colors && (body || n == 0), "null argument");
        ply_decode_run(ctx, body, n, stride, offsets, positions, colors, normals);
    });
}

int sfb_spl1_decode(sfb_ctx *ctx, const float *rows, int64_t n, double *c, double *s, double *q,
                    double *o, double *col, double *nrm) {
    return guard(ctx, [&] {
        SFB_REQUIRE(n == 0 || (rows && c && s && q && o && col && nrm), "null argument");
        spl1_decode_run(ctx, rows, n, c, s, q, o, col, nrm);
    });
}

int sfb_spl1_encode(sfb_ctx *ctx, const sfb_splats *splats, float *rows) {
    return guard(ctx, [&] {
        SFB_REQUIRE(splats && (rows || splats->n == 0), "null argument");
        spl1_encode_run(ctx, *splats, rows);
    });
}

int sfb_render_backward(sfb_ctx *ctx, const sfb_splats *splats, const sfb_camera *cam,
                        const sfb_render_options *opts, int32_t mode, const double *bg,
                        const double *upstream, double *d_centers, double *d_scales,
                        double *d_quaternions, double *d_opacities, double *d_colors,
                        double *d_normals) {
    return guard(ctx, [&] {
        SFB_REQUIRE(splats && cam && opts && upstream, "null argument");
        SFB_REQUIRE(d_centers && d_scales && d_quaternions && d_opacities, "null gradient buffer");
        FrameParams *P = params(ctx, camera_params(cam, bg));
        DevCounts *C = new_counts(ctx);
        render_backward_run(ctx, splat_inputs(splats), P, cam->width, cam->height, *opts, mode, C,
                            upstream, d_centers, d_scales, d_quaternions, d_opacities, d_colors,
                            d_normals);
    });
}

int sfb_render_rgba(sfb_ctx *ctx, const sfb_splats *splats, const sfb_camera *cam,
                    const sfb_render_options *opts, const sfb_shading *shading, const double *bg,
                    uint8_t *rgba) {
    return guard(ctx, [&] {
        SFB_REQUIRE(splats && cam && opts && rgba, "null argument");
        FrameParams host = camera_params(cam, bg);
        const int mask = apply_shading(host, shading);
        FrameParams *P = params(ctx, host);
        DevCounts *C = new_counts(ctx);
        render_run(ctx, splat_inputs(splats), P, cam->width, cam->height, *opts, mask, C, nullptr,
                   nullptr, nullptr, nullptr, rgba);
    });
}

int sfb_project(sfb_ctx *ctx, const sfb_splats *s, const sfb_camera *cam, double z_near,
                double dilation, double *sx, double *sy, double *depth, double *ca, double *cb,
                double *cc, double *radius, uint8_t *keep) {
    return guard(ctx, [&] {
        FrameParams *P = params(ctx, camera_params(cam, nullptr));
        project_run(ctx, s->centers, s->quaternions, s->scales, nullptr, s->n, P, z_near, dilation,
                    sx, sy, depth, ca, cb, cc, radius, keep);
    });
}

int sfb_prepare_debug(sfb_ctx *ctx, const sfb_splats *s, const sfb_camera *cam, int32_t tile,
                      int64_t *source, double *radius, int64_t *offsets, int64_t *ids,
                      int64_t cap, int64_t *k_host, int64_t *e_host) {
    return guard(ctx, [&] {
        SFB_REQUIRE(tile >= 1, "tile_size must be positive");
        FrameParams *P = params(ctx, camera_params(cam, nullptr));
        DevCounts *C = new_counts(ctx);
        prepare_debug_run(ctx, splat_inputs(s), P, cam->width, cam->height, tile, C, source,
                          radius, offsets, ids, cap, k_host, e_host);
    });
}

static int frame_impl(sfb_ctx *ctx, const double *positions, const double *colors, int64_t n,
                      double s, const double *lo_hi_host, const sfb_camera *cam,
                      const sfb_render_options *opts, int32_t plane_mask, const double *bg,
                      float *rgb, float *normal, float *depth, float *trans, uint8_t *rgba,
                      const sfb_shading *shading) {
    return guard(ctx, [&] {
        SFB_REQUIRE(cam && opts, "null argument");
        SFB_REQUIRE(n >= 2, "voxelization needs at least 2 points");
        FrameParams host = camera_params(cam, bg);
        if (rgba) plane_mask = apply_shading(host, shading);
        voxel_layout(lo_hi_host, s, host);
        // the graph bakes in the voxel-key radix pass count (8-bit digits) and the
        // key width (32 / 64 bit): key on the pass count in both ranges
        const int key_bits = ((std::max(host.total, 1) + 7) / 8) * 8;
        if (!ctx->use_graphs || ctx->timing || ctx->frame_debug.cap > 0 || ctx->entry_cap_override > 0) {
            FrameParams *P = ctx->arena.alloc<FrameParams>(1);
            enqueue_frame(ctx, positions, colors, n, host, P, cam, opts, plane_mask, rgb, normal,
                          depth, trans, rgba);
            return;
        }
        // ---- graph path: find / build the graph of this shape
        sfb_frame_graph *G = nullptr;
        const void *ptrs[7] = {positions, colors, rgb, normal, depth, trans, rgba};
        int64_t lb[9] = {};
        if (ctx->net.loaded) unet_level_bounds(host, n, std::min(ctx->net.levels, 8), lb);
        for (auto *g : ctx->graphs)
            if (g->n == n && g->width == cam->width && g->height == cam->height &&
                g->tile == opts->tile_size && g->terminate == opts->early_termination &&
                g->alpha_max == opts->alpha_max && g->mask == plane_mask && g->key_bits == key_bits &&
                g->net_mode == ctx->net_mode && g->net_epoch == ctx->net_epoch &&
                std::equal(ptrs, ptrs + 7, g->ptrs) && std::equal(lb, lb + 9, g->level_bound))
                G = g;
        if (!G) {
            G = new sfb_frame_graph();
            G->n = n;
            G->width = cam->width;
            G->height = cam->height;
            G->tile = opts->tile_size;
            G->terminate = opts->early_termination;
            G->alpha_max = opts->alpha_max;
            G->mask = plane_mask;
            G->key_bits = key_bits;
            G->net_mode = ctx->net_mode;
            G->net_epoch = ctx->net_epoch;
            std::copy(ptrs, ptrs + 7, G->ptrs);
            std::copy(lb, lb + 9, G->level_bound);
            if (ctx->graphs.size() >= 32) {
                delete ctx->graphs.front();
                ctx->graphs.erase(ctx->graphs.begin());
            }
            ctx->graphs.push_back(G);
        }
        if (!G->exec && G->seen == 0) {
            // first call of this shape: eager run (grows the arena, sets kernel attributes)
            FrameParams *P = ctx->arena.alloc<FrameParams>(1);
            enqueue_frame(ctx, positions, colors, n, host, P, cam, opts, plane_mask, rgb, normal,
                          depth, trans, rgba);
            G->seen = 1;
            // size hints for the capture (grids only; kernels loop over device counts)
            DevCounts c{};
            SFB_CUDA(cudaMemcpyAsync(&c, ctx->last_counts, sizeof(c), cudaMemcpyDeviceToHost,
                                     ctx->stream));
            SFB_CUDA(cudaStreamSynchronize(ctx->stream));
            for (int l = 0; l < 9; ++l) ctx->hint_m[l] = c.m[l];
            ctx->hint_kept = c.kept;
            ctx->hint_runs = c.runs;
            ctx->hint_e = c.es_req + c.ef_req;
            return;
        }
        if (!G->exec) {
            // capture on the library's own stream; the caller's stream replays it
            cudaStream_t user = ctx->stream;
            SFB_CUDA(cudaStreamSynchronize(user));
            ctx->stream = ctx->capture_stream;
            FrameParams *P = ctx->arena.alloc<FrameParams>(1);
            G->dev_params = P;
            SFB_CUDA(cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal));
            ctx->arena.no_grow = true;
            try {
                enqueue_frame(ctx, positions, colors, n, host, P, cam, opts, plane_mask, rgb,
                              normal, depth, trans, rgba);
                ctx->arena.no_grow = false;
            } catch (const ArenaGrowth &) {
                // the eager run used less scratch (size hints changed a path):
                // drop the capture, run this frame eagerly (growing the arena),
                // capture on the next call
                ctx->arena.no_grow = false;
                join_forked(ctx);   // side / aux branches of the abandoned capture
                cudaGraph_t junk = nullptr;
                cudaStreamEndCapture(ctx->stream, &junk);
                if (junk) cudaGraphDestroy(junk);
                cudaGetLastError();
                ctx->stream = user;
                ctx->arena.reset();
                FrameParams *P2 = ctx->arena.alloc<FrameParams>(1);
                enqueue_frame(ctx, positions, colors, n, host, P2, cam, opts, plane_mask, rgb, normal,
                              depth, trans, rgba);
                return;
            } catch (...) {
                ctx->arena.no_grow = false;
                join_forked(ctx);
                cudaGraph_t junk = nullptr;
                cudaStreamEndCapture(ctx->stream, &junk);
                if (junk) cudaGraphDestroy(junk);
                ctx->stream = user;
                throw;
            }
            cudaError_t e = cudaStreamEndCapture(ctx->stream, &G->graph);
            ctx->stream = user;
            SFB_CUDA(e);
            SFB_CUDA(cudaGraphInstantiate(&G->exec, G->graph, 0));
            size_t nn = 0;
            SFB_CUDA(cudaGraphGetNodes(G->graph, nullptr, &nn));
            std::vector<cudaGraphNode_t> nodes(nn);
            SFB_CUDA(cudaGraphGetNodes(G->graph, nodes.data(), &nn));
            for (auto nd : nodes) {
                cudaGraphNodeType ty;
                SFB_CUDA(cudaGraphNodeGetType(nd, &ty));
                if (ty != cudaGraphNodeTypeKernel) continue;
                cudaKernelNodeParams kp;
                SFB_CUDA(cudaGraphKernelNodeGetParams(nd, &kp));
                if (kp.func == write_params_func()) {
                    G->param_node = nd;
                    break;
                }
            }
            SFB_REQUIRE(G->param_node, "frame graph has no parameter node");
            ctx->graph_nodes = (int64_t)nn;
        }
        // replay: new parameters into the first node, then the whole frame
        cudaKernelNodeParams kp{};
        FrameParams *dst = G->dev_params;
        void *args[2] = {&host, &dst};
        kp.func = const_cast<void *>(write_params_func());
        kp.gridDim = dim3(1);
        kp.blockDim = dim3(1);
        kp.sharedMemBytes = 0;
        kp.kernelParams = args;
        SFB_CUDA(cudaGraphExecKernelNodeSetParams(G->exec, G->param_node, &kp));
        SFB_CUDA(cudaGraphLaunch(G->exec, ctx->stream));
    });
}

int sfb_frame(sfb_ctx *ctx, const double *positions, const double *colors, int64_t n, double s,
              const double *lo_hi_host, const sfb_camera *cam, const sfb_render_options *opts,
              int32_t plane_mask, const double *bg, float *rgb, float *normal, float *depth,
              float *trans) {
    return frame_impl(ctx, positions, colors, n, s, lo_hi_host, cam, opts, plane_mask, bg, rgb,
                      normal, depth, trans, nullptr, nullptr);
}

int sfb_frame_rgba(sfb_ctx *ctx, const double *positions, const double *colors, int64_t n,
                   double s, const double *lo_hi_host, const sfb_camera *cam,
                   const sfb_render_options *opts, const sfb_shading *shading, const double *bg,
                   uint8_t *rgba) {
    if (!rgba) return SFB_ERR_ARG;
    return frame_impl(ctx, positions, colors, n, s, lo_hi_host, cam, opts, 0, bg, nullptr, nullptr,
                      nullptr, nullptr, rgba, shading);
}

}  // extern "C"
