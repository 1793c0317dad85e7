// C ABI of libsfb200 (declared in include/sfb200.h): argument checks, error
// codes, arena reset per call, and the fused pipelines built from the stages
// in voxelize.cu / hashmap.cu / net.cu / render.cu.
#include "common.cuh"

using namespace sfb;

namespace {

template <class F>
int guard(sfb_ctx *ctx, F &&f) {
    if (!ctx) return SFB_ERR_ARG;
    try {
        SFB_CUDA(cudaSetDevice(ctx->device));
        ctx->arena.reset();
        ctx->n_marks = 0;
        ctx->mark(ST_BEGIN);
        f();
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

__global__ void k_expand_splats(const int32_t *__restrict__ p2v, int64_t n,
                                const double *__restrict__ vc, const double *__restrict__ vs,
                                const double *__restrict__ vq, const double *__restrict__ vo,
                                const double *__restrict__ vn, const double *__restrict__ col,
                                double *centers, double *scales, double *quats, double *opac,
                                double *colors, double *normals) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    int64_t v = p2v[i];
    for (int a = 0; a < 3; ++a) {
        centers[3 * i + a] = vc[3 * v + a];
        scales[3 * i + a] = vs[3 * v + a];
        normals[3 * i + a] = vn[3 * v + a];
        if (colors) colors[3 * i + a] = col[3 * i + a];
    }
    for (int a = 0; a < 4; ++a) quats[4 * i + a] = vq[4 * v + a];
    opac[i] = vo[v];
}

__global__ void k_tap_transpose(const int32_t *__restrict__ tm, int64_t m, int taps,
                                int32_t *__restrict__ out) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= m * taps) return;
    int64_t r = i / taps;
    int t = (int)(i % taps);
    out[i] = tm[(int64_t)t * m + r];
}

struct VoxelSplats {
    VoxelOut vox;
    double *c, *s, *q, *o, *n;
};

VoxelSplats neural_voxels(sfb_ctx *ctx, const double *pos, const double *col, int64_t n, double s,
                          const double *lo_hi) {
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
    voxelize_run(ctx, pos, col, n, s, lo_hi, o);
    ctx->mark(ST_VOXELIZE);
    int64_t m = o.m;
    float *raw = ctx->arena.alloc<float>(14 * m);
    unet_run(ctx, o.coords, o.feats, m, raw);
    ctx->mark(ST_UNET);
    double *blk = ctx->arena.alloc<double>(14 * m);
    V.c = blk;
    V.s = blk + 3 * m;
    V.q = blk + 6 * m;
    V.o = blk + 10 * m;
    V.n = blk + 11 * m;
    head_to_voxel_splats(ctx, raw, o.coords, o.feats, m, 1.0 / s, V.c, V.s, V.q, V.o, V.n);
    ctx->mark(ST_HEAD);
    return V;
}

}  // namespace

extern "C" {

int sfb_version(void) { return 1; }

int sfb_ctx_create(int device, sfb_ctx **out) {
    if (!out) return SFB_ERR_ARG;
    *out = nullptr;
    auto *ctx = new (std::nothrow) sfb_ctx();
    if (!ctx) return SFB_ERR_OOM;
    ctx->device = device;
    if (cudaSetDevice(device) != cudaSuccess ||
        cudaDeviceGetAttribute(&ctx->num_sms, cudaDevAttrMultiProcessorCount, device) != cudaSuccess ||
        cudaMallocHost(&ctx->pinned, 4096) != cudaSuccess) {
        delete ctx;
        return SFB_ERR_CUDA;
    }
    *out = ctx;
    return SFB_OK;
}

int sfb_ctx_destroy(sfb_ctx *ctx) {
    if (!ctx) return SFB_ERR_ARG;
    cudaSetDevice(ctx->device);
    if (ctx->stream) cudaStreamSynchronize(ctx->stream);
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
    *out = ctx->stats;
    return SFB_OK;
}

int sfb_bbox(sfb_ctx *ctx, const double *positions, int64_t n, double *lo_hi_host) {
    return guard(ctx, [&] { bbox_run(ctx, positions, n, lo_hi_host); });
}

int sfb_voxelize(sfb_ctx *ctx, const double *positions, const double *colors, int64_t n, double s,
                 const double *lo_hi_host, int32_t *coords, double *feats, int64_t *keys,
                 int32_t *p2v, int32_t *order, int32_t *offsets, int64_t *m_host) {
    return guard(ctx, [&] {
        VoxelOut o{coords, feats, keys, p2v, order, offsets, 0};
        voxelize_run(ctx, positions, colors, n, s, lo_hi_host, o);
        *m_host = o.m;
    });
}

int sfb_kernel_map(sfb_ctx *ctx, const int32_t *coords, int64_t m, int32_t stride, int32_t kernel,
                   int32_t *map_out) {
    return guard(ctx, [&] {
        SFB_REQUIRE(kernel >= 1 && (kernel & 1), "conv kernels must be odd");
        SFB_REQUIRE(stride >= 1, "stride must be positive");
        HashTable h = hash_build(ctx, coords, m);
        int taps = kernel * kernel * kernel;
        int32_t *tm = ctx->arena.alloc<int32_t>((size_t)taps * (m > 0 ? m : 1));
        kernel_map_build(ctx, h, coords, m, stride, kernel, tm);
        // (taps, m) -> (m, taps) for the caller
        if (m > 0) {
            k_tap_transpose<<<grid_for(m * taps, 256), 256, 0, ctx->stream>>>(tm, m, taps, map_out);
            SFB_CHECK_LAUNCH();
        }
    });
}

int sfb_transposed_map(sfb_ctx *ctx, const int32_t *parent_coords, int64_t m_parent,
                       int32_t parent_stride, const int32_t *targets, int64_t m_targets,
                       int32_t *parent_out, int32_t *tap_out) {
    return guard(ctx, [&] {
        SFB_REQUIRE(parent_stride >= 2 && (parent_stride & (parent_stride - 1)) == 0,
                    "transposed conv needs a stride >= 2 grid to subdivide");
        HashTable h = hash_build(ctx, parent_coords, m_parent);
        transposed_lookup(ctx, h, parent_stride, targets, m_targets, parent_out, tap_out);
    });
}

int sfb_pool(sfb_ctx *ctx, const int32_t *coords, const float *feats, int64_t m, int32_t c,
             int32_t stride, int32_t *parent_coords, float *parent_feats, int32_t *c2p,
             int64_t *m_parent_host) {
    return guard(ctx, [&] {
        *m_parent_host = pool_build(ctx, coords, m, stride, feats, c, c, parent_coords,
                                    parent_feats, c, c2p);
    });
}

int sfb_net_load(sfb_ctx *ctx, const void *blob, size_t nbytes) {
    return guard(ctx, [&] { net_load(ctx, blob, nbytes); });
}

int sfb_net_set_mode(sfb_ctx *ctx, int mode) {
    if (!ctx || (mode != SFB_NET_SIMT_F32 && mode != SFB_NET_TC_TF32X3)) return SFB_ERR_ARG;
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
        HashTable h = hash_build(ctx, coords, m);
        int32_t *nbr = ctx->arena.alloc<int32_t>((size_t)L.taps * (m > 0 ? m : 1));
        kernel_map_build(ctx, h, coords, m, stride, L.kernel, nbr);
        conv_layer(ctx, L, feats, L.cin, nbr, m, relu, out, L.cout);
    });
}

int sfb_transposed_conv(sfb_ctx *ctx, int layer, const int32_t *parent_coords,
                        const float *parent_feats, int64_t m_parent, int32_t parent_stride,
                        const int32_t *targets, int64_t m_targets, int relu, float *out) {
    return guard(ctx, [&] {
        const NetLayer &L = pick_layer(ctx, layer);
        SFB_REQUIRE(L.kind == 1, "expected a transposed_conv spec");
        HashTable h = hash_build(ctx, parent_coords, m_parent);
        int32_t *parent = ctx->arena.alloc<int32_t>(m_targets + 1);
        int32_t *tap = ctx->arena.alloc<int32_t>(m_targets + 1);
        transposed_lookup(ctx, h, parent_stride, targets, m_targets, parent, tap);
        tconv_layer(ctx, L, parent_feats, L.cin, parent, tap, m_targets, relu, out, L.cout);
    });
}

int sfb_unet_forward(sfb_ctx *ctx, const int32_t *coords, const double *feats9, int64_t m0,
                     float *raw_out) {
    return guard(ctx, [&] { unet_run(ctx, coords, feats9, m0, raw_out); });
}

int sfb_activate_head(sfb_ctx *ctx, const float *raw, int64_t m, double scale, double *delta,
                      double *sigma, double *quat, double *opacity, double *normal) {
    return guard(ctx, [&] { activate_run(ctx, raw, m, scale, delta, sigma, quat, opacity, normal); });
}

int sfb_estimate_neural(sfb_ctx *ctx, const double *positions, const double *colors, int64_t n,
                        double s, const double *lo_hi_host, double *centers, double *scales,
                        double *quaternions, double *opacities, double *colors_out,
                        double *normals) {
    return guard(ctx, [&] {
        VoxelSplats V = neural_voxels(ctx, positions, colors, n, s, lo_hi_host);
        k_expand_splats<<<grid_for(n, 256), 256, 0, ctx->stream>>>(
            V.vox.p2v, n, V.c, V.s, V.q, V.o, V.n, colors, centers, scales, quaternions, opacities,
            colors_out, normals);
        SFB_CHECK_LAUNCH();
    });
}

static RenderInputs splat_inputs(const sfb_splats *s) {
    RenderInputs in{};
    in.centers = s->centers;
    in.scales = s->scales;
    in.quats = s->quaternions;
    in.opac = s->opacities;
    in.n_geom = s->n;
    in.colors = s->colors;
    in.normals = s->normals;
    in.n_points = s->n;
    return in;
}

int sfb_render(sfb_ctx *ctx, const sfb_splats *splats, const sfb_camera *cam,
               const sfb_render_options *opts, int32_t plane_mask, const double *bg, float *rgb,
               float *normal, float *depth, float *trans) {
    return guard(ctx, [&] {
        SFB_REQUIRE(splats && cam && opts, "null argument");
        render_run(ctx, splat_inputs(splats), *cam, *opts, plane_mask, bg, rgb, normal, depth, trans);
    });
}

int sfb_project(sfb_ctx *ctx, const sfb_splats *s, const sfb_camera *cam, double z_near,
                double dilation, double *sx, double *sy, double *depth, double *ca, double *cb,
                double *cc, double *radius, uint8_t *keep) {
    return guard(ctx, [&] {
        project_run(ctx, s->centers, s->quaternions, s->scales, s->n, *cam, z_near, dilation, sx,
                    sy, depth, ca, cb, cc, radius, keep);
    });
}

int sfb_prepare_debug(sfb_ctx *ctx, const sfb_splats *s, const sfb_camera *cam, int32_t tile,
                      int64_t *source, double *radius, int64_t *offsets, int64_t *ids,
                      int64_t cap, int64_t *k_host, int64_t *e_host) {
    return guard(ctx, [&] {
        SFB_REQUIRE(tile >= 1, "tile_size must be positive");
        prepare_debug_run(ctx, splat_inputs(s), *cam, tile, source, radius, offsets, ids, cap,
                          k_host, e_host);
    });
}

int sfb_frame(sfb_ctx *ctx, const double *positions, const double *colors, int64_t n, double s,
              const double *lo_hi_host, const sfb_camera *cam, const sfb_render_options *opts,
              int32_t plane_mask, const double *bg, float *rgb, float *normal, float *depth,
              float *trans) {
    return guard(ctx, [&] {
        SFB_REQUIRE(cam && opts, "null argument");
        VoxelSplats V = neural_voxels(ctx, positions, colors, n, s, lo_hi_host);
        RenderInputs in{};
        in.centers = V.c;
        in.scales = V.s;
        in.quats = V.q;
        in.opac = V.o;
        in.n_geom = V.vox.m;
        in.point_to_geom = V.vox.p2v;
        in.colors = colors;
        in.normals = V.n;
        in.n_points = n;
        render_run(ctx, in, *cam, *opts, plane_mask, bg, rgb, normal, depth, trans);
    });
}

}  // extern "C"
