/*
 * sfb200 — B200-native (sm_100a) P2ENet + Gaussian-splat render path, C ABI.
 *
 * The drop-in boundary of this repo. Every entry point takes plain pointers
 * and sizes (no torch types); array arguments are DEVICE pointers unless the
 * name says host, and are caller-owned (the library never frees them).
 * Scratch comes from a per-context grow-only arena; all work is stream-ordered
 * on the context's stream (sfb_set_stream). Calls return SFB_OK (0) or an
 * error code; sfb_last_error(ctx) gives the message.
 *
 * Each entry cites the reference interface it replaces (paths relative to
 * /root/reference/pkg/src/splatforge). Layouts follow the reference:
 * float64 SoA splats (gaussians.py:28-84, quaternions w,x,y,z), camera
 * p_cam = R p + t (gaussians.py:87-137), planes row-major (H, W[, 3]).
 */
#ifndef SFB200_H
#define SFB200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
    SFB_OK = 0,
    SFB_ERR_ARG = 1,    /* invalid argument (the reference raises ValueError) */
    SFB_ERR_OOM = 2,    /* device allocation failed */
    SFB_ERR_CUDA = 3,   /* CUDA runtime / launch error */
    SFB_ERR_STATE = 4,  /* e.g. network not loaded */
};

/* Render planes (bit mask for sfb_render). */
enum { SFB_PLANE_RGB = 1, SFB_PLANE_NORMAL = 2, SFB_PLANE_DEPTH = 4 };

/* P2ENet arithmetic: fp32 SIMT gather-GEMM; tcgen05 tf32 hi/lo split
 * (fp32-accurate, the default and the parity mode); tcgen05 single bf16
 * operands with fp32 accumulation (the north star's fast mode; does not meet
 * the 1e-3 Gaussian-parameter bound). */
enum { SFB_NET_SIMT_F32 = 0, SFB_NET_TC_TF32X3 = 1, SFB_NET_TC_BF16 = 2, SFB_NET_SIMT_F64 = 3 };
/* SFB_NET_SIMT_F64: float64 features with float32 weights upcast, the
 * reference network's own arithmetic (sparsenet.py:207-210), on the FP64
 * pipe — the end-to-end exactness mode (parameters ~1e-13 from the
 * reference instead of ~1e-6). */

typedef struct sfb_ctx sfb_ctx;

typedef struct {
    double rot[9];      /* row-major; rows are the camera axes */
    double trans[3];
    double fx, fy, cx, cy;
    int32_t width, height;
} sfb_camera;

typedef struct {        /* rasterizer.py:25-29 RenderOptions */
    int32_t tile_size;  /* 16 */
    int32_t early_termination;
    double alpha_max;   /* 0.99 */
} sfb_render_options;

typedef struct {        /* gaussians.py:28-84 Splats, float64 SoA, device */
    const double *centers;      /* (n,3) */
    const double *scales;       /* (n,3) sigma, strictly positive */
    const double *quaternions;  /* (n,4) w,x,y,z */
    const double *opacities;    /* (n,) */
    const double *colors;       /* (n,3) */
    const double *normals;      /* (n,3) */
    int64_t n;
} sfb_splats;

typedef struct {        /* per-call timing / size report (host struct) */
    int64_t kept;       /* splats surviving the cull */
    int64_t runs;       /* depth-ordered runs of identical geometry */
    int64_t fine_entries, super_entries, global_entries;
    int64_t voxels[8];  /* per-level voxel counts of the last network pass */
} sfb_stats;

/* ---- context ------------------------------------------------------------ */
int sfb_ctx_create(int device, sfb_ctx **out);
int sfb_ctx_destroy(sfb_ctx *ctx);
const char *sfb_last_error(sfb_ctx *ctx);
int sfb_set_stream(sfb_ctx *ctx, void *cuda_stream);     /* cudaStream_t */
int sfb_get_stats(sfb_ctx *ctx, sfb_stats *out);         /* host out */
int sfb_version(void);
/* Stage timing with CUDA events on the context stream (off by default):
 * after a call, sfb_stage_times returns (stage id, ms) per completed stage:
 * 1 voxelize, 2 unet, 3 head, 4 project, 5 depth sort, 6 runs+binning,
 * 7 composite (in the frame), 8 four more back-to-back compositor launches
 * (the kernel's own duration, free of eager launch gaps; same output),
 * 9 untimed. Synchronises on the recorded events. */
int sfb_set_timing(sfb_ctx *ctx, int on);
/* CUDA-graph replay of sfb_frame (default on): the first call of a shape runs
 * eagerly, the second captures, later calls update parameters and replay. */
int sfb_set_graphs(sfb_ctx *ctx, int on);
/* Capacity (entries) of the fine / super tile-list buffers; 0 (default) sizes
 * them from the previous eager frame's demand. A frame needing more renders
 * every run from the global list instead (identical planes, slower). Tests. */
int sfb_set_entry_capacity(sfb_ctx *ctx, int64_t capacity);
/* How the tcgen05 convs stage their gathered A rows: 0 register prefetch one
 * tap batch ahead (default, fastest measured), 1 TMA tile::gather4 into a
 * shared-memory ring RS batches ahead, 2 per-thread cp.async ring. Results are
 * bitwise identical across modes. */
int sfb_set_conv_staging(sfb_ctx *ctx, int mode);
/* Diagnostics: when set (device buffer of 4 int64 per tile, zeroed by the
 * caller) the compositor accumulates windows, list entries and alpha
 * evaluations per tile. NULL disables. */
int sfb_set_debug_counters(sfb_ctx *ctx, int64_t *dev_counters);
int sfb_stage_times(sfb_ctx *ctx, int32_t *stage_ids, float *ms, int32_t cap, int32_t *n_out);
/* Parity export of the fused frame (sfb_frame / sfb_frame_rgba), for tests:
 * device buffers of `capacity` >= points rows receive the rank -> point order
 * (source, rasterizer.py:105), the runs of identical geometry (start rank,
 * point count, tile rect x0 x1 y0 y1 of _raster_kernels.py:123-130; the
 * first sfb_stats.runs entries), and per UNet level l < levels the level's
 * coordinates (3 capacity) and tap-major kernel map (27 capacity, rows in
 * the level's own order; sparsenet.py:201-207). Frames run eagerly while set;
 * capacity 0 disables. */
int sfb_set_frame_debug(sfb_ctx *ctx, int64_t capacity, int64_t *source, int32_t *run_start,
                        int32_t *run_count, int32_t *run_rect, int32_t levels,
                        int32_t *level_coords, int32_t *level_maps);

/* ---- voxelization (voxelgrid.py:125-168, voxelize_adaptive) ------------- */
/* bbox of (n,3) device positions -> host lo_hi[6] = (lo xyz, hi xyz). The
 * caller forms s = (n / prod(hi-lo)) ** (1/3) in host float64 exactly as
 * voxelgrid.py:133-141 does, so the lattice scale is bit-identical. */
int sfb_bbox(sfb_ctx *ctx, const double *positions, int64_t n, double *lo_hi_host);
/* Enqueue-only bbox: the six order-preserving 64-bit words (lo xyz, hi xyz;
 * u ^ (sign ? ~0 : 1<<63) of the float64 bits) are copied into caller PINNED
 * memory when the stream gets there; the caller synchronises (event) and
 * decodes. Lets an upload pipeline keep the copy engine busy. */
int sfb_bbox_async(sfb_ctx *ctx, const double *positions, int64_t n, uint64_t *ordered_pinned);

/* Density-1 voxelization at scale s. Outputs (capacity n / n+1):
 * coords (M,3) int32 in canonical packed-key order, feats (M,9) float64
 * [centroid/s, mean colour, clipped residual], keys (M,) int64 packed as
 * voxelgrid.py:22-27, point_to_voxel (n,), source_order (n,),
 * source_offsets (M+1,) int32; *m_host receives M. */
int sfb_voxelize(sfb_ctx *ctx, const double *positions, const double *colors, int64_t n,
                 double s, const double *lo_hi_host, int32_t *coords, double *feats,
                 int64_t *keys, int32_t *point_to_voxel, int32_t *source_order,
                 int32_t *source_offsets, int64_t *m_host);

/* ---- kernel maps (sparsenet.py:178-214 lookups, voxelgrid.py:88-94) ------- */
/* Neighbour rows of a canonical grid for a k^3 stride-s conv, (m, k^3) int32,
 * -1 where empty; taps in lexicographic (dz,dy,dx) order. Bit-exact with the
 * reference's searchsorted lookups. */
int sfb_kernel_map(sfb_ctx *ctx, const int32_t *coords, int64_t m, int32_t stride,
                   int32_t kernel, int32_t *map_out);
/* Parent row (-1 = orphan) and child tap (dz*4+dy*2+dx) of each target
 * (sparsenet.py:233-238). parent grid given by canonical coords. */
int sfb_transposed_map(sfb_ctx *ctx, const int32_t *parent_coords, int64_t m_parent,
                       int32_t parent_stride, const int32_t *targets, int64_t m_targets,
                       int32_t *parent_out, int32_t *tap_out);
/* pool_2x2x2 (voxelgrid.py:171-185) on float32 features: parent coords
 * (canonical), means of occupied children in child-row order, child->parent. */
int sfb_pool(sfb_ctx *ctx, const int32_t *coords, const float *feats, int64_t m, int32_t c,
             int32_t stride, int32_t *parent_coords, float *parent_feats,
             int32_t *child_to_parent, int64_t *m_parent_host);

/* pool_2x2x2 on float64 features (the reference API's dtype): same parents
 * and child->parent map, means summed in child-row order as np.add.at. */
int sfb_pool_f64(sfb_ctx *ctx, const int32_t *coords, const double *feats, int64_t m, int32_t c,
                 int32_t stride, int32_t *parent_coords, double *parent_feats,
                 int32_t *child_to_parent, int64_t *m_parent_host);
/* SparseVoxelGrid.lookup (voxelgrid.py:88-94): row of each (nq,3) query in
 * the canonical grid (m,3), -1 where unoccupied; rows (nq,) int64. */
int sfb_lookup(sfb_ctx *ctx, const int32_t *coords, int64_t m, const int32_t *query, int64_t nq,
               int64_t *rows);

/* ---- P2ENet (sparsenet.py:187-287, 310-341) ------------------------------ */
/* Parse a P2EN weight blob (host bytes, sparsenet.py:344-434 layout) and
 * upload the packed per-layer operands; replaces load_weights/NetworkWeights. */
int sfb_net_load(sfb_ctx *ctx, const void *p2en_blob_host, size_t nbytes);
int sfb_net_set_mode(sfb_ctx *ctx, int mode);          /* SFB_NET_* */
/* A standalone conv (kind 0) / transposed_conv (kind 1) layer from host
 * float32 weights (k,k,k,in,out) and bias, addressed as layer -1 below
 * (sparse_conv / transposed_conv_pruned take their own weights,
 * sparsenet.py:187, 217). */
int sfb_layer_set(sfb_ctx *ctx, int kind, int kernel, int cin, int cout, const float *w_host,
                  const float *b_host);
/* Single layers on caller tensors (float32 features); layer = index into the
 * loaded network, or -1 for the standalone layer. */
int sfb_sparse_conv(sfb_ctx *ctx, int layer, const int32_t *coords, const float *feats,
                    int64_t m, int32_t stride, int relu, float *out);
int sfb_transposed_conv(sfb_ctx *ctx, int layer, const int32_t *parent_coords,
                        const float *parent_feats, int64_t m_parent, int32_t parent_stride,
                        const int32_t *targets, int64_t m_targets, int relu, float *out);
/* Full UNet + head on a voxelized cloud: raw (m0,14) per voxel, float32 —
 * float64 when the network mode is SFB_NET_SIMT_F64. */
int sfb_unet_forward(sfb_ctx *ctx, const int32_t *coords, const double *feats9, int64_t m0,
                     void *raw_out);
/* activate_head per row (sparsenet.py:310-341): float64 raw in, float64 out. */
int sfb_activate_head(sfb_ctx *ctx, const double *raw, int64_t m, double voxel_scale,
                      double *delta, double *sigma, double *quat, double *opacity,
                      double *normal);

/* ---- estimate_neural (estimators.py:214-231) ----------------------------- */
/* Cloud -> per-point Splats (float64 SoA, caller buffers of n rows). colors
 * are copied from the input. s as for sfb_voxelize. */
int sfb_estimate_neural(sfb_ctx *ctx, const double *positions, const double *colors,
                        int64_t n, double s, const double *lo_hi_host, double *centers,
                        double *scales, double *quaternions, double *opacities,
                        double *colors_out, double *normals);

/* ---- render (rasterizer.py:152-166, _raster_kernels.py:20-201) ------------ */
/* Tiled front-to-back splatting of any Splats batch. plane_mask selects the
 * planes written in ONE pass (alpha/T do not depend on the attribute):
 * rgb (H,W,3) = sum + T*bg, normal (H,W,3) renormalised, depth (H,W),
 * trans (H,W) clipped to [0,1]; all float32, NULL for planes not requested. */
int sfb_render(sfb_ctx *ctx, const sfb_splats *splats, const sfb_camera *cam,
               const sfb_render_options *opts, int32_t plane_mask, const double *background3,
               float *rgb, float *normal, float *depth, float *trans);

/* project_kernel seam (_raster_kernels.py:20-105): per splat, float64. */
int sfb_project(sfb_ctx *ctx, const sfb_splats *splats, const sfb_camera *cam, double z_near,
                double dilation, double *sx, double *sy, double *depth, double *cov_a,
                double *cov_b, double *cov_c, double *radius, uint8_t *keep);

/* _prepare + bin_tiles seam (rasterizer.py:99-130, _raster_kernels.py:108-143):
 * materialises the reference CSR for parity checks. source (capacity n)
 * rank->splat, offsets (ntx*nty+1), ids (capacity ids_capacity); K and E out.
 * If E > ids_capacity nothing is written to ids (call again with room). */
int sfb_prepare_debug(sfb_ctx *ctx, const sfb_splats *splats, const sfb_camera *cam,
                      int32_t tile_size, int64_t *source, double *radius, int64_t *offsets,
                      int64_t *ids, int64_t ids_capacity, int64_t *k_host, int64_t *e_host);

/* ---- analytic estimators (estimators.py:41-211, _neighbors.py:33-128) ---- */
/* Exact k nearest neighbours of every point among the others: (n,k) squared
 * distances ascending and int64 indices, ties broken by index — bit-identical
 * to the reference's uniform-grid search. k <= 64, n > k. */
int sfb_knn(sfb_ctx *ctx, const double *positions, int64_t n, int32_t k, double *d2_out,
            int64_t *idx_out);
/* sqrt of the first column of a (n,k) kNN distance array (per-point nearest
 * distance; the caller averages it into d-bar). */
int sfb_nn_distance(sfb_ctx *ctx, const double *d2, int64_t n, int32_t k, double *dist_out);
/* estimate_local_pca per point from the kNN indices: covariance of the k
 * neighbours, symeig3x3 frame with the reference's sign rules, scales =
 * max(sigma_mult*sqrt(lambda), 0.1*dbar), quaternion of the frame, normal =
 * smallest-eigenvalue direction flipped away from centroid_host. */
int sfb_local_pca(sfb_ctx *ctx, const double *positions, int64_t n, int32_t k,
                  const int64_t *knn_idx, double sigma_mult, double dbar,
                  const double *centroid_host, double *scales, double *quaternions,
                  double *normals);

/* ---- file formats decoded on the device (pcio.py:210-257, gaussians.py:277-311) */
/* Binary little-endian PLY vertex rows (the file body as read, device bytes)
 * -> PointCloud arrays: positions (n,3) float64, colors (n,3) = uchar/255,
 * normals (n,3) renormalised ((0,0,1) below 1e-12) or NULL. offsets_host: byte
 * offsets of x y z red green blue nx ny nz within a row (-1 = absent). */
int sfb_ply_decode(sfb_ctx *ctx, const uint8_t *body, int64_t n, int32_t stride,
                   const int32_t *offsets_host, double *positions, double *colors,
                   double *normals);
/* SPL1 cache rows ((n,17) little-endian float32, device) <-> float64 Splats. */
int sfb_spl1_decode(sfb_ctx *ctx, const float *rows, int64_t n, double *centers, double *scales,
                    double *quaternions, double *opacities, double *colors, double *normals);
int sfb_spl1_encode(sfb_ctx *ctx, const sfb_splats *splats, float *rows);

/* ---- render_backward (rasterizer.py:229-354, _raster_kernels.py:204-310) -- */
/* Analytic gradients of render(splats, cam, mode) w.r.t. every splat
 * parameter. upstream: dL/d(plane), (H,W,3) float64 device (depth: channel 0
 * used). Outputs (n,3)/(n,4)/(n,) float64 device, zeros for culled splats;
 * d_colors is written for mode rgb, d_normals for mode normal (either may be
 * NULL otherwise). mode: 0 rgb (background composited), 1 normal, 2 depth.
 * tile_size <= 16. */
int sfb_render_backward(sfb_ctx *ctx, const sfb_splats *splats, const sfb_camera *cam,
                        const sfb_render_options *opts, int32_t mode, const double *background3,
                        const double *upstream, double *d_centers, double *d_scales,
                        double *d_quaternions, double *d_opacities, double *d_colors,
                        double *d_normals);

/* ---- render_pose epilogue (service.py:116-136, rasterizer.py:209-226) ------ */
/* RGBA8 output of service.render_pose: mode rgb -> to_rgba(rgb, T); normal ->
 * to_rgba(normal*0.5+0.5, T); relit -> to_rgba(relight(normal, rgb, light,
 * ambient, diffuse), T), the relit rgb and normal planes from ONE compositing
 * pass. Quantisation as to_rgba: clip(rint(v*255), 0, 255), alpha from
 * coverage 1-T; computed from the float64 accumulators. */
enum { SFB_MODE_RGB = 0, SFB_MODE_NORMAL = 1, SFB_MODE_RELIT = 2 };
typedef struct {
    int32_t mode;       /* SFB_MODE_* (service.py MODE_CODES) */
    double light[3];    /* unit light direction (relit) */
    double ambient, diffuse;
} sfb_shading;

/* render_pose on a Splats batch: rgba (H,W,4) uint8, device. */
int sfb_render_rgba(sfb_ctx *ctx, const sfb_splats *splats, const sfb_camera *cam,
                    const sfb_render_options *opts, const sfb_shading *shading,
                    const double *background3, uint8_t *rgba);

/* ---- fused frame: cloud -> P2ENet -> splat, no per-point splats ---------- */
/* The bench hot path: voxelize, UNet, head, then render the per-voxel
 * Gaussians broadcast to their points (colours per point) straight to planes. */
int sfb_frame(sfb_ctx *ctx, const double *positions, const double *colors, int64_t n, double s,
              const double *lo_hi_host, const sfb_camera *cam, const sfb_render_options *opts,
              int32_t plane_mask, const double *background3, float *rgb, float *normal,
              float *depth, float *trans);

/* The fused frame straight to RGBA8 (render_pose of the estimated splats):
 * the streaming path of service.py, 4 bytes per pixel instead of 28. */
int sfb_frame_rgba(sfb_ctx *ctx, const double *positions, const double *colors, int64_t n,
                   double s, const double *lo_hi_host, const sfb_camera *cam,
                   const sfb_render_options *opts, const sfb_shading *shading,
                   const double *background3, uint8_t *rgba);

#ifdef __cplusplus
}
#endif
#endif
