// Shared runtime pieces of libsfb200: context, scratch arena, error plumbing.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/sfb200.h"

namespace sfb {

struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string &m) : std::runtime_error(m), code(c) {}
};

#define SFB_CUDA(expr)                                                                      \
    do {                                                                                    \
        cudaError_t _e = (expr);                                                            \
        if (_e != cudaSuccess)                                                              \
            throw ::sfb::Error(_e == cudaErrorMemoryAllocation ? SFB_ERR_OOM : SFB_ERR_CUDA, \
                               std::string(#expr) + ": " + cudaGetErrorString(_e));         \
    } while (0)

#define SFB_CHECK_LAUNCH() SFB_CUDA(cudaGetLastError())

#define SFB_REQUIRE(cond, msg)                                    \
    do {                                                          \
        if (!(cond)) throw ::sfb::Error(SFB_ERR_ARG, (msg));      \
    } while (0)

// thrown when a frame being captured into a CUDA graph needs more scratch than
// the eager run that preceded it (cudaMalloc is illegal during capture)
struct ArenaGrowth : std::runtime_error {
    ArenaGrowth() : std::runtime_error("scratch arena must grow during graph capture") {}
};

// Grow-only device scratch: a list of chunks; a top-level call resets the
// cursor, allocations bump through existing chunks and only allocate a new
// chunk when none has room (so steady-state frames never call cudaMalloc).
class Arena {
  public:
    ~Arena() {
        for (auto &c : chunks_) cudaFree(c.ptr);
    }
    void reset() {
        cur_ = 0;
        off_ = 0;
    }
    template <class T>
    T *alloc(size_t count) {
        return static_cast<T *>(alloc_bytes(count * sizeof(T)));
    }
    void *alloc_bytes(size_t bytes) {
        bytes = (bytes + 255) & ~size_t(255);
        if (bytes == 0) bytes = 256;
        while (cur_ < chunks_.size()) {
            if (off_ + bytes <= chunks_[cur_].size) {
                void *p = static_cast<char *>(chunks_[cur_].ptr) + off_;
                off_ += bytes;
                return p;
            }
            ++cur_;
            off_ = 0;
        }
        if (no_grow) throw ArenaGrowth();   // capturing: the caller retries eagerly
        size_t sz = bytes < (size_t(64) << 20) ? (size_t(64) << 20) : bytes;
        void *p = nullptr;
        SFB_CUDA(cudaMalloc(&p, sz));
        chunks_.push_back({p, sz});
        cur_ = chunks_.size() - 1;
        off_ = bytes;
        return p;
    }
    size_t reserved() const {
        size_t s = 0;
        for (auto &c : chunks_) s += c.size;
        return s;
    }

    bool no_grow = false;   // set while a frame is captured into a graph

  private:
    struct Chunk {
        void *ptr;
        size_t size;
    };
    std::vector<Chunk> chunks_;
    size_t cur_ = 0, off_ = 0;
};

struct NetLayer {
    int kind;            // 0 conv, 1 transposed_conv, 2 mlp
    int kernel, cin, cout, taps;
    float *w = nullptr;  // device, [taps][cin][cout] float32 (reference order)
    float *b = nullptr;  // device, [cout]
    // tcgen05 operands (split tf32 hi/lo, K-major per tap, padded)
    float *w_tc = nullptr;
    uint16_t *w_bf16 = nullptr;   // single bf16 operands, same canonical layout (fast mode)
    // transposed convs with Cin > 32: the same split operands as two K halves
    // per tap (pseudo-taps 2t, 2t+1), so a CTA stages half the tile
    float *w_tc_k2 = nullptr;
    int cin_pad = 0, cout_pad = 0;
};

struct Net {
    bool loaded = false;
    std::vector<int> enc, dec;
    int head_hidden = 0, levels = 0;
    std::vector<NetLayer> layers;
    std::vector<void *> allocations;
    void release() {
        for (void *p : allocations) cudaFree(p);
        allocations.clear();
        layers.clear();
        loaded = false;
    }
};

struct DevCounts;

// Parity export of the fused frame (sfb_set_frame_debug): caller device
// buffers of `cap` (>= points) rows; frames run eagerly while set
struct FrameDebug {
    int64_t cap = 0;
    int64_t *source = nullptr;                                        // (cap) rank -> point
    int32_t *run_start = nullptr, *run_count = nullptr, *run_rect = nullptr;   // (cap) (cap) (4 cap)
    int32_t levels = 0;
    int32_t *level_coords = nullptr;   // (levels, 3 cap) the UNet's per-level coordinates
    int32_t *level_maps = nullptr;     // (levels, 27, cap) its tap-major kernel maps
};
}  // namespace sfb

struct sfb_frame_graph;

struct sfb_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    sfb::Arena arena;
    sfb::Net net;
    sfb::NetLayer adhoc;  // standalone layer for single-layer calls
    int net_mode = SFB_NET_TC_TF32X3;
    uint64_t net_epoch = 0;
    // CUDA graphs of the fused frame, keyed by shape (api.cu)
    bool use_graphs = true;
    cudaStream_t capture_stream = nullptr;
    cudaEvent_t fork_event = nullptr;
    // side branch of the frame (coordinate structure of the UNet levels runs
    // concurrently with the convolutions): its stream and fork/join events
    cudaStream_t side_stream = nullptr;
    cudaStream_t aux_stream = nullptr;   // the voxel feature sums, beside both
    // events: UNet levels + fork (0..L), then the voxel-feature sums' fork /
    // join and the binning stage's fork / join (the last four)
    static constexpr int kSideEvents = 14;
    static constexpr int kEvFeatsFork = kSideEvents - 4, kEvFeatsJoin = kSideEvents - 3;
    static constexpr int kEvBinFork = kSideEvents - 2, kEvBinJoin = kSideEvents - 1;
    cudaEvent_t side_ev[kSideEvents] = {};
    bool feats_pending = false;   // voxel features still being summed on the side stream
    std::vector<sfb_frame_graph *> graphs;
    int64_t graph_nodes = 0;
    int64_t *debug_counters = nullptr;   // compositor per-tile counters (diagnostics)
    sfb::FrameDebug frame_debug;         // fused-frame parity export (tests)
    int64_t entry_cap_override = 0;      // tests: pyramid entry capacity (0 = automatic)
    // tcgen05 conv A-row staging: 0 register prefetch (default: fastest, A/B in
    // DESIGN.md §4), 1 TMA gather4 ring, 2 cp.async ring (sfb_set_conv_staging)
    int conv_stage = 0;
    sfb::DevCounts *last_counts = nullptr;   // device counts of the last call
    // launch-size hints (host copies of the counts of the last eager frame):
    // every kernel loops over its device count, so hints only size grids
    int64_t hint_m[9] = {}, hint_kept = 0, hint_runs = 0, hint_e = 0;
    int64_t grid_bound(int64_t bound, int64_t hint) const {
        if (hint <= 0) return bound;
        int64_t g = hint + hint / 4 + 1024;
        return g < bound ? g : bound;
    }
    int num_sms = 148;
    // end of the previous call's work (its scratch arena lives on): a call on
    // another stream waits for it first (api.cu guard)
    cudaEvent_t done_event = nullptr;
    cudaStream_t done_stream = nullptr;
    bool done_valid = false;
    std::string last_error;
    sfb_stats stats{};
    // pinned host staging for small D2H reads (sizes, bbox)
    int64_t *pinned = nullptr;
    // optional stage timing: CUDA events recorded on the stream at stage ends
    static constexpr int kMaxMarks = 16;
    bool timing = false;
    cudaEvent_t ev[kMaxMarks] = {};
    int stage_id[kMaxMarks] = {};
    int n_marks = 0;
    void mark(int stage) {
        if (!timing || n_marks >= kMaxMarks) return;
        if (!ev[n_marks]) cudaEventCreate(&ev[n_marks]);
        cudaEventRecord(ev[n_marks], stream);
        stage_id[n_marks++] = stage;
    }
    ~sfb_ctx() {
        net.release();
        for (void *p : {(void *)adhoc.w, (void *)adhoc.b, (void *)adhoc.w_tc, (void *)adhoc.w_bf16})
            if (p) cudaFree(p);
        if (pinned) cudaFreeHost(pinned);
        for (auto &e : ev)
            if (e) cudaEventDestroy(e);
        if (capture_stream) cudaStreamDestroy(capture_stream);
        if (side_stream) cudaStreamDestroy(side_stream);
        if (aux_stream) cudaStreamDestroy(aux_stream);
        for (auto &e : side_ev)
            if (e) cudaEventDestroy(e);
        if (fork_event) cudaEventDestroy(fork_event);
        if (done_event) cudaEventDestroy(done_event);
    }
    // read `count` int64 values back from device (one sync)
    void read_back(const void *dev, size_t bytes) {
        SFB_CUDA(cudaMemcpyAsync(pinned, dev, bytes, cudaMemcpyDeviceToHost, stream));
        SFB_CUDA(cudaStreamSynchronize(stream));
    }
};

namespace sfb {

// stage ids reported by sfb_stage_times
enum Stage { ST_BEGIN = 0, ST_VOXELIZE, ST_UNET, ST_HEAD, ST_PROJECT, ST_SORT, ST_BIN, ST_COMPOSITE,
             ST_COMPOSITE_REPS, ST_BEGIN_REPS };

inline unsigned grid_for(int64_t n, int block, int64_t cap = 1 << 20) {
    int64_t g = (n + block - 1) / block;
    if (g < 1) g = 1;
    if (g > cap) g = cap;
    return static_cast<unsigned>(g);
}

inline int bits_for(uint64_t range_inclusive_max) {
    int b = 0;
    while (b < 64 && (range_inclusive_max >> b) != 0) ++b;
    return b;
}

// Packed voxel key of voxelgrid.py:22-27: ((z+B)<<42)|((y+B)<<21)|(x+B).
__host__ __device__ inline int64_t pack_key(int64_t x, int64_t y, int64_t z) {
    const int64_t B = int64_t(1) << 20;
    return ((z + B) << 42) | ((y + B) << 21) | (x + B);
}
__host__ __device__ inline bool key_in_range(int64_t x, int64_t y, int64_t z) {
    const int64_t L = int64_t(1) << 20;
    return x > -L && x < L && y > -L && y < L && z > -L && z < L;
}
// Python floor division by a positive power of two (every caller divides by
// a lattice stride): an arithmetic shift, not a 64-bit integer division
__host__ __device__ inline int64_t floor_div(int64_t a, int64_t d) {
#ifdef __CUDA_ARCH__
    const int sh = __ffsll(d) - 1;
#else
    const int sh = __builtin_ctzll((unsigned long long)d);
#endif
    return a >> sh;
}

// grid-stride loop over a count that may live in device memory
#define SFB_FOR(i, n)                                                              \
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < (n);    \
         i += (int64_t)gridDim.x * blockDim.x)

// grid for a grid-stride kernel: enough CTAs for `bound` items, capped
inline unsigned dgrid(int64_t bound, int block, int per_sm = 8) {
    int64_t g = (bound + block - 1) / block;
    int64_t cap = 148 * per_sm;
    if (g > cap) g = cap;
    if (g < 1) g = 1;
    return (unsigned)g;
}

// Device-resident sizes of one pipeline call (all data-dependent counts).
struct DevCounts {
    int64_t n;          // points
    int64_t m[9];       // voxels per UNet level (m[0] = M0)
    int64_t kept;       // points surviving the cull
    int64_t runs;       // depth-ordered runs of identical geometry
    int64_t runs1;      // runs + 1
    int64_t ef, es, g;  // fine / super / global pyramid entries
    int64_t ef_req, es_req, overflow;   // entries the runs asked for; 1 = over capacity
    int64_t scratch[4];
    // kept depths' range as atomicMax words (zero = identity): zr[0] = ~min
    // bits, zr[1] = max bits (depth > 0, so the bits order like the values)
    unsigned long long zr[2];
};

struct Cam {
    double r[9], t[3], fx, fy, cx, cy;
    int64_t w, h;
};
Cam to_cam(const sfb_camera &c);

// Per-call parameters that change frame to frame (lattice scale, key layout,
// camera, background). Written to device memory by the first kernel of a
// call, so a captured CUDA graph replays with new values after a single
// kernel-node parameter update.
struct FrameParams {
    double s, inv_s;
    int64_t lo[3], hi[3];   // lattice range of the level-0 voxel coordinates
    int32_t bits[3];
    int32_t total;
    Cam cam;
    double bg[3];
    // render_pose epilogue (RGBA8 output): mode, light, ambient, diffuse
    int32_t shade_mode;
    double light[3], ambient, diffuse;
};

// devprims.cu
void dscan(sfb_ctx *ctx, const int32_t *in, int32_t *out, const int64_t *d_n, int64_t n_fixed,
           int64_t *total_out, bool inclusive);
void dscan3(sfb_ctx *ctx, const int32_t *in0, const int32_t *in1, const int32_t *in2, int32_t *out0,
            int32_t *out1, int32_t *out2, const int64_t *d_n, int64_t n_fixed, int64_t *tot0,
            int64_t *tot1, int64_t *tot2);
template <class K>
int dsort_pairs(sfb_ctx *ctx, K *k0, uint32_t *v0, K *k1, uint32_t *v1, const int64_t *d_n,
                int64_t n_fixed, int bits);
void write_params(sfb_ctx *ctx, const FrameParams &host, FrameParams *dev);
// cudaFuncAttributeMaxDynamicSharedMemorySize for `func` on the current
// device, set once per (device, kernel) under a lock (kernel attributes are
// per device; several host threads may launch the first frame concurrently)
void set_max_dyn_smem(const void *func, int bytes);

// ---- cross-file launchers (defined in the .cu files) ----------------------

// hashmap.cu
struct HashTable {
    unsigned long long *keys = nullptr;
    int32_t *vals = nullptr;
    uint32_t *mask = nullptr;  // device: capacity - 1, sized from the device count
};
// counts: device pointer d_m (or nullptr -> m_bound is the exact count)
HashTable hash_build(sfb_ctx *ctx, const int32_t *coords, const int64_t *d_m, int64_t m_bound,
                     int64_t m_grid = -1);
void kernel_map_build(sfb_ctx *ctx, const HashTable &h, const int32_t *coords, const int64_t *d_m,
                      int64_t m_bound, int stride, int kernel, int32_t *map_tap_major,
                      int64_t m_grid = -1);
void transposed_lookup(sfb_ctx *ctx, const HashTable &h, int parent_stride,
                       const int32_t *targets, const int64_t *d_m, int64_t m_bound,
                       int32_t *parent_out, int32_t *tap_out);
// pooled parents in canonical order; parent count -> *d_mp (device)
void pool_build(sfb_ctx *ctx, const int32_t *coords, const int64_t *d_m, int64_t m_bound,
                int stride, const FrameParams &host, const FrameParams *P, const float *feats,
                int c, int ld_in, int32_t *parent_coords, float *parent_feats, int ld_out,
                int32_t *child_to_parent, int64_t *d_mp);
void pool_build(sfb_ctx *ctx, const int32_t *coords, const int64_t *d_m, int64_t m_bound,
                int stride, const FrameParams &host, const FrameParams *P, const double *feats,
                int c, int ld_in, int32_t *parent_coords, double *parent_feats, int ld_out,
                int32_t *child_to_parent, int64_t *d_mp);
void lookup_run(sfb_ctx *ctx, const int32_t *coords, int64_t m, const int32_t *query, int64_t nq,
                int64_t *rows);
void coords_layout(sfb_ctx *ctx, const int32_t *coords, int64_t m, FrameParams &P);
// children of a level grouped by their tap under the parent, each bucket
// padded to whole 128-row tiles (the tap-bucketed transposed conv)
struct TapBuckets {
    int32_t *perm;       // padded row -> child row (-1 pad)
    int32_t *src;        // padded row -> parent row (-1 pad)
    int32_t *off;        // 9 padded bucket offsets (device)
    int64_t *d_rows;     // padded row count (device)
    int64_t rows_bound, rows_grid;
};
// fused UNet pooling, split: coordinate structure (side stream) + means
struct PoolStructure {
    TapBuckets buckets;
    HashTable table;        // parent key -> parent row (the coarse level's hash)
    int32_t *c2p, *tap;     // per child: parent row, tap under the parent
    int32_t *tmap;          // (8, m) tap-major map of the transposed conv
    int32_t *nkids, *kids;  // per parent: child count, up to 8 child rows
};
PoolStructure pool_structure(sfb_ctx *ctx, const int32_t *coords, const int64_t *d_m,
                             int64_t m_bound, int64_t m_grid, int stride, int32_t *parent_coords,
                             int64_t *d_mp);
void pool_means(sfb_ctx *ctx, const PoolStructure &P, const int64_t *d_mp, int64_t mp_grid,
                const float *feats, int c, int ld_in, float *parent_feats, int ld_out);
// sort-free pooling for the fused UNet: parents in first-child order
void pool_fast(sfb_ctx *ctx, const int32_t *coords, const int64_t *d_m, int64_t m_bound,
               int64_t m_grid, int stride, const float *feats, int c, int ld_in,
               int32_t *parent_coords, float *parent_feats, int ld_out, int32_t *child_to_parent,
               int64_t *d_mp);

// voxelize.cu
struct VoxelOut {
    int32_t *coords;
    double *feats;
    int64_t *keys;
    int32_t *p2v, *order, *offsets;
    float *feats32 = nullptr;   // optional: the (M, 9) features also as float32 (UNet input)
};
void bbox_run(sfb_ctx *ctx, const double *pos, int64_t n, double *lo_hi_host);
void bbox_async_run(sfb_ctx *ctx, const double *pos, int64_t n, uint64_t *ordered_host);
void voxel_layout(const double *lo_hi, double s, FrameParams &P);
// voxel count lands in C->m[0] (device)
// feats_on_side: the per-voxel feature sums go to the aux stream (they only
// feed the first convolution, so the level-0 hash and kernel map overlap
// them); ctx->feats_pending tells unet_run to join before it
void voxelize_run(sfb_ctx *ctx, const double *pos, const double *col, int64_t n,
                  const FrameParams &host, const FrameParams *P, VoxelOut &out, DevCounts *C,
                  bool feats_on_side = false);

// net.cu
void net_load(sfb_ctx *ctx, const void *blob, size_t n);
// per-voxel raw head (M0 x 14) float32 into `raw`; M0 = C->m[0] (device), bound m_bound
// Host bounds on the voxel count of UNet level l (stride 2^l): the cloud's
// point count, and the number of stride-2^l lattice cells the level-0
// coordinate range [lo, hi] touches, rounded up to 3 significant bits (so a
// CUDA graph keyed on them survives small bbox changes). Buffers of level l
// are sized by it instead of by the point count.
void unet_level_bounds(const FrameParams &host, int64_t n, int levels, int64_t *bound);
// raw: float32, or float64 in SFB_NET_SIMT_F64 mode
// feats32: the level-0 features already as float32 (voxelization writes them), or null
void unet_run(sfb_ctx *ctx, const int32_t *coords, const double *feats9, int64_t m_bound,
              const FrameParams &host, const FrameParams *P, DevCounts *C, void *raw,
              const float *feats32 = nullptr);
void activate_run(sfb_ctx *ctx, const double *raw, int64_t m, double scale, double *delta,
                  double *sigma, double *quat, double *opac, double *normal);
void conv_layer(sfb_ctx *ctx, const NetLayer &L, const float *in, int ld_in, const int32_t *nbr,
                int64_t nbr_ld, const int64_t *d_m, int64_t m_bound, int relu, float *out,
                int ld_out, int64_t m_grid = -1, int csplit = -1);
void tconv_layer(sfb_ctx *ctx, const NetLayer &L, const float *in, int ld_in,
                 const int32_t *parent, const int32_t *tap, const int64_t *d_m, int64_t m_bound,
                 int relu, float *out, int ld_out, int64_t m_grid = -1,
                 const int32_t *tmap = nullptr, const struct TapBuckets *tb = nullptr,
                 int csplit = -1);
void layer_set(sfb_ctx *ctx, int kind, int kernel, int cin, int cout, const float *w_host,
               const float *b_host);
// per-voxel Gaussians for the fused frame: centres, sigma, quat, opacity, normal
void head_to_voxel_splats(sfb_ctx *ctx, const void *raw, const int32_t *coords,
                          const double *feats9, const int64_t *d_m, int64_t m_bound,
                          const FrameParams *P, double *centers, double *sigma, double *quat,
                          double *opac, double *normal);

// knn.cu
void knn_run(sfb_ctx *ctx, const double *pos, int64_t n, int k, double *out_d2, int64_t *out_idx);
void local_pca_run(sfb_ctx *ctx, const double *pos, int64_t n, int k, double sigma_mult,
                   const int64_t *idx, double dbar, const double *mean_c, double *scales,
                   double *quats, double *normals);
void nn_dist_run(sfb_ctx *ctx, const double *d2, int64_t n, int k, double *dist);

// formats.cu
void ply_decode_run(sfb_ctx *ctx, const uint8_t *body, int64_t n, int32_t stride,
                    const int32_t *offsets, double *pos, double *col, double *nrm);
void spl1_decode_run(sfb_ctx *ctx, const float *rows, int64_t n, double *c, double *s, double *q,
                     double *o, double *col, double *nrm);
void spl1_encode_run(sfb_ctx *ctx, const sfb_splats &sp, float *rows);

// render.cu
struct RenderInputs {
    // geometry, either per splat (n rows) or per voxel (geometry rows) with a
    // point->geometry map; attributes: colours per point, normals per geometry
    const double *centers, *scales, *quats, *opac;
    int64_t n_geom;                 // host bound on geometry rows
    const int64_t *d_n_geom;        // device count of geometry rows (nullptr: n_geom exact)
    const int32_t *point_to_geom;   // nullptr: identity (geometry per point)
    // CSR of the points of each geometry row in increasing index order
    // (voxelgrid.py:165-168 source_order/offsets); enables the voxel-level order
    const int32_t *geom_offsets, *geom_order;
    const double *colors, *normals;
    int64_t n_points;               // exact, host
};
void render_run(sfb_ctx *ctx, const RenderInputs &in, const FrameParams *FP, int64_t width,
                int64_t height, const sfb_render_options &opts, int plane_mask, DevCounts *C,
                float *rgb, float *normal, float *depth, float *trans, uint8_t *rgba = nullptr);
void project_run(sfb_ctx *ctx, const double *centers, const double *quats, const double *scales,
                 const int64_t *d_n, int64_t n_bound, const FrameParams *FP, double z_near,
                 double dilation, double *sx, double *sy, double *depth, double *ca, double *cb,
                 double *cc, double *radius, uint8_t *keep, unsigned long long *zr = nullptr);
void render_backward_run(sfb_ctx *ctx, const RenderInputs &in, const FrameParams *FP, int64_t width,
                         int64_t height, const sfb_render_options &opts, int mode, DevCounts *C,
                         const double *upstream, double *d_centers, double *d_scales,
                         double *d_quats, double *d_opac, double *d_colors, double *d_normals);
void prepare_debug_run(sfb_ctx *ctx, const RenderInputs &in, const FrameParams *FP, int64_t width,
                       int64_t height, int tile, DevCounts *C, int64_t *source, double *radius,
                       int64_t *offsets, int64_t *ids, int64_t cap, int64_t *k_host,
                       int64_t *e_host);

}  // namespace sfb
