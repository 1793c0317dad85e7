// On-device decoding of the reference's file formats:
// binary little-endian PLY vertex rows (pcio.py:210-257: x y z float32,
// red green blue uchar, optional nx ny nz float32) and the SPL1 splat cache
// (gaussians.py:277-311: 17 little-endian float32 per splat). The host only
// reads the file and parses the header; the body crosses PCIe as the file's
// own bytes (15 B per PLY vertex instead of the 48 B of float64 PointCloud
// arrays) and is widened to float64 here.
#include "common.cuh"

namespace sfb {

struct PlyLayout {
    int32_t stride;
    int32_t off[9];   // x y z red green blue nx ny nz (byte offsets; -1 absent)
};

__device__ __forceinline__ float ld_f32(const uint8_t *p) {
    uint32_t u = (uint32_t)p[0] | ((uint32_t)p[1] << 8) | ((uint32_t)p[2] << 16) | ((uint32_t)p[3] << 24);
    return __uint_as_float(u);
}

// colors come back divided by 255; normals renormalised, (0,0,1) where the
// file normal has norm < 1e-12 (pcio.py:242-254)
__global__ void k_ply_decode(const uint8_t *__restrict__ body, int64_t n, PlyLayout L,
                             double *__restrict__ pos, double *__restrict__ col,
                             double *__restrict__ nrm) {
    SFB_FOR(i, n) {
        const uint8_t *row = body + i * (int64_t)L.stride;
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            pos[3 * i + a] = (double)ld_f32(row + L.off[a]);
            col[3 * i + a] = (double)row[L.off[3 + a]] / 255.0;
        }
        if (nrm) {
            const double x = ld_f32(row + L.off[6]), y = ld_f32(row + L.off[7]), z = ld_f32(row + L.off[8]);
            const double nn = sqrt(x * x + y * y + z * z);
            const bool fb = nn < 1e-12;
            const double d = fb ? 1.0 : nn;
            nrm[3 * i + 0] = fb ? 0.0 : x / d;
            nrm[3 * i + 1] = fb ? 0.0 : y / d;
            nrm[3 * i + 2] = fb ? 1.0 : z / d;
        }
    }
}

// SPL1 rows <-> float64 SoA splats (centre 3, scales 3, quaternion 4,
// opacity, colour 3, normal 3)
__global__ void k_spl1_decode(const float *__restrict__ rows, int64_t n, double *__restrict__ c,
                              double *__restrict__ s, double *__restrict__ q, double *__restrict__ o,
                              double *__restrict__ col, double *__restrict__ nrm) {
    SFB_FOR(i, n) {
        const float *r = rows + 17 * i;
        for (int a = 0; a < 3; ++a) {
            c[3 * i + a] = r[a];
            s[3 * i + a] = r[3 + a];
            col[3 * i + a] = r[11 + a];
            nrm[3 * i + a] = r[14 + a];
        }
        for (int a = 0; a < 4; ++a) q[4 * i + a] = r[6 + a];
        o[i] = r[10];
    }
}

__global__ void k_spl1_encode(int64_t n, const double *__restrict__ c, const double *__restrict__ s,
                              const double *__restrict__ q, const double *__restrict__ o,
                              const double *__restrict__ col, const double *__restrict__ nrm,
                              float *__restrict__ rows) {
    SFB_FOR(i, n) {
        float *r = rows + 17 * i;
        for (int a = 0; a < 3; ++a) {
            r[a] = __double2float_rn(c[3 * i + a]);
            r[3 + a] = __double2float_rn(s[3 * i + a]);
            r[11 + a] = __double2float_rn(col[3 * i + a]);
            r[14 + a] = __double2float_rn(nrm[3 * i + a]);
        }
        for (int a = 0; a < 4; ++a) r[6 + a] = __double2float_rn(q[4 * i + a]);
        r[10] = __double2float_rn(o[i]);
    }
}

void ply_decode_run(sfb_ctx *ctx, const uint8_t *body, int64_t n, int32_t stride,
                    const int32_t *offsets, double *pos, double *col, double *nrm) {
    SFB_REQUIRE(n >= 0 && stride > 0, "bad PLY body layout");
    PlyLayout L;
    L.stride = stride;
    for (int k = 0; k < 9; ++k) L.off[k] = offsets[k];
    for (int k = 0; k < 6; ++k) SFB_REQUIRE(L.off[k] >= 0, "PLY rows need x y z red green blue");
    for (int k = 0; k < 3; ++k) SFB_REQUIRE(L.off[k] + 4 <= stride && L.off[3 + k] < stride, "PLY offset past row");
    if (nrm) for (int k = 6; k < 9; ++k) SFB_REQUIRE(L.off[k] >= 0 && L.off[k] + 4 <= stride, "PLY normals missing");
    if (n == 0) return;
    k_ply_decode<<<dgrid(n, 256), 256, 0, ctx->stream>>>(body, n, L, pos, col, nrm);
    SFB_CHECK_LAUNCH();
}

void spl1_decode_run(sfb_ctx *ctx, const float *rows, int64_t n, double *c, double *s, double *q,
                     double *o, double *col, double *nrm) {
    if (n == 0) return;
    k_spl1_decode<<<dgrid(n, 256), 256, 0, ctx->stream>>>(rows, n, c, s, q, o, col, nrm);
    SFB_CHECK_LAUNCH();
}

void spl1_encode_run(sfb_ctx *ctx, const sfb_splats &sp, float *rows) {
    if (sp.n == 0) return;
    k_spl1_encode<<<dgrid(sp.n, 256), 256, 0, ctx->stream>>>(sp.n, sp.centers, sp.scales, sp.quaternions,
                                                             sp.opacities, sp.colors, sp.normals, rows);
    SFB_CHECK_LAUNCH();
}

}  // namespace sfb
