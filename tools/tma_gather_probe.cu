// Probe of the sm_100 TMA row gather (cp.async.bulk.tensor.2d.tile::gather4)
// on a feature matrix F[rows][cols] (float32): which bytes land where in
// shared memory for a given box / swizzle. Diagnostic tool, not product code.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -o tools/_tma_probe tools/tma_gather_probe.cu
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

__global__ void k_probe(const __grid_constant__ CUtensorMap tm, int col, int r0, int r1, int r2, int r3,
                        float *out, int nfloats) {
    __shared__ __align__(1024) float sm[2048];
    __shared__ __align__(8) unsigned long long bar;
    for (int i = threadIdx.x; i < 2048; i += blockDim.x) sm[i] = -1.f;
    __syncthreads();
    const unsigned sbar = (unsigned)__cvta_generic_to_shared(&bar);
    const unsigned sdst = (unsigned)__cvta_generic_to_shared(sm);
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sbar));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sbar),
                     "r"(nfloats * 4)
                     : "memory");
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes "
            "[%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(sdst),
            "l"(&tm), "r"(col), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(sbar)
            : "memory");
        unsigned done = 0;
        while (!done) {
            asm volatile(
                "{\n\t.reg .pred P;\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%1], 0;\n\t"
                "selp.u32 %0, 1, 0, P;\n\t}"
                : "=r"(done)
                : "r"(sbar)
                : "memory");
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < 2048; i += blockDim.x) out[i] = sm[i];
}

int main() {
    const int rows = 1000, cols = 64;
    std::vector<float> h(rows * cols);
    for (int r = 0; r < rows; ++r)
        for (int c = 0; c < cols; ++c) h[r * cols + c] = r * 100.f + c;
    float *d, *o;
    cudaMalloc(&d, h.size() * 4);
    cudaMalloc(&o, 2048 * 4);
    cudaMemcpy(d, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
    PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void **)&enc, cudaEnableDefault, &q);
    if (!enc) {
        printf("no cuTensorMapEncodeTiled\n");
        return 1;
    }
    struct Case {
        int box_inner, box_outer;
        CUtensorMapSwizzle sw;
        const char *name;
    } cases[] = {{4, 1, CU_TENSOR_MAP_SWIZZLE_NONE, "box 4x1 none"},
                 {16, 1, CU_TENSOR_MAP_SWIZZLE_NONE, "box 16x1 none"},
                 {16, 1, CU_TENSOR_MAP_SWIZZLE_64B, "box 16x1 sw64"},
                 {32, 1, CU_TENSOR_MAP_SWIZZLE_128B, "box 32x1 sw128"},
                 {8, 1, CU_TENSOR_MAP_SWIZZLE_32B, "box 8x1 sw32"},
                 {16, 4, CU_TENSOR_MAP_SWIZZLE_NONE, "box 16x4 none"}};
    for (auto &cs : cases) {
        CUtensorMap tm;
        cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
        cuuint64_t strides[1] = {(cuuint64_t)cols * 4};
        cuuint32_t box[2] = {(cuuint32_t)cs.box_inner, (cuuint32_t)cs.box_outer};
        cuuint32_t es[2] = {1, 1};
        CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, d, dims, strides, box, es,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, cs.sw, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        printf("== %s: encode rc=%d\n", cs.name, (int)r);
        if (r) continue;
        const int nf = 4 * cs.box_inner;
        k_probe<<<1, 128>>>(tm, 4, 7, 3, 500, 999, o, nf);
        cudaError_t e = cudaDeviceSynchronize();
        printf("   kernel: %s\n", cudaGetErrorString(e));
        if (e) return 2;
        std::vector<float> g(2048);
        cudaMemcpy(g.data(), o, 2048 * 4, cudaMemcpyDeviceToHost);
        for (int i = 0; i < nf + 8 && i < 2048; ++i) {
            printf("%8.0f%s", g[i], (i % cs.box_inner == cs.box_inner - 1) ? "\n" : " ");
        }
        printf("\n");
    }
    return 0;
}
