// Probe (development tool): 3D cp.async.bulk.tensor load of an fp64 box with negative/OOB
// coordinates into shared memory, checked against the host.  Variants: argv[1] selects
//   0: plain, 1: + prefetch.tensormap, 2: box wider than the tensor, 3: descriptor in global memory
// argv[2] dtype (0 FLOAT64, 1 UINT64), argv[3] L2 promotion (0 none, 1 128B), argv[4] coords
// (0 negative, 1 non-negative)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_probe tma_probe.cu
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <cstdio>
#include <cstdlib>
#include <vector>

__device__ __forceinline__ uint32_t su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int MODE>
__global__ void k(const __grid_constant__ CUtensorMap m, const CUtensorMap *gm, int bx, int by, int c0, int c1, int c2,
                  double *out) {
    extern __shared__ __align__(128) double sm[];
    __shared__ uint64_t bar;
    const void *desc = MODE == 3 ? (const void *)gm : (const void *)&m;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
        if (MODE == 1) asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(desc)) : "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar)), "r"(bx * by * 8));
        asm volatile(
            "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
                su32(sm)),
            "l"(reinterpret_cast<uint64_t>(desc)), "r"(c0), "r"(c1), "r"(c2), "r"(su32(&bar))
            : "memory");
    }
    asm volatile("{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W_%=;\n}" ::"r"(
                     su32(&bar)) : "memory");
    for (int i = threadIdx.x; i < bx * by; i += blockDim.x) out[i] = sm[i];
}

int main(int argc, char **argv) {
    const int mode = argc > 1 ? atoi(argv[1]) : 0;
    const int nx = 24, ny = 24, nz = 24;
    const int bx = mode == 2 ? 34 : 18, by = mode == 2 ? 34 : 10;
    std::vector<double> h((size_t)nx * ny * nz);
    for (size_t i = 0; i < h.size(); ++i) h[i] = (double)i + 1;
    double *d, *o;
    cudaMalloc(&d, h.size() * 8);
    cudaMalloc(&o, 34 * 34 * 8);
    cudaMemcpy(d, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
    void *fp = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
    auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fp);
    CUtensorMap m;
    cuuint64_t dims[3] = {(cuuint64_t)nx, (cuuint64_t)ny, (cuuint64_t)nz};
    cuuint64_t str[2] = {(cuuint64_t)nx * 8, (cuuint64_t)nx * ny * 8};
    cuuint32_t box[3] = {(cuuint32_t)bx, (cuuint32_t)by, 1}, es[3] = {1, 1, 1};
    const int dt = argc > 2 ? atoi(argv[2]) : 0, l2p = argc > 3 ? atoi(argv[3]) : 1, nonneg = argc > 4 ? atoi(argv[4]) : 0;
    CUresult r = enc(&m, dt ? CU_TENSOR_MAP_DATA_TYPE_UINT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, d, dims, str, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                     l2p ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B : CU_TENSOR_MAP_L2_PROMOTION_NONE,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    CUtensorMap *gm;
    cudaMalloc(&gm, sizeof(CUtensorMap));
    cudaMemcpy(gm, &m, sizeof(m), cudaMemcpyHostToDevice);
    // argv[4]: 0 -> (-1, -1), 1 -> (2, 3), 2 -> (1, 3) odd inner start, 3 -> (-2, -1), 4 -> (2, -1),
    //         5 -> (20, 20) far side out of bounds
    const int cs[6][2] = {{-1, -1}, {2, 3}, {1, 3}, {-2, -1}, {2, -1}, {20, 20}};
    const int c0 = cs[nonneg][0], c1 = cs[nonneg][1], c2 = 3;
    if (mode == 0) k<0><<<1, 128, 34 * 34 * 8>>>(m, gm, bx, by, c0, c1, c2, o);
    if (mode == 1) k<1><<<1, 128, 34 * 34 * 8>>>(m, gm, bx, by, c0, c1, c2, o);
    if (mode == 2) k<0><<<1, 128, 34 * 34 * 8>>>(m, gm, bx, by, c0, c1, c2, o);
    if (mode == 3) k<3><<<1, 128, 34 * 34 * 8>>>(m, gm, bx, by, c0, c1, c2, o);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<double> got((size_t)bx * by);
    cudaMemcpy(got.data(), o, got.size() * 8, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int y = 0; y < by; ++y)
        for (int x = 0; x < bx; ++x) {
            const int gx = c0 + x, gy = c1 + y;
            const double want = (gx >= 0 && gx < nx && gy >= 0 && gy < ny) ? h[gx + (size_t)nx * gy + (size_t)nx * ny * c2] : 0.0;
            bad += got[x + (size_t)bx * y] != want;
        }
    printf("{\"args\": \"%d %d %d %d\", \"encode\": %d, \"kernel\": \"%s\", \"bad\": %d}\n", mode, dt, l2p, nonneg, (int)r, cudaGetErrorString(e), bad);
    return 0;
}
