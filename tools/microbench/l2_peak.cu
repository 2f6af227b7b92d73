// Microbenchmark (measurement tool, not product code): the L2 (LTS) roofline denominators the
// L2-bound kernels are reported against (config 2's working set and the CSR pattern
// kernel's x windows live in L2; Schur is bound by random L2 sectors).
//
//   A  HBM stream      : LDG.128 (__ldcs) over a 2 GiB buffer                  -> GB/s from DRAM
//   B  L2 coalesced    : LDG.128 over a 32 MiB L2-resident buffer, many passes  -> GB/s from L2
//   C  L2 bulk (TMA)   : cp.async.bulk 16 KiB chunks of the same buffer into smem, 4 in flight
//   D  L2 random 8 B   : one 8 B gather per thread at hashed addresses in the buffer
//                        -> useful GB/s and 32 B sectors/s (each gather costs a sector)
//   E  L2 copy         : read + write of two 16 MiB L2-resident halves (config-2-like stream)
//
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/l2_peak tools/microbench/l2_peak.cu
// /tmp/l2_peak  -> one JSON line (CUDA events, best of 5 after warm-up)
#include <cuda_runtime.h>
#include <stdint.h>
#include <cstdio>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("{\"error\": \"%s line %d\"}\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__global__ void k_stream(const double2 *__restrict__ a, size_t n2, double *sink) {
    double s = 0.0;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n2; i += (size_t)gridDim.x * blockDim.x) {
        const double2 v = __ldcs(a + i);
        s += v.x + v.y;
    }
    if (s == 12345.678) *sink = s;
}

__global__ void k_l2read(const double2 *__restrict__ a, size_t n2, int passes, double *sink) {
    double s = 0.0;
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    for (int p = 0; p < passes; ++p) {
        // each pass starts at a block-dependent offset so that CTAs do not march in lockstep
        const size_t off = ((size_t)blockIdx.x * 7919 + (size_t)p * 104729) % n2;
        for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n2; i += stride) {
            size_t j = i + off;
            if (j >= n2) j -= n2;
            const double2 v = __ldcg(a + j);
            s += v.x + v.y;
        }
    }
    if (s == 12345.678) *sink = s;
}

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void k_l2bulk(const double *__restrict__ a, size_t nchunks, int passes, double *sink) {
    constexpr int CH = 16384, NB = 4;  // bytes per chunk, chunks in flight per CTA
    extern __shared__ __align__(16) unsigned char sm[];
    __shared__ uint64_t bar[NB];
    if (threadIdx.x == 0) {
        for (int b = 0; b < NB; ++b)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[b])));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    double s = 0.0;
    const size_t total = nchunks * (size_t)passes;
    uint32_t phase[NB] = {0, 0, 0, 0};
    size_t it = 0;
    // every CTA walks chunk indices blockIdx.x, +gridDim.x, ... over `passes` passes
    auto issue = [&](size_t k, int b) {
        const size_t c = (k * gridDim.x + blockIdx.x) % nchunks;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar[b])), "r"(CH));
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         smem_u32(sm + b * CH)), "l"(a + c * (CH / 8)), "r"(CH), "r"(smem_u32(&bar[b]))
                     : "memory");
    };
    const size_t mine = total / gridDim.x;
    if (threadIdx.x == 0)
        for (int b = 0; b < NB && (size_t)b < mine; ++b) issue(b, b);
    for (it = 0; it < mine; ++it) {
        const int b = it % NB;
        asm volatile("{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n}" ::"r"(
                         smem_u32(&bar[b])), "r"(phase[b]) : "memory");
        phase[b] ^= 1;
        s += reinterpret_cast<const double *>(sm + b * CH)[threadIdx.x];
        __syncthreads();  // everyone read the chunk before it is overwritten
        if (threadIdx.x == 0 && it + NB < mine) issue(it + NB, b);
    }
    if (s == 12345.678) *sink = s;
}

__global__ void k_l2rand(const double *__restrict__ a, size_t n, size_t nread, double *sink) {
    double s = 0.0;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < nread; i += (size_t)gridDim.x * blockDim.x) {
        uint64_t h = i * 0x9E3779B97F4A7C15ull;
        h ^= h >> 29;
        s += __ldcg(a + (h % n));
    }
    if (s == 12345.678) *sink = s;
}

__global__ void k_l2copy(const double2 *__restrict__ a, double2 *__restrict__ b, size_t n2, int passes) {
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    for (int p = 0; p < passes; ++p)
        for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n2; i += stride) {
            const double2 v = __ldcg(a + i);
            b[i] = make_double2(v.x + 1.0, v.y);
        }
}

template <class F>
float best_ms(F f, int reps = 5) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    f();
    cudaDeviceSynchronize();
    float best = 1e30f;
    for (int r = 0; r < reps; ++r) {
        cudaEventRecord(e0);
        f();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    return best;
}

int main() {
    int sms = 0, clk = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const size_t big = (size_t)2 << 30, l2buf = (size_t)32 << 20;
    double *hb, *lb, *sink;
    CK(cudaMalloc(&hb, big));
    CK(cudaMalloc(&lb, l2buf * 2));
    CK(cudaMalloc(&sink, 8));
    CK(cudaMemset(hb, 0, big));
    CK(cudaMemset(lb, 0, l2buf * 2));
    const int G = sms * 8, T = 256;
    const float ta = best_ms([&] { k_stream<<<G, T>>>((const double2 *)hb, big / 16, sink); });
    const int passes = 40;
    const float tb = best_ms([&] { k_l2read<<<G, T>>>((const double2 *)lb, l2buf / 16, passes, sink); });
    CK(cudaFuncSetAttribute(k_l2bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 16384));
    const int Gc = sms * 3;
    const size_t nch = l2buf / 16384;
    const float tc = best_ms([&] { k_l2bulk<<<Gc, T, 4 * 16384>>>(lb, nch, passes, sink); });
    const size_t nread = (size_t)256 << 20;
    const float td = best_ms([&] { k_l2rand<<<G, T>>>(lb, l2buf / 8, nread, sink); });
    const float te = best_ms([&] { k_l2copy<<<G, T>>>((const double2 *)lb, (double2 *)(lb + l2buf / 8), l2buf / 32, passes); });
    CK(cudaGetLastError());
    const double gb_a = big / (ta * 1e-3) / 1e9;
    const double gb_b = (double)l2buf * passes / (tb * 1e-3) / 1e9;
    const double bytes_c = (double)(nch * passes / Gc) * Gc * 16384;
    const double gb_c = bytes_c / (tc * 1e-3) / 1e9;
    const double useful_d = (double)nread * 8 / (td * 1e-3) / 1e9, sectors_d = (double)nread / (td * 1e-3);
    const double gb_e = (double)l2buf * passes / (te * 1e-3) / 1e9;  // read 16 MiB + write 16 MiB per pass
    printf("{\"sms\": %d, \"clock_khz\": %d, \"hbm_stream_read_gbs\": %.1f, \"l2_ldg128_read_gbs\": %.1f, "
           "\"l2_bulk_tma_read_gbs\": %.1f, \"l2_random8B_useful_gbs\": %.1f, \"l2_random8B_sectors_per_s\": %.4g, "
           "\"l2_random8B_sector_gbs\": %.1f, \"l2_copy_rw_gbs\": %.1f, \"l2_buffer_mib\": 32}\n",
           sms, clk, gb_a, gb_b, gb_c, useful_d, sectors_d, sectors_d * 32 / 1e9, gb_e);
    return 0;
}
