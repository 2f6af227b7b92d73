// vec_kernels.cu -- vector kernels shared by the drivers: deterministic reductions of
// per-block partials, scaled copies (degree 0: z = r / theta_bar, Alg. 2
// step 2), the stand-alone recurrence epilogue for callback operators, permutations and
// a counter-hash vector generator.
#include "device_util.cuh"
#include "npc_internal.cuh"

namespace npc {

static constexpr int VT = 256;  // threads per block of the vector kernels

npc_status allow_max_dynamic_smem_ptr(const void *kern) {
    static std::mutex mu;
    static std::vector<const void *> done;
    std::lock_guard<std::mutex> lk(mu);
    for (const void *k : done)
        if (k == kern) return NPC_SUCCESS;
    int dev = 0, optin = 0;
    cudaFuncAttributes fa{};
    // may run while a PCG iteration is being stream-captured (a kernel variant's first launch):
    // these are not stream operations, so let this thread make them in relaxed capture mode
    cudaStreamCaptureMode mode = cudaStreamCaptureModeRelaxed;
    cudaThreadExchangeStreamCaptureMode(&mode);
    cudaError_t e = cudaGetDevice(&dev);
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    if (e == cudaSuccess) e = cudaFuncGetAttributes(&fa, kern);
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, optin - (int)fa.sharedSizeBytes);
    cudaThreadExchangeStreamCaptureMode(&mode);
    NPC_CUDA_TRY(e);
    done.push_back(kern);
    return NPC_SUCCESS;
}

int vec_grid(int n) {
    // 4 elements per thread per pass; at most 8 blocks/SM * 148 SMs; fixed for a given n so
    // the number of partials (and the reduction order) never changes between calls.
    int g = ceil_div((long long)n, (long long)VT * 4);
    if (g > 148 * 8) g = 148 * 8;
    if (g < 1) g = 1;
    return g;
}

// ---------------------------------------------------------------- reductions
// One block sums up to two partial arrays in a fixed order (thread t takes t, t+NT, ...).
__global__ void __launch_bounds__(1024) k_reduce2(const double *__restrict__ p1, int n1, double *out1,
                                                  const double *__restrict__ p2, int n2, double *out2) {
    __shared__ double red[32];
    double s = 0.0;
    for (int i = threadIdx.x; i < n1; i += 1024) s += p1[i];
    s = block_sum<1024>(s, red);
    if (threadIdx.x == 0) *out1 = s;
    if (p2) {
        __syncthreads();
        double t = 0.0;
        for (int i = threadIdx.x; i < n2; i += 1024) t += p2[i];
        t = block_sum<1024>(t, red);
        if (threadIdx.x == 0) *out2 = t;
    }
}

npc_status launch_reduce_sum(Context *ctx, const double *partials, int n, double *out, int, const double *partials2,
                             int n2, double *out2) {
    k_reduce2<<<1, 1024, 0, ctx->stream>>>(partials, n, out, partials2, n2, out2);
    NPC_LAUNCH_CHECK();
    return NPC_SUCCESS;
}

// ---------------------------------------------------------------- scale (+dot)
template <bool DOT>
__global__ void __launch_bounds__(VT) k_scale(const double *__restrict__ in, double *__restrict__ out, double alpha,
                                              int n, const double *__restrict__ dotv, double *partials,
                                              const int *done) {
    if (done && *done) return;
    __shared__ double red[VT / 32];
    double acc = 0.0;
    for (int i = blockIdx.x * VT + threadIdx.x; i < n; i += gridDim.x * VT) {
        double v = alpha * in[i];
        out[i] = v;
        if (DOT) acc += v * dotv[i];
    }
    if (DOT) {
        acc = block_sum<VT>(acc, red);
        if (threadIdx.x == 0) partials[blockIdx.x] = acc;
    }
}

npc_status launch_scale(Context *ctx, const double *in, double *out, double alpha, int n, const double *dotv,
                        double *partials, int *nparts, const int *done) {
    int g = vec_grid(n);
    if (nparts) *nparts = g;
    if (dotv)
        k_scale<true><<<g, VT, 0, ctx->stream>>>(in, out, alpha, n, dotv, partials, done);
    else
        k_scale<false><<<g, VT, 0, ctx->stream>>>(in, out, alpha, n, nullptr, nullptr, done);
    NPC_LAUNCH_CHECK();
    return NPC_SUCCESS;
}

// ---------------------------------------------------------------- dot partials
__global__ void __launch_bounds__(VT) k_dot(const double *__restrict__ a, const double *__restrict__ b, int n,
                                            double *partials) {
    __shared__ double red[VT / 32];
    double acc = 0.0;
    for (int i = blockIdx.x * VT + threadIdx.x; i < n; i += gridDim.x * VT) acc += a[i] * b[i];
    acc = block_sum<VT>(acc, red);
    if (threadIdx.x == 0) partials[blockIdx.x] = acc;
}

npc_status launch_dot(Context *ctx, const double *a, const double *b, int n, double *partials, int *nparts) {
    int g = vec_grid(n);
    *nparts = g;
    k_dot<<<g, VT, 0, ctx->stream>>>(a, b, n, partials);
    NPC_LAUNCH_CHECK();
    return NPC_SUCCESS;
}

// ---------------------------------------------------------------- recurrence epilogue
// out = a*y + b*x + c*s2 + d*r (+ partial <out, dotv>): the Chebyshev update of Alg. 2
// steps 5-6 for operators whose A-application is not fused (callback).
template <bool HAS_S2, bool HAS_R, bool DOT>
__global__ void __launch_bounds__(VT) k_axpby(const double *__restrict__ y, const double *__restrict__ x,
                                              const double *s2, const double *__restrict__ r, double *out, int n,
                                              double a, double b, double c, double d,
                                              const double *__restrict__ dotv, double *partials, const int *done) {
    if (done && *done) return;
    __shared__ double red[VT / 32];
    double acc = 0.0;
    for (int i = blockIdx.x * VT + threadIdx.x; i < n; i += gridDim.x * VT) {
        double v = a * y[i] + b * x[i];
        if (HAS_S2) v += c * s2[i];
        if (HAS_R) v += d * r[i];
        out[i] = v;
        if (DOT) acc += v * dotv[i];
    }
    if (DOT) {
        acc = block_sum<VT>(acc, red);
        if (threadIdx.x == 0) partials[blockIdx.x] = acc;
    }
}

npc_status launch_axpby_step(Context *ctx, const double *y, const StepArgs &s, int n) {
    int g = vec_grid(n);
    const bool h2 = s.s2 != nullptr, hr = s.r != nullptr, dt = s.dotv != nullptr;
#define NPC_AXPBY(H2, HR, DT)                                                                                 \
    k_axpby<H2, HR, DT><<<g, VT, 0, ctx->stream>>>(y, s.x, s.s2, s.r, s.out, n, s.a, s.b, s.c, s.d, s.dotv, \
                                                   s.partials, s.done)
    if (h2 && hr && dt) NPC_AXPBY(true, true, true);
    else if (h2 && hr) NPC_AXPBY(true, true, false);
    else if (h2 && dt) NPC_AXPBY(true, false, true);
    else if (h2) NPC_AXPBY(true, false, false);
    else if (hr && dt) NPC_AXPBY(false, true, true);
    else if (hr) NPC_AXPBY(false, true, false);
    else if (dt) NPC_AXPBY(false, false, true);
    else NPC_AXPBY(false, false, false);
#undef NPC_AXPBY
    NPC_LAUNCH_CHECK();
    return NPC_SUCCESS;
}

// ---------------------------------------------------------------- permutations, fill
__global__ void k_gather(const double *__restrict__ in, const int *__restrict__ idx, double *__restrict__ out, int n) {
    for (int i = blockIdx.x * VT + threadIdx.x; i < n; i += gridDim.x * VT) out[i] = in[idx[i]];
}
__global__ void k_scatter(const double *__restrict__ in, const int *__restrict__ idx, double *__restrict__ out, int n) {
    for (int i = blockIdx.x * VT + threadIdx.x; i < n; i += gridDim.x * VT) out[idx[i]] = in[i];
}
__global__ void k_fill(double *out, double v, int n) {
    for (int i = blockIdx.x * VT + threadIdx.x; i < n; i += gridDim.x * VT) out[i] = v;
}

npc_status launch_gather(Context *ctx, const double *in, const int *idx, double *out, int n) {
    if (n <= 0) return NPC_SUCCESS;
    k_gather<<<vec_grid(n), VT, 0, ctx->stream>>>(in, idx, out, n);
    NPC_LAUNCH_CHECK();
    return NPC_SUCCESS;
}
npc_status launch_scatter(Context *ctx, const double *in, const int *idx, double *out, int n) {
    if (n <= 0) return NPC_SUCCESS;
    k_scatter<<<vec_grid(n), VT, 0, ctx->stream>>>(in, idx, out, n);
    NPC_LAUNCH_CHECK();
    return NPC_SUCCESS;
}
npc_status launch_fill(Context *ctx, double *out, double v, int n) {
    if (n <= 0) return NPC_SUCCESS;
    k_fill<<<vec_grid(n), VT, 0, ctx->stream>>>(out, v, n);
    NPC_LAUNCH_CHECK();
    return NPC_SUCCESS;
}

__global__ void k_sum_rows(const double *__restrict__ rows, int P, int m, double *__restrict__ out) {
    for (int i = blockIdx.x * VT + threadIdx.x; i < m; i += gridDim.x * VT) {
        double a = 0.0;
        for (int q = 0; q < P; ++q) a += rows[(size_t)q * m + i];
        out[i] = a;
    }
}

npc_status launch_sum_rows(Context *ctx, const double *rows, int P, int m, double *out, cudaStream_t s) {
    (void)ctx;
    if (m <= 0) return NPC_SUCCESS;
    k_sum_rows<<<vec_grid(m), VT, 0, s>>>(rows, P, m, out);
    NPC_LAUNCH_CHECK();
    return NPC_SUCCESS;
}

// splitmix64 of (seed, global index) -> uniform [-1, 1): identical for any rank count.
__global__ void k_hash(double *out, int n, long long offset, unsigned long long seed) {
    for (int i = blockIdx.x * VT + threadIdx.x; i < n; i += gridDim.x * VT) {
        unsigned long long z = seed + 0x9E3779B97F4A7C15ull * (unsigned long long)(offset + i + 1);
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        z ^= z >> 31;
        out[i] = 2.0 * ((double)(z >> 11) * (1.0 / 9007199254740992.0)) - 1.0;
    }
}
npc_status launch_hash_vector(Context *ctx, double *out, int n, long long offset, unsigned long long seed) {
    if (n <= 0) return NPC_SUCCESS;
    k_hash<<<vec_grid(n), VT, 0, ctx->stream>>>(out, n, offset, seed);
    NPC_LAUNCH_CHECK();
    return NPC_SUCCESS;
}

}  // namespace npc
