// csr_cluster.cu -- the whole polynomial p_k(A) r in ONE launch for small CSR operators, on a
// thread-block cluster whose CTAs keep their rows of A and of every recurrence vector in
// shared memory and read their neighbours' entries of s_{j-1} through distributed shared
// memory (DSMEM), with one cluster barrier per degree.
//
// Why: at n = 4,096 (BASELINE config 1) a degree moves 0.39 MB; a grid launch per degree costs
// more than the work (launch + ramp + tail ≈ 4-5 µs per degree), so the polynomial is latency
// bound.  Here the k degrees of Alg. 2 run inside one cluster: the matrix
// is read from HBM once per application instead of k times, and a degree costs a few DSMEM
// gathers per row plus a barrier.  Same arithmetic and operation order per row as
// k_csr_step (row sums in stored column order, then the fused three-term epilogue).
#include <cooperative_groups.h>

#include <algorithm>
#include <mutex>

#include "device_util.cuh"
#include "npc_internal.cuh"

namespace cg = cooperative_groups;

namespace npc {

__global__ void k_csr_poly_cluster(SmallCsrDev A, const double *__restrict__ r, double *__restrict__ z,
                                   const double *__restrict__ coef, int k, double tb,
                                   const double *__restrict__ dotv, double *partials, const int *done) {
    if (done && *done) return;  // uniform over the cluster
    cg::cluster_group cl = cg::this_cluster();
    const int c = (int)cl.block_rank();
    const int R = A.R;
    const int row0 = c * R, row1 = min(A.n, row0 + R), nr = max(0, row1 - row0);
    extern __shared__ __align__(16) double sm[];
    double *bufA = sm, *bufB = sm + R, *rs = sm + 2 * R;  // s_even, s_odd, r (own rows)
    double *vs = sm + 3 * R;
    int *cs = reinterpret_cast<int *>(vs + A.nnz_cta);
    int *rp = cs + A.nnz_cta;
    const int p0 = A.rowptr[row0 < A.n ? row0 : A.n], p1 = A.rowptr[row1 < A.n ? row1 : A.n];
    for (int e = threadIdx.x; e < p1 - p0; e += blockDim.x) {
        vs[e] = A.vals[p0 + e];
        cs[e] = A.cols[p0 + e];
    }
    if (nr > 0)
        for (int i = threadIdx.x; i <= nr; i += blockDim.x) rp[i] = A.rowptr[row0 + i] - p0;
    for (int i = threadIdx.x; i < nr; i += blockDim.x) rs[i] = r[row0 + i];
    cl.sync();  // every CTA's r is in place (degree 1 gathers it)
    for (int j = 1; j <= k; ++j) {
        const double *cf = coef + 4 * (j - 1);
        double a, b, cc = 0.0, d = 0.0;
        const double *xs;  // s_{j-1} (own rows), at the same offset in every CTA
        double *out = (j & 1) ? bufB : bufA;  // s_j over s_{j-2}
        if (j == 1) {
            xs = rs;
            a = cf[0] / tb;
            b = cf[1] / tb + cf[3];
        } else if (j == 2) {
            xs = bufB;
            a = cf[0];
            b = cf[1];
            d = cf[2] / tb + cf[3];
        } else {
            xs = (j & 1) ? bufA : bufB;
            a = cf[0];
            b = cf[1];
            cc = cf[2];
            d = cf[3];
        }
        for (int i = threadIdx.x; i < nr; i += blockDim.x) {
            double y = 0.0;
            for (int p = rp[i]; p < rp[i + 1]; ++p) {
                const int col = cs[p];
                const int owner = col / R;
                double xv;
                if (owner == c) {
                    xv = xs[col - row0];
                } else {
                    const double *remote = cl.map_shared_rank(xs, owner);
                    xv = remote[col - owner * R];
                }
                y += vs[p] * xv;
            }
            double o = a * y + b * xs[i];
            if (j >= 3) o += cc * out[i];
            if (j >= 2) o += d * rs[i];
            out[i] = o;
        }
        cl.sync();  // s_j complete everywhere before anyone gathers it (and s_{j-1} is free)
    }
    const double *fin = (k & 1) ? bufB : bufA;
    double acc = 0.0;
    for (int i = threadIdx.x; i < nr; i += blockDim.x) {
        const double v = fin[i];
        z[row0 + i] = v;
        if (dotv) acc += v * dotv[row0 + i];
    }
    if (dotv) {  // block sum over the actual warps of this launch
        __shared__ double red[32];
        acc = warp_sum(acc);
        const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
        if (lane == 0) red[w] = acc;
        __syncthreads();
        if (w == 0) {
            double t = lane < nw ? red[lane] : 0.0;
            t = warp_sum(t);
            if (lane == 0) partials[c] = t;
        }
    }
}

// Non-portable cluster size (16) and the dynamic shared memory limit, set once per process.
static cudaError_t cluster_attrs() {
    static std::once_flag once;
    static cudaError_t err = cudaSuccess;
    std::call_once(once, [] {
        err = cudaFuncSetAttribute(k_csr_poly_cluster, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        if (err == cudaSuccess)
            err = cudaFuncSetAttribute(k_csr_poly_cluster, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    });
    return err;
}

npc_status launch_csr_poly_cluster(Context *ctx, const SmallCsrDev &A, int cl_size, int threads, size_t smem,
                                   const double *r, double *z, const double *coef, int k, double tb,
                                   const double *dotv, double *partials, const int *done) {
    NPC_CUDA_TRY(cluster_attrs());
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cl_size, 1, 1);
    cfg.blockDim = dim3(threads, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = ctx->stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cl_size;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    NPC_CUDA_TRY(cudaLaunchKernelEx(&cfg, k_csr_poly_cluster, A, r, z, coef, k, tb, dotv, partials, done));
    NPC_LAUNCH_CHECK();
    return NPC_SUCCESS;
}

// Can this operator run the cluster-resident polynomial?  Picks the cluster size (<= 16) and
// block size; false if the device cannot co-schedule such a cluster.
bool plan_csr_poly_cluster(int n, const int *rowptr, SmallCsrPlan &pl) {
    if (n <= 0 || n > 16384) return false;
    for (int cl_size : {16, 8}) {  // more SMs first (gathers in parallel), 8 = portable size
        const int R = (n + cl_size - 1) / cl_size;
        int nnz_cta = 0;
        for (int c = 0; c < cl_size; ++c) {
            const int r0 = std::min(n, c * R), r1 = std::min(n, r0 + R);
            nnz_cta = std::max(nnz_cta, rowptr[r1] - rowptr[r0]);
        }
        nnz_cta = (nnz_cta + 1) & ~1;
        const size_t smem = sizeof(double) * (3 * (size_t)R + nnz_cta) + sizeof(int) * ((size_t)nnz_cta + R + 1);
        if (smem > 200 * 1024) continue;
        const int threads = std::min(1024, std::max(32, (R + 31) / 32 * 32));
        if (cluster_attrs() != cudaSuccess) {
            cudaGetLastError();
            return false;
        }
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(cl_size, 1, 1);
        cfg.blockDim = dim3(threads, 1, 1);
        cfg.dynamicSmemBytes = smem;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = cl_size;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        int nclusters = 0;
        if (cudaOccupancyMaxActiveClusters(&nclusters, k_csr_poly_cluster, &cfg) != cudaSuccess || nclusters < 1) {
            cudaGetLastError();
            continue;
        }
        pl.cl_size = cl_size;
        pl.R = R;
        pl.nnz_cta = nnz_cta;
        pl.threads = threads;
        pl.smem = smem;
        return true;
    }
    return false;
}

}  // namespace npc
