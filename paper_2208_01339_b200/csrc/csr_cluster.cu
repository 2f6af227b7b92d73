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

// ================================================================== whole PCG in one cluster
// The single-reduction PCG of solvers.cu (same recurrences, scalars, stopping rule, true-
// residual check and residual replacement -- DESIGN.md readings A5, A23) run to convergence
// inside ONE cluster launch: every vector lives in the CTAs' shared memory, the polynomial is
// the loop above, inner products are block sums exchanged through DSMEM (each CTA sums the
// cluster's partials in rank order, so every CTA holds identical scalars), and the host syncs
// once per solve instead of once per chunk of graph replays.
struct ClusterReduce {
    double *slots;  // [2 sets][3 values][16 ranks] in every CTA (only CTA 0's are written)
    int set = 0;
};

__device__ __forceinline__ void block_sums3(double &a, double &b, double &c, double *red /* 3 x 32 */) {
    a = warp_sum(a);
    b = warp_sum(b);
    c = warp_sum(c);
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
    __syncthreads();  // red reuse
    if (lane == 0) {
        red[w] = a;
        red[32 + w] = b;
        red[64 + w] = c;
    }
    __syncthreads();
    if (w == 0) {
        double x = lane < nw ? red[lane] : 0.0, y = lane < nw ? red[32 + lane] : 0.0,
               z = lane < nw ? red[64 + lane] : 0.0;
        x = warp_sum(x);
        y = warp_sum(y);
        z = warp_sum(z);
        if (lane == 0) {
            red[96] = x;
            red[97] = y;
            red[98] = z;
        }
    }
    __syncthreads();
    a = red[96];
    b = red[97];
    c = red[98];
}

// Cluster-wide sums of up to 3 values (all threads of all CTAs get identical results).
__device__ __forceinline__ void cluster_sums3(cg::cluster_group &cl, ClusterReduce &cr, double *red, double &a,
                                              double &b, double &c) {
    block_sums3(a, b, c, red);
    const int nb = (int)cl.num_blocks(), me = (int)cl.block_rank();
    double *s0 = cl.map_shared_rank(cr.slots, 0) + cr.set * 48;
    if (threadIdx.x == 0) {
        s0[me] = a;
        s0[16 + me] = b;
        s0[32 + me] = c;
    }
    cl.sync();
    double x = 0.0, y = 0.0, z = 0.0;
    for (int q = 0; q < nb; ++q) {  // rank order: identical bits in every CTA
        x += s0[q];
        y += s0[16 + q];
        z += s0[32 + q];
    }
    a = x;
    b = y;
    c = z;
    cr.set ^= 1;
}

// out_i = a (A xs)_i + b xs_i + c s2_i + d rr_i for the CTA's rows (xs gathered over DSMEM)
__device__ __forceinline__ double row_apply(cg::cluster_group &cl, int c, int R, int row0, const int *rp,
                                            const int *cs, const double *vs, const double *xs, int i) {
    double y = 0.0;
    for (int p = rp[i]; p < rp[i + 1]; ++p) {
        const int col = cs[p];
        const int owner = col / R;
        const double xv = owner == c ? xs[col - row0] : cl.map_shared_rank(xs, owner)[col - owner * R];
        y += vs[p] * xv;
    }
    return y;
}

__global__ void k_csr_pcg_cluster(SmallCsrDev A, const double *__restrict__ b, double *__restrict__ x_io,
                                  const double *__restrict__ coef, int k, double tb, int use_poly, double tol2b,
                                  int maxit, ClusterPcgOut *out, double *history) {
    cg::cluster_group cl = cg::this_cluster();
    const int c = (int)cl.block_rank();
    const int R = A.R;
    const int row0 = c * R, row1 = min(A.n, row0 + R), nr = max(0, row1 - row0);
    extern __shared__ __align__(16) double sm[];
    double *X = sm, *Rv = sm + R, *U = sm + 2 * R, *Wv = sm + 3 * R, *Pv = sm + 4 * R, *Sv = sm + 5 * R;
    double *bufA = sm + 6 * R, *bufB = sm + 7 * R, *Bv = sm + 8 * R;
    double *vs = sm + 9 * R;
    int *cs = reinterpret_cast<int *>(vs + A.nnz_cta);
    int *rp = cs + A.nnz_cta;
    __shared__ double slots[2 * 48];
    __shared__ double red[100];
    ClusterReduce cr{slots, 0};
    const int p0 = A.rowptr[row0 < A.n ? row0 : A.n], p1 = A.rowptr[row1 < A.n ? row1 : A.n];
    for (int e = threadIdx.x; e < p1 - p0; e += blockDim.x) {
        vs[e] = A.vals[p0 + e];
        cs[e] = A.cols[p0 + e];
    }
    if (nr > 0)
        for (int i = threadIdx.x; i <= nr; i += blockDim.x) rp[i] = A.rowptr[row0 + i] - p0;
    double bb = 0.0, xx = 0.0, dummy = 0.0;
    for (int i = threadIdx.x; i < nr; i += blockDim.x) {
        const double bi = b[row0 + i], xi = x_io[row0 + i];
        Bv[i] = bi;
        X[i] = xi;
        Pv[i] = 0.0;
        Sv[i] = 0.0;
        bb += bi * bi;
        xx += xi * xi;
    }
    cluster_sums3(cl, cr, red, bb, xx, dummy);  // also publishes X for the gathers below
    const double bnorm2 = bb;
    if (tol2b < 0.0) tol2b = -tol2b * bnorm2;  // given as -tol^2: the threshold is tol^2 ||b||^2
    const bool x0_nonzero = xx != 0.0;
    int iters = 0, converged = 0, breakdown = 0, true_checks = 0, applications = 0, reductions = 1;
    double rr = 0.0, relres_true = 0.0;
    if (bnorm2 == 0.0) {  // b = 0 -> x = 0
        for (int i = threadIdx.x; i < nr; i += blockDim.x) x_io[row0 + i] = 0.0;
        cl.sync();  // CTA 0's reduction slots may still be read by the others: nobody leaves early
        if (c == 0 && threadIdx.x == 0) {
            out->iters = 0;
            out->converged = 1;
            out->breakdown = 0;
            out->applications = 0;
            out->reductions = 1;
            out->rr = 0.0;
            out->relres_true = 0.0;
            out->bnorm2 = 0.0;
        }
        return;
    }
    // r0 = b - A x0 (or b)
    double t0 = 0.0, t1 = 0.0, t2 = 0.0;
    for (int i = threadIdx.x; i < nr; i += blockDim.x) {
        const double ri = x0_nonzero ? Bv[i] - row_apply(cl, c, R, row0, rp, cs, vs, X, i) : Bv[i];
        Rv[i] = ri;
        t0 += ri * ri;
    }
    if (x0_nonzero) ++applications;
    cluster_sums3(cl, cr, red, t0, t1, t2);
    ++reductions;
    rr = t0;
    if (history && c == 0 && threadIdx.x == 0) history[0] = sqrt(rr / bnorm2);
    bool want_true = rr <= tol2b, have_true = false;  // have_true: relres_true is for the current x
    double gamma_old = 0.0, alpha_old = 0.0;
    bool first = true;
    for (;;) {
        if (want_true) {
            // true residual b - A x; accept or replace r and continue (reading A23)
            double q = 0.0, u1 = 0.0, u2 = 0.0;
            cl.sync();  // X final everywhere
            for (int i = threadIdx.x; i < nr; i += blockDim.x) {
                const double ti = Bv[i] - row_apply(cl, c, R, row0, rp, cs, vs, X, i);
                U[i] = ti;
                q += ti * ti;
            }
            ++applications;
            cluster_sums3(cl, cr, red, q, u1, u2);
            ++reductions;
            relres_true = sqrt(q / bnorm2);
            have_true = true;
            if (q <= tol2b || ++true_checks > 50) {
                converged = q <= tol2b;
                break;
            }
            for (int i = threadIdx.x; i < nr; i += blockDim.x) Rv[i] = U[i];
            rr = q;
            converged = 0;
            want_true = false;
            first = true;  // restart the recurrence from the current x (reading A23)
            if (iters >= maxit) break;
            cl.sync();  // replaced r visible before the polynomial gathers it
        }
        if (iters >= maxit) break;
        // u = p_k(A) r (Alg. 2, the same recurrence as k_csr_poly_cluster)
        double *ufin;
        if (!use_poly) {
            for (int i = threadIdx.x; i < nr; i += blockDim.x) U[i] = Rv[i];
            ufin = U;
        } else if (k == 0) {
            for (int i = threadIdx.x; i < nr; i += blockDim.x) U[i] = Rv[i] / tb;
            ufin = U;
        } else {
            for (int j = 1; j <= k; ++j) {
                const double *cf = coef + 4 * (j - 1);
                double a, bq, cc = 0.0, d = 0.0;
                const double *xs;
                double *o = (j & 1) ? bufB : bufA;
                if (j == 1) {
                    xs = Rv;
                    a = cf[0] / tb;
                    bq = cf[1] / tb + cf[3];
                } else if (j == 2) {
                    xs = bufB;
                    a = cf[0];
                    bq = cf[1];
                    d = cf[2] / tb + cf[3];
                } else {
                    xs = (j & 1) ? bufA : bufB;
                    a = cf[0];
                    bq = cf[1];
                    cc = cf[2];
                    d = cf[3];
                }
                for (int i = threadIdx.x; i < nr; i += blockDim.x) {
                    const double y = row_apply(cl, c, R, row0, rp, cs, vs, xs, i);
                    double ov = a * y + bq * xs[i];
                    if (j >= 3) ov += cc * o[i];
                    if (j >= 2) ov += d * Rv[i];
                    o[i] = ov;
                }
                cl.sync();
            }
            ufin = (k & 1) ? bufB : bufA;
        }
        applications += use_poly ? k : 0;
        if (!use_poly || k == 0) cl.sync();  // u visible for w = A u
        // w = A u; gamma = <r, u>, delta = <u, w>
        double g = 0.0, dl = 0.0, unused = 0.0;
        for (int i = threadIdx.x; i < nr; i += blockDim.x) {
            const double ui = ufin[i];
            const double wi = row_apply(cl, c, R, row0, rp, cs, vs, ufin, i);
            Wv[i] = wi;
            g += Rv[i] * ui;
            dl += ui * wi;
        }
        ++applications;
        cluster_sums3(cl, cr, red, g, dl, unused);
        ++reductions;
        if (!(g > 0.0)) {
            breakdown = 1;
            break;
        }
        double beta = 0.0, denom = dl;
        if (!first) {
            beta = g / gamma_old;
            denom = dl - beta * g / alpha_old;
        }
        if (!(denom > 0.0)) {
            breakdown = 2;
            break;
        }
        const double alpha = g / denom;
        gamma_old = g;
        alpha_old = alpha;
        first = false;
        // p = u + beta p; s = w + beta s; x += alpha p; r -= alpha s; ||r||^2
        double q = 0.0, u1 = 0.0, u2 = 0.0;
        for (int i = threadIdx.x; i < nr; i += blockDim.x) {
            const double pi = ufin[i] + beta * Pv[i];
            const double si = Wv[i] + beta * Sv[i];
            Pv[i] = pi;
            Sv[i] = si;
            X[i] += alpha * pi;
            const double ri = Rv[i] - alpha * si;
            Rv[i] = ri;
            q += ri * ri;
        }
        cluster_sums3(cl, cr, red, q, u1, u2);  // also publishes the new r for the next polynomial
        ++iters;
        have_true = false;
        rr = q;
        if (history && c == 0 && threadIdx.x == 0) history[iters] = sqrt(rr / bnorm2);
        if (rr <= tol2b) want_true = true;
        else if (iters >= maxit) break;
    }
    for (int i = threadIdx.x; i < nr; i += blockDim.x) x_io[row0 + i] = X[i];
    if (!have_true && !converged) {
        // maxit: report the true residual of the final iterate
        double q = 0.0, u1 = 0.0, u2 = 0.0;
        cl.sync();
        for (int i = threadIdx.x; i < nr; i += blockDim.x) {
            const double ti = Bv[i] - row_apply(cl, c, R, row0, rp, cs, vs, X, i);
            q += ti * ti;
        }
        ++applications;
        cluster_sums3(cl, cr, red, q, u1, u2);
        ++reductions;
        relres_true = sqrt(q / bnorm2);
    }
    cl.sync();  // no CTA leaves while others may still read its shared memory
    if (c == 0 && threadIdx.x == 0) {
        out->iters = iters;
        out->converged = converged;
        out->breakdown = breakdown;
        out->applications = applications;
        out->reductions = reductions;
        out->rr = rr;
        out->relres_true = relres_true;
        out->bnorm2 = bnorm2;
    }
}

// ================================================================== Lanczos in one cluster
// The m-step Lanczos of solvers.cu (same recurrence and operation order: q = v0 / ||v0||;
// w = A q - beta_{j-1} q_prev; alpha_j = <q, w>; w -= alpha_j q; beta_j = ||w||; stop when
// beta_j = 0) for small CSR operators, all steps in one launch.  Writes alpha, beta and the
// number of steps taken; the host then forms the Ritz values exactly as for the grid path.
__global__ void k_csr_lanczos_cluster(SmallCsrDev A, const double *__restrict__ v0, int m, double *alphas,
                                      double *betas, int *steps_out) {
    cg::cluster_group cl = cg::this_cluster();
    const int c = (int)cl.block_rank();
    const int R = A.R;
    const int row0 = c * R, row1 = min(A.n, row0 + R), nr = max(0, row1 - row0);
    extern __shared__ __align__(16) double sm[];
    double *Q = sm, *Qp = sm + R, *Wv = sm + 2 * R;
    double *vs = sm + 9 * R;  // same layout as the PCG kernel (fits whenever it does)
    int *cs = reinterpret_cast<int *>(vs + A.nnz_cta);
    int *rp = cs + A.nnz_cta;
    __shared__ double slots[2 * 48];
    __shared__ double red[100];
    ClusterReduce cr{slots, 0};
    const int p0 = A.rowptr[row0 < A.n ? row0 : A.n], p1 = A.rowptr[row1 < A.n ? row1 : A.n];
    for (int e = threadIdx.x; e < p1 - p0; e += blockDim.x) {
        vs[e] = A.vals[p0 + e];
        cs[e] = A.cols[p0 + e];
    }
    if (nr > 0)
        for (int i = threadIdx.x; i <= nr; i += blockDim.x) rp[i] = A.rowptr[row0 + i] - p0;
    double vn = 0.0, u1 = 0.0, u2 = 0.0;
    for (int i = threadIdx.x; i < nr; i += blockDim.x) {
        const double v = v0[row0 + i];
        Wv[i] = v;
        vn += v * v;
    }
    cluster_sums3(cl, cr, red, vn, u1, u2);
    const double inv0 = 1.0 / sqrt(vn);
    for (int i = threadIdx.x; i < nr; i += blockDim.x) {
        Q[i] = Wv[i] * inv0;
        Qp[i] = 0.0;
    }
    cl.sync();
    double beta_prev = 0.0;
    int steps = 0;
    for (int j = 0; j < m; ++j) {
        double a = 0.0, t1 = 0.0, t2 = 0.0;
        for (int i = threadIdx.x; i < nr; i += blockDim.x) {
            double wi = row_apply(cl, c, R, row0, rp, cs, vs, Q, i);
            if (j) wi -= beta_prev * Qp[i];
            Wv[i] = wi;
            a += Q[i] * wi;
        }
        cluster_sums3(cl, cr, red, a, t1, t2);
        double bb = 0.0;
        t1 = t2 = 0.0;
        for (int i = threadIdx.x; i < nr; i += blockDim.x) {
            const double wi = Wv[i] - a * Q[i];
            Wv[i] = wi;
            bb += wi * wi;
        }
        cluster_sums3(cl, cr, red, bb, t1, t2);
        const double bj = sqrt(bb);
        if (c == 0 && threadIdx.x == 0) {
            alphas[j] = a;
            betas[j] = bj;
        }
        steps = j + 1;
        if (bj == 0.0) break;
        const double inv = 1.0 / bj;
        for (int i = threadIdx.x; i < nr; i += blockDim.x) {
            Qp[i] = Q[i];
            Q[i] = Wv[i] * inv;
        }
        beta_prev = bj;
        cl.sync();  // new q visible before the next gathers
    }
    cl.sync();
    if (c == 0 && threadIdx.x == 0) *steps_out = steps;
}

// Non-portable cluster size (16) and the dynamic shared memory limit, set once per process.
static cudaError_t cluster_attrs() {
    static std::once_flag once;
    static cudaError_t err = cudaSuccess;
    std::call_once(once, [] {
        err = cudaFuncSetAttribute(k_csr_poly_cluster, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        if (err == cudaSuccess)
            err = cudaFuncSetAttribute(k_csr_poly_cluster, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        if (err == cudaSuccess)
            err = cudaFuncSetAttribute(k_csr_pcg_cluster, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        if (err == cudaSuccess)
            err = cudaFuncSetAttribute(k_csr_pcg_cluster, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        if (err == cudaSuccess)
            err = cudaFuncSetAttribute(k_csr_lanczos_cluster, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        if (err == cudaSuccess)
            err = cudaFuncSetAttribute(k_csr_lanczos_cluster, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       200 * 1024);
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
        // whole-PCG kernel: 9 vectors instead of 3
        const size_t smem_pcg = smem + sizeof(double) * 6 * (size_t)R;
        pl.smem_pcg = 0;
        if (smem_pcg <= 200 * 1024) {
            cfg.dynamicSmemBytes = smem_pcg;
            int nc2 = 0;
            if (cudaOccupancyMaxActiveClusters(&nc2, k_csr_pcg_cluster, &cfg) == cudaSuccess && nc2 >= 1)
                pl.smem_pcg = smem_pcg;
            else
                cudaGetLastError();
        }
        return true;
    }
    return false;
}

}  // namespace npc

namespace npc {

npc_status launch_csr_pcg_cluster(Context *ctx, const SmallCsrDev &A, const SmallCsrPlan &pl, const double *b,
                                  double *x, const double *coef, int k, double tb, int use_poly, double tol2b,
                                  int maxit, ClusterPcgOut *out, double *history) {
    NPC_CUDA_TRY(cluster_attrs());
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(pl.cl_size, 1, 1);
    cfg.blockDim = dim3(pl.threads, 1, 1);
    cfg.dynamicSmemBytes = pl.smem_pcg;
    cfg.stream = ctx->stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = pl.cl_size;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    NPC_CUDA_TRY(cudaLaunchKernelEx(&cfg, k_csr_pcg_cluster, A, b, x, coef, k, tb, use_poly, tol2b, maxit, out,
                                    history));
    NPC_LAUNCH_CHECK();
    return NPC_SUCCESS;
}

}  // namespace npc

namespace npc {

npc_status launch_csr_lanczos_cluster(Context *ctx, const SmallCsrDev &A, const SmallCsrPlan &pl, const double *v0,
                                      int m, double *alphas, double *betas, int *steps) {
    NPC_CUDA_TRY(cluster_attrs());
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(pl.cl_size, 1, 1);
    cfg.blockDim = dim3(pl.threads, 1, 1);
    cfg.dynamicSmemBytes = pl.smem_pcg;
    cfg.stream = ctx->stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = pl.cl_size;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    NPC_CUDA_TRY(cudaLaunchKernelEx(&cfg, k_csr_lanczos_cluster, A, v0, m, alphas, betas, steps));
    NPC_LAUNCH_CHECK();
    return NPC_SUCCESS;
}

}  // namespace npc
