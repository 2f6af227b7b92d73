// lowrank.cu -- low-rank spectral correction of the polynomial preconditioner (PAPER.md:483-508,
// Sec. "Low-rank acceleration"):
//
//     P = P_0 + V (V^T A V)^{-1} V^T,     V = [v_1 .. v_p]  (approximate leftmost eigenvectors)
//
// P_0 = p_k(A) (Alg. 2, or Newton Alg. 1).  On an exact eigenvector v_j (j <= p) the
// preconditioned eigenvalue becomes mu_j + 1 (Eq. plusone), which moves the smallest
// eigenvalues of P_0 A into the interior of the spectrum.
//
// Device layout: V in the operator's internal row order, column-major (column j at V + j*ldv,
// ldv = n_local), G^{-1} = (V^T A V)^{-1} as p x p row-major (inverted on the host from the
// Cholesky factor at setup).  One application of the correction costs one fused multi-dot
// (V^T r, p partial sums per block), one reduction (+ one allreduce of p scalars when
// nranks > 1), a one-thread p x p product c = G^{-1} s, and one fused kernel
// z += V c (+ the PCG partial <z, r>).  These are the only inner products inside the
// preconditioner: the price of the correction the paper accepts.
//
// Ritz vectors (approximate leftmost eigenvectors): Lanczos with full reorthogonalisation
// (classical Gram-Schmidt twice against the stored basis Q), the tridiagonal eigenpairs on the
// host (Sturm bisection + inverse iteration), V = Q S on the device.
#include <algorithm>
#include <cmath>
#include <vector>

#include "device_util.cuh"
#include "npc_internal.cuh"

namespace npc {

static constexpr int LR_T = 256;

// partials[j * G + block] = sum_i V_j[i] r[i] over the block's rows, j < p (p <= NPC_LOWRANK_MAX)
__global__ void __launch_bounds__(LR_T) k_multidot(const double *__restrict__ V, long long ldv, int p,
                                                   const double *__restrict__ r, int n, double *partials,
                                                   const int *done) {
    if (done && *done) return;
    __shared__ double red[LR_T / 32];
    double acc[NPC_LOWRANK_MAX];
#pragma unroll
    for (int j = 0; j < NPC_LOWRANK_MAX; ++j) acc[j] = 0.0;
    for (int i = blockIdx.x * LR_T + threadIdx.x; i < n; i += gridDim.x * LR_T) {
        const double ri = r[i];
#pragma unroll
        for (int j = 0; j < NPC_LOWRANK_MAX; ++j)
            if (j < p) acc[j] += V[j * ldv + i] * ri;
    }
    for (int j = 0; j < p; ++j) {
        const double t = block_sum<LR_T>(acc[j], red);
        if (threadIdx.x == 0) partials[(size_t)j * gridDim.x + blockIdx.x] = t;
        __syncthreads();
    }
}

// sums[j] = sum of row j of partials (fixed order), one warp-block per row
__global__ void __launch_bounds__(1024) k_reduce_rows(const double *__restrict__ partials, int G, int p,
                                                      double *sums, const int *done) {
    if (done && *done) return;
    __shared__ double red[32];
    for (int j = 0; j < p; ++j) {
        double t = 0.0;
        for (int i = threadIdx.x; i < G; i += 1024) t += partials[(size_t)j * G + i];
        t = block_sum<1024>(t, red);
        if (threadIdx.x == 0) sums[j] = t;
        __syncthreads();
    }
}

// c = Ginv s (p x p row-major)
__global__ void k_lr_coef(const double *__restrict__ Ginv, int p, const double *s, double *c, const int *done) {
    if (done && *done) return;
    for (int a = 0; a < p; ++a) {
        double t = 0.0;
        for (int b = 0; b < p; ++b) t += Ginv[a * p + b] * s[b];
        c[a] = t;
    }
}

// z += sum_j V_j c_j  (+ partial <z, dotv>)
template <bool DOT>
__global__ void __launch_bounds__(LR_T) k_lr_correct(double *__restrict__ z, const double *__restrict__ V,
                                                     long long ldv, int p, const double *__restrict__ c, int n,
                                                     const double *__restrict__ dotv, double *partials,
                                                     const int *done) {
    if (done && *done) return;
    __shared__ double red[LR_T / 32];
    __shared__ double cs[NPC_LOWRANK_MAX];
    if (threadIdx.x < p) cs[threadIdx.x] = c[threadIdx.x];
    __syncthreads();
    double acc = 0.0;
    for (int i = blockIdx.x * LR_T + threadIdx.x; i < n; i += gridDim.x * LR_T) {
        double zi = z[i];
        for (int j = 0; j < p; ++j) zi += V[j * ldv + i] * cs[j];
        z[i] = zi;
        if (DOT) acc += zi * dotv[i];
    }
    if (DOT) {
        acc = block_sum<LR_T>(acc, red);
        if (threadIdx.x == 0) partials[blockIdx.x] = acc;
    }
}

// w -= sum_{l<q} Q_l h_l  (Gram-Schmidt update), Q column-major with stride ldq
__global__ void __launch_bounds__(LR_T) k_gs_update(double *__restrict__ w, const double *__restrict__ Q,
                                                    long long ldq, int q, const double *__restrict__ h, int n) {
    for (int i = blockIdx.x * LR_T + threadIdx.x; i < n; i += gridDim.x * LR_T) {
        double wi = w[i];
        for (int l = 0; l < q; ++l) wi -= Q[l * ldq + i] * h[l];
        w[i] = wi;
    }
}

// out_l[i] = sum_j Q_j[i] S[j * p + l]  (V = Q S; S is m x p row-major)
__global__ void __launch_bounds__(LR_T) k_basis_combine(const double *__restrict__ Q, long long ldq, int m,
                                                        const double *__restrict__ S, int p, double *out,
                                                        long long ldo, int n) {
    for (int i = blockIdx.x * LR_T + threadIdx.x; i < n; i += gridDim.x * LR_T)
        for (int l = 0; l < p; ++l) {
            double t = 0.0;
            for (int j = 0; j < m; ++j) t += Q[j * ldq + i] * S[j * p + l];
            out[l * ldo + i] = t;
        }
}

// s[0..p) = V^T r over all ranks (p <= NPC_LOWRANK_MAX), on ctx->stream.
static npc_status multidot(Context *ctx, const double *V, long long ldv, int p, const double *r, int n,
                           double *part, double *sums, const int *done) {
    const int G = vec_grid(n);
    if (n > 0) {
        k_multidot<<<G, LR_T, 0, ctx->stream>>>(V, ldv, p, r, n, part, done);
        NPC_LAUNCH_CHECK();
        k_reduce_rows<<<1, 1024, 0, ctx->stream>>>(part, G, p, sums, done);
        NPC_LAUNCH_CHECK();
    } else {
        NPC_CUDA_TRY(cudaMemsetAsync(sums, 0, sizeof(double) * p, ctx->stream));
    }
    return ctx->allreduce_sum(sums, p);
}

// Host Cholesky G = L L^T and G^{-1} = L^{-T} L^{-1}; false if G is not SPD.
static bool spd_inverse(int p, const std::vector<double> &G, std::vector<double> &Ginv) {
    std::vector<double> L(p * p, 0.0), Li(p * p, 0.0);
    for (int i = 0; i < p; ++i)
        for (int j = 0; j <= i; ++j) {
            double t = G[i * p + j];
            for (int k = 0; k < j; ++k) t -= L[i * p + k] * L[j * p + k];
            if (i == j) {
                if (!(t > 0.0) || !std::isfinite(t)) return false;
                L[i * p + i] = std::sqrt(t);
            } else {
                L[i * p + j] = t / L[j * p + j];
            }
        }
    for (int c = 0; c < p; ++c)  // Li = L^{-1}, column by column (forward substitution)
        for (int i = 0; i < p; ++i) {
            double t = (i == c) ? 1.0 : 0.0;
            for (int k = 0; k < i; ++k) t -= L[i * p + k] * Li[k * p + c];
            Li[i * p + c] = t / L[i * p + i];
        }
    Ginv.assign(p * p, 0.0);
    for (int a = 0; a < p; ++a)
        for (int b = 0; b < p; ++b) {
            double t = 0.0;
            for (int k = 0; k < p; ++k) t += Li[k * p + a] * Li[k * p + b];
            Ginv[a * p + b] = t;
        }
    return true;
}

npc_status set_lowrank(npc_poly P, int p, const double *V_ext) {
    Operator *op = P->op->op.get();
    Context *ctx = op->ctx;
    const int n = op->n_local;
    const size_t nn = std::max(n, 1);
    P->pcg.invalidate();  // the captured PCG iteration bakes in the preconditioner
    P->lr_p = 0;
    P->lr_V.release();
    P->lr_Ginv.release();
    P->lr_scratch.release();
    if (p == 0) return NPC_SUCCESS;
    NPC_TRY(P->lr_V.alloc(sizeof(double) * nn * p));
    double *V = P->lr_V.as<double>();
    for (int j = 0; j < p; ++j) {
        if (op->permuted())
            NPC_TRY(op->to_internal(V_ext + (size_t)j * n, V + j * nn));
        else if (n)
            NPC_CUDA_TRY(cudaMemcpyAsync(V + j * nn, V_ext + (size_t)j * n, sizeof(double) * n,
                                         cudaMemcpyDeviceToDevice, ctx->stream));
    }
    const int G = vec_grid(n);
    // scratch: partials (p x G) | sums (p) | c (p)
    NPC_TRY(P->lr_scratch.alloc(sizeof(double) * ((size_t)p * G + 2 * NPC_LOWRANK_MAX)));
    double *part = P->lr_scratch.as<double>(), *sums = part + (size_t)p * G;
    // G = V^T A V, column b at a time: t = A v_b, then V^T t
    DevBuf t;
    NPC_TRY(t.alloc(sizeof(double) * nn));
    std::vector<double> Gh(p * p), col(p);
    for (int b = 0; b < p; ++b) {
        StepArgs s;
        s.x = V + b * nn;
        s.out = t.as<double>();
        s.a = 1.0;
        {
            TimedScope ts(ctx, T_OPERATOR);
            NPC_TRY(op->step(s));
        }
        NPC_TRY(multidot(ctx, V, nn, p, t.as<double>(), n, part, sums, nullptr));
        NPC_CUDA_TRY(cudaMemcpyAsync(col.data(), sums, sizeof(double) * p, cudaMemcpyDeviceToHost, ctx->stream));
        NPC_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
        for (int a = 0; a < p; ++a) Gh[a * p + b] = col[a];
    }
    for (int a = 0; a < p; ++a)  // symmetrise the rounding
        for (int b = 0; b < a; ++b) Gh[a * p + b] = Gh[b * p + a] = 0.5 * (Gh[a * p + b] + Gh[b * p + a]);
    std::vector<double> Ginv;
    if (!spd_inverse(p, Gh, Ginv)) {
        set_error("set_lowrank: V^T A V is not SPD (V rank-deficient or A not SPD)");
        P->lr_V.release();
        P->lr_scratch.release();
        return NPC_ERR_BREAKDOWN;
    }
    NPC_TRY(P->lr_Ginv.alloc(sizeof(double) * p * p));
    NPC_CUDA_TRY(cudaMemcpyAsync(P->lr_Ginv.p, Ginv.data(), sizeof(double) * p * p, cudaMemcpyHostToDevice,
                                 ctx->stream));
    NPC_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    P->lr_p = p;
    return NPC_SUCCESS;
}

// Before p_k: s = V^T r, c = G^{-1} s (device scalars in lr_scratch).
npc_status lowrank_pre(npc_poly P, const double *r, const int *done) {
    Operator *op = P->op->op.get();
    Context *ctx = op->ctx;
    const int n = op->n_local, p = P->lr_p, G = vec_grid(n);
    double *part = P->lr_scratch.as<double>(), *sums = part + (size_t)p * G, *c = sums + NPC_LOWRANK_MAX;
    TimedScope ts(ctx, T_VECTOR);
    NPC_TRY(multidot(ctx, P->lr_V.as<double>(), std::max(n, 1), p, r, n, part, sums, done));
    k_lr_coef<<<1, 1, 0, ctx->stream>>>(P->lr_Ginv.as<double>(), p, sums, c, done);
    NPC_LAUNCH_CHECK();
    return NPC_SUCCESS;
}

// After p_k: z += V c (+ partials of <z, dotv>).
npc_status lowrank_post(npc_poly P, double *z, const double *dotv, double *partials, int *nparts, const int *done) {
    Operator *op = P->op->op.get();
    Context *ctx = op->ctx;
    const int n = op->n_local, p = P->lr_p, G = vec_grid(n);
    const double *c = P->lr_scratch.as<double>() + (size_t)p * G + NPC_LOWRANK_MAX;
    TimedScope ts(ctx, T_VECTOR);
    if (dotv) {
        if (nparts) *nparts = G;
        k_lr_correct<true><<<G, LR_T, 0, ctx->stream>>>(z, P->lr_V.as<double>(), std::max(n, 1), p, c, n, dotv,
                                                         partials, done);
    } else {
        k_lr_correct<false><<<G, LR_T, 0, ctx->stream>>>(z, P->lr_V.as<double>(), std::max(n, 1), p, c, n,
                                                          nullptr, nullptr, done);
    }
    NPC_LAUNCH_CHECK();
    return NPC_SUCCESS;
}

// Sturm bisection / inverse iteration helpers live in solvers.cu
double tridiag_eigenvalue(const std::vector<double> &a, const std::vector<double> &b, int idx);
void tridiag_inverse_iteration(const std::vector<double> &a, const std::vector<double> &b, double mu,
                               std::vector<double> &x);

npc_status ritz_vectors(Operator *op, int m, int p, const double *v0_ext, double *V_ext, double *theta) {
    Context *ctx = op->ctx;
    const int n = op->n_local;
    const size_t nn = std::max(n, 1);
    DevBuf Qb, wb, sc;
    NPC_TRY(Qb.alloc(sizeof(double) * nn * (m + 1)));
    NPC_TRY(wb.alloc(sizeof(double) * nn));
    double *Q = Qb.as<double>(), *w = wb.as<double>();
    const int G = vec_grid(n);
    NPC_TRY(sc.alloc(sizeof(double) * ((size_t)NPC_LOWRANK_MAX * G + 4 * NPC_LOWRANK_MAX + (size_t)m * p)));
    double *part = sc.as<double>(), *sums = part + (size_t)NPC_LOWRANK_MAX * G, *hbuf = sums + NPC_LOWRANK_MAX;
    double *Sdev = hbuf + 2 * NPC_LOWRANK_MAX;
    // q_0 = v0 / ||v0||
    if (v0_ext) {
        if (op->permuted())
            NPC_TRY(op->to_internal(v0_ext, w));
        else if (n)
            NPC_CUDA_TRY(cudaMemcpyAsync(w, v0_ext, sizeof(double) * n, cudaMemcpyDeviceToDevice, ctx->stream));
    } else {
        NPC_TRY(launch_hash_vector(ctx, Q, n, op->row_begin, 0x5EEDull));
        if (op->permuted())
            NPC_TRY(op->to_internal(Q, w));
        else if (n)
            NPC_CUDA_TRY(cudaMemcpyAsync(w, Q, sizeof(double) * n, cudaMemcpyDeviceToDevice, ctx->stream));
    }
    auto norm2 = [&](const double *x, double *out) -> npc_status {
        NPC_TRY(multidot(ctx, x, nn, 1, x, n, part, sums, nullptr));
        NPC_CUDA_TRY(cudaMemcpyAsync(out, sums, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
        NPC_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
        return NPC_SUCCESS;
    };
    double vn2;
    NPC_TRY(norm2(w, &vn2));
    if (!(vn2 > 0.0)) {
        set_error("ritz_vectors: start vector is zero");
        return NPC_ERR_INVALID_ARGUMENT;
    }
    NPC_TRY(launch_scale(ctx, w, Q, 1.0 / std::sqrt(vn2), n, nullptr, nullptr, nullptr, nullptr));
    std::vector<double> alpha, beta;
    int steps = 0;
    for (int j = 0; j < m; ++j) {
        double *q = Q + j * nn;
        StepArgs s;
        s.x = q;
        s.out = w;
        s.a = 1.0;
        {
            TimedScope ts(ctx, T_OPERATOR);
            NPC_TRY(op->step(s));
        }
        double aj;
        NPC_TRY(multidot(ctx, q, nn, 1, w, n, part, sums, nullptr));
        NPC_CUDA_TRY(cudaMemcpyAsync(&aj, sums, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
        // classical Gram-Schmidt against q_0..q_j, twice, in chunks of NPC_LOWRANK_MAX vectors
        for (int pass = 0; pass < 2; ++pass)
            for (int l0 = 0; l0 <= j; l0 += NPC_LOWRANK_MAX) {
                const int cnt = std::min(NPC_LOWRANK_MAX, j + 1 - l0);
                NPC_TRY(multidot(ctx, Q + l0 * nn, nn, cnt, w, n, part, sums, nullptr));
                if (n) {
                    k_gs_update<<<G, LR_T, 0, ctx->stream>>>(w, Q + l0 * nn, nn, cnt, sums, n);
                    NPC_LAUNCH_CHECK();
                }
            }
        double b2;
        NPC_TRY(norm2(w, &b2));
        const double bj = std::sqrt(std::max(b2, 0.0));
        alpha.push_back(aj);
        beta.push_back(bj);
        steps = j + 1;
        if (!(bj > 0.0)) break;
        NPC_TRY(launch_scale(ctx, w, Q + (j + 1) * nn, 1.0 / bj, n, nullptr, nullptr, nullptr, nullptr));
    }
    if (p > steps) {
        set_error("ritz_vectors: Lanczos stopped after %d steps (< p = %d): invariant subspace", steps, p);
        return NPC_ERR_BREAKDOWN;
    }
    // p smallest eigenpairs of T_steps (Sturm bisection, inverse iteration)
    std::vector<double> ta(alpha.begin(), alpha.begin() + steps), tb(beta.begin(), beta.begin() + steps - 1);
    std::vector<double> S((size_t)steps * p);
    for (int l = 0; l < p; ++l) {
        const double th = tridiag_eigenvalue(ta, tb, l);
        theta[l] = th;
        std::vector<double> x(steps);
        for (int i = 0; i < steps; ++i) x[i] = 1.0 + 0.01 * ((i * 7 + l * 3) % 11);  // generic start
        for (int it = 0; it < 4; ++it) {
            // deflate the eigenvectors already found (clustered Ritz values)
            for (int k = 0; k < l; ++k) {
                double h = 0.0;
                for (int i = 0; i < steps; ++i) h += S[(size_t)i * p + k] * x[i];
                for (int i = 0; i < steps; ++i) x[i] -= h * S[(size_t)i * p + k];
            }
            tridiag_inverse_iteration(ta, tb, th, x);
            double nrm = 0.0;
            for (double v : x) nrm += v * v;
            nrm = std::sqrt(nrm);
            if (!(nrm > 0.0) || !std::isfinite(nrm)) {
                set_error("ritz_vectors: inverse iteration failed for Ritz value %d", l);
                return NPC_ERR_BREAKDOWN;
            }
            for (double &v : x) v /= nrm;
        }
        for (int i = 0; i < steps; ++i) S[(size_t)i * p + l] = x[i];
    }
    NPC_CUDA_TRY(cudaMemcpyAsync(Sdev, S.data(), sizeof(double) * S.size(), cudaMemcpyHostToDevice, ctx->stream));
    // V = Q S in internal order (reuse the tail of Q's buffer is not safe; use a fresh one)
    DevBuf Vi;
    NPC_TRY(Vi.alloc(sizeof(double) * nn * p));
    if (n) {
        k_basis_combine<<<G, LR_T, 0, ctx->stream>>>(Q, nn, steps, Sdev, p, Vi.as<double>(), nn, n);
        NPC_LAUNCH_CHECK();
    }
    for (int l = 0; l < p; ++l) {
        if (op->permuted())
            NPC_TRY(op->to_external(Vi.as<double>() + l * nn, V_ext + (size_t)l * n));
        else if (n)
            NPC_CUDA_TRY(cudaMemcpyAsync(V_ext + (size_t)l * n, Vi.as<double>() + l * nn, sizeof(double) * n,
                                         cudaMemcpyDeviceToDevice, ctx->stream));
    }
    NPC_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    if (ctx->timing) ctx->t_flush();
    return NPC_SUCCESS;
}

}  // namespace npc
