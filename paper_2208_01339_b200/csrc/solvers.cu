// solvers.cu -- drivers on top of the fused operator steps:
//   * poly_coefficients / apply_poly: Alg. 2 with theta_bar (Eq. thetamod)
//     rewritten as one fused step per degree, s_j = a_j A s_{j-1} + b_j s_{j-1} + c_j s_{j-2}
//     + d_j r, in place over s_{j-2};
//   * pcg: single-reduction (Chronopoulos-Gear) PCG with the inner products fused into the
//     kernels that produce the vectors and device-resident scalars;
//   * lanczos: the spectrum estimate + Sturm bisection on the host.
#include <math.h>

#include <algorithm>
#include <chrono>

#include "device_util.cuh"
#include "npc_internal.cuh"

namespace npc {

// ================================================================== context helpers
npc_status Context::ensure_partials(size_t n) {
    if (n <= partial_cap) return NPC_SUCCESS;
    size_t cap = std::max<size_t>(n, 4096);
    NPC_TRY(partials.alloc(sizeof(double) * cap * 4));
    partial_cap = cap;
    return NPC_SUCCESS;
}

npc_status Context::allreduce_sum(double *dev, int count) {
    if (!distributed()) return NPC_SUCCESS;
    TimedScope ts(this, T_REDUCE);
    return tr->allreduce_sum(this, dev, count, stream);
}

// While a PCG iteration is being stream-captured (timing on), the events become event-record
// nodes of the graph (cudaEventRecordExternal) and are collected in `captured`: the graph owns
// them and every replay re-records them, so the solver reads them after each replay.
static void record_timing_event(Context *c, cudaEvent_t e) {
    if (c->capturing)
        cudaEventRecordWithFlags(e, c->stream, cudaEventRecordExternal);
    else
        cudaEventRecord(e, c->stream);
}

int Context::t_begin(int cls, int count) {
    cudaEvent_t e0;
    if (capturing || ev_free.empty()) {
        if (cudaEventCreate(&e0) != cudaSuccess) return -1;
    } else {
        e0 = ev_free.back();
        ev_free.pop_back();
    }
    record_timing_event(this, e0);
    auto &list = capturing ? captured : pending;
    list.push_back({cls, e0, nullptr, count});
    return (capturing ? (1 << 30) : 0) + (int)list.size() - 1;
}

void Context::t_end(int idx) {
    cudaEvent_t e1;
    if (capturing || ev_free.empty()) {
        if (cudaEventCreate(&e1) != cudaSuccess) return;
    } else {
        e1 = ev_free.back();
        ev_free.pop_back();
    }
    record_timing_event(this, e1);
    if (idx >= (1 << 30))
        captured[idx - (1 << 30)].e1 = e1;
    else
        pending[idx].e1 = e1;
}

// Accumulate the intervals of a replayed graph's timing events (the replay has completed).
void Context::t_flush_graph(const std::vector<Pending> &ev) {
    for (const auto &p : ev) {
        float ms = 0.f;
        if (p.e1 && cudaEventElapsedTime(&ms, p.e0, p.e1) == cudaSuccess) {
            t_ms[p.cls] += ms;
            t_cnt[p.cls] += p.count;
        }
    }
}

void Context::t_flush() {
    for (auto &p : pending) {
        if (p.e1) {
            float ms = 0.f;
            cudaEventSynchronize(p.e1);
            if (cudaEventElapsedTime(&ms, p.e0, p.e1) == cudaSuccess) {
                t_ms[p.cls] += ms;
                t_cnt[p.cls] += p.count;
            }
            ev_free.push_back(p.e1);
        }
        ev_free.push_back(p.e0);
    }
    pending.clear();
}

Context::~Context() {
    if (graph_stream) cudaStreamDestroy(graph_stream);
    if (body_stream) cudaStreamDestroy(body_stream);
    if (ev_fork) cudaEventDestroy(ev_fork);
    if (ev_join) cudaEventDestroy(ev_join);
    if (ev_rr0) cudaEventDestroy(ev_rr0);
    if (ev_rr1) cudaEventDestroy(ev_rr1);
    for (auto &p : pending) {
        cudaEventDestroy(p.e0);
        if (p.e1) cudaEventDestroy(p.e1);
    }
    for (auto e : ev_free) cudaEventDestroy(e);
}

// ================================================================== coefficients (host)
// theta = (beta + alpha)/2, delta = (beta - alpha)/2, theta_bar =
// theta (1 + xi) (Eq. thetamod; delta unchanged, reading A1), sigma =
// theta_bar/delta, rho_0 = 1/sigma, rho_j = 1/(2 sigma - rho_{j-1}) (Eq. rhocheb).  From the
// three-term form s_j = rho_j (2 sigma s_{j-1} - rho_{j-1} s_{j-2} + (2/delta)(r - A s_{j-1}))
// (PAPER.md:262-266):  a_j = -2 rho_j/delta, b_j = 2 sigma rho_j, c_j = -rho_j rho_{j-1},
// d_j = 2 rho_j/delta.
npc_status poly_coefficients(int k, double lmin, double lmax, double xi, double *theta_bar, double *delta,
                             double *sigma, double *coef) {
    if (k < 0 || !(xi >= 0.0) || !std::isfinite(xi) || !(lmin > 0.0) || !std::isfinite(lmax) || lmax < lmin) {
        set_error("set_poly: need degree >= 0, xi >= 0, 0 < lmin <= lmax (got k=%d, [%g, %g], xi=%g)", k, lmin, lmax, xi);
        return NPC_ERR_INVALID_ARGUMENT;
    }
    const double theta = 0.5 * (lmax + lmin);
    const double dl = 0.5 * (lmax - lmin);
    if (!(dl > 0.0)) {
        set_error("set_poly: degenerate interval lmin == lmax (delta = 0)");
        return NPC_ERR_DEGENERATE_INTERVAL;
    }
    const double tb = theta * (1.0 + xi);
    const double sg = tb / dl;
    *theta_bar = tb;
    *delta = dl;
    *sigma = sg;
    double rho_prev = 1.0 / sg;
    for (int j = 1; j <= k; ++j) {
        const double rho = 1.0 / (2.0 * sg - rho_prev);
        if (coef) {
            coef[4 * (j - 1) + 0] = -2.0 * rho / dl;
            coef[4 * (j - 1) + 1] = 2.0 * sg * rho;
            coef[4 * (j - 1) + 2] = -rho * rho_prev;
            coef[4 * (j - 1) + 3] = 2.0 * rho / dl;
        }
        rho_prev = rho;
    }
    return NPC_SUCCESS;
}

// ================================================================== p_k(A) r
// Internal-order application.  Buffers: z and tmp alternate so that s_k lands in z; s_j is
// written over s_{j-2}.  j = 1 folds s_0 = r/theta_bar into the coefficients (reads only r),
// j = 2 folds c_2 s_0 into the r term (no s_{j-2} read).  With dotv != null the last kernel
// emits partials of <z, dotv> into 'partials' (count returned in *nparts).
// ================================================================== Newton (Alg. 1)
// zeta_0 = 1/theta_bar; zeta_1 = 2/(1 + 2 a' zeta_0 - (a' zeta_0)^2) with a' = theta_bar - delta
// (reading A1: Newton on the interval shifted by xi*theta); zeta_i = 2/(1 + 2 zeta_{i-1} -
// zeta_{i-1}^2) (Eq. zetaNewt).  P_0 r = zeta_0 r, P_{j+1} r = zeta_{j+1}
// (2 P_j r - P_j A P_j r) (Alg. 1 step 4): 2^nlev - 1 applications of A.
npc_status newton_zetas(int nlev, double lmin, double lmax, double xi, std::vector<double> &zeta) {
    double tb, dl, sg;
    NPC_TRY(poly_coefficients(0, lmin, lmax, xi, &tb, &dl, &sg, nullptr));
    const double ap = tb - dl;
    zeta.assign(nlev + 1, 0.0);
    zeta[0] = 1.0 / tb;
    if (nlev >= 1) zeta[1] = 2.0 / (1.0 + 2.0 * ap * zeta[0] - (ap * zeta[0]) * (ap * zeta[0]));
    for (int i = 2; i <= nlev; ++i) zeta[i] = 2.0 / (1.0 + 2.0 * zeta[i - 1] - zeta[i - 1] * zeta[i - 1]);
    return NPC_SUCCESS;
}

// out = zeta (2 t1 - out)  (+ partial <out, dotv>)
template <bool DOT>
__global__ void __launch_bounds__(256) k_newton_combine(double *out, const double *__restrict__ t1, double zeta,
                                                        int n, const double *__restrict__ dotv, double *partials,
                                                        const int *done) {
    if (done && *done) return;
    __shared__ double red[8];
    double acc = 0.0;
    for (int i = blockIdx.x * 256 + threadIdx.x; i < n; i += gridDim.x * 256) {
        const double o = zeta * (2.0 * t1[i] - out[i]);
        out[i] = o;
        if (DOT) acc += o * dotv[i];
    }
    if (DOT) {
        acc = block_sum<256>(acc, red);
        if (threadIdx.x == 0) partials[blockIdx.x] = acc;
    }
}

static npc_status newton_level(npc_poly P, int j, const double *in, double *out, const double *dotv,
                               double *partials, int *nparts, const int *done) {
    Operator *op = P->op->op.get();
    Context *ctx = op->ctx;
    const std::vector<double> &z = P->zeta;
    if (j == 0) {
        TimedScope ts(ctx, T_DEGREE);
        return launch_scale(ctx, in, out, z[0], op->n_local, dotv, partials, nparts, done);
    }
    if (j == 1) {  // P_1 in = zeta_1 (2 zeta_0 in - zeta_0^2 A in): one fused step
        StepArgs s;
        s.x = in;
        s.out = out;
        s.a = -z[1] * z[0] * z[0];
        s.b = 2.0 * z[1] * z[0];
        s.done = done;
        if (dotv) {
            s.dotv = dotv;
            s.partials = partials;
            if (nparts) *nparts = op->num_partials();
        }
        TimedScope ts(ctx, T_DEGREE);
        return op->step(s);
    }
    const size_t nn = std::max(op->n_local, 1);
    double *t1 = P->nbuf.as<double>() + (size_t)2 * (j - 2) * nn, *t2 = t1 + nn;
    NPC_TRY(newton_level(P, j - 1, in, t1, nullptr, nullptr, nullptr, done));
    {
        StepArgs s;  // t2 = A t1
        s.x = t1;
        s.out = t2;
        s.a = 1.0;
        s.done = done;
        TimedScope ts(ctx, T_DEGREE);
        NPC_TRY(op->step(s));
    }
    NPC_TRY(newton_level(P, j - 1, t2, out, nullptr, nullptr, nullptr, done));
    const int g = vec_grid(op->n_local);
    TimedScope ts(ctx, T_VECTOR);
    if (dotv) {
        if (nparts) *nparts = g;
        k_newton_combine<true><<<g, 256, 0, ctx->stream>>>(out, t1, z[j], op->n_local, dotv, partials, done);
    } else {
        k_newton_combine<false><<<g, 256, 0, ctx->stream>>>(out, t1, z[j], op->n_local, nullptr, nullptr, done);
    }
    NPC_LAUNCH_CHECK();
    return NPC_SUCCESS;
}

static npc_status apply_poly_core(npc_poly P, const double *r, double *z, const double *dotv, double *partials,
                                  int *nparts, const int *done);

// z = P r with P = p_k(A) (+ V (V^T A V)^{-1} V^T when a low-rank correction is set); the
// partials of <z, dotv> come from the last kernel that writes z.
npc_status apply_poly_internal(npc_poly P, const double *r, double *z, const double *dotv, double *partials,
                               int *nparts, const int *done) {
    // timing: ONE event pair around the k degree launches (credited as k launches) -- per-launch
    // events inside a graph replay perturb short kernels by several microseconds each
    Context *ctx = P->op->op->ctx;
    TimedScope ts(ctx, T_DEGREE, std::max(P->degree, 1));
    TimingGroup grp(ctx);
    if (P->lr_p == 0) return apply_poly_core(P, r, z, dotv, partials, nparts, done);
    NPC_TRY(lowrank_pre(P, r, done));
    NPC_TRY(apply_poly_core(P, r, z, nullptr, nullptr, nullptr, done));
    return lowrank_post(P, z, dotv, partials, nparts, done);
}

static npc_status apply_poly_core(npc_poly P, const double *r, double *z, const double *dotv, double *partials,
                                  int *nparts, const int *done) {
    if (P->kind == 1) return newton_level(P, P->nlev, r, z, dotv, partials, nparts, done);
    Operator *op = P->op->op.get();
    Context *ctx = op->ctx;
    const int k = P->degree;
    const double tb = P->theta_bar;
    if (k == 0) {
        TimedScope ts(ctx, T_DEGREE);
        return launch_scale(ctx, r, z, 1.0 / tb, op->n_local, dotv, partials, nparts, done);
    }
    double *tmp = P->tmp.as<double>();
    if (op->supports_fused_poly() && P->coef_dev.p) {  // all k degrees in one cluster launch
        TimedScope ts(ctx, T_DEGREE);
        return op->apply_poly_fused(r, z, P->coef_dev.as<double>(), k, tb, dotv, partials, nparts, done);
    }
    if (k >= 4 && op->supports_step2() && P->tmp2.p) {
        // Temporal blocking: degrees 1, 2 single, then pairs (j, j+1) in one pass, a single tail
        // step if k is odd.  A pair's outputs must not alias its inputs (neighbouring tiles still
        // read them), so four buffers rotate; labels are assigned forward and renamed at the end
        // so that s_k lands in z.
        struct Act {
            int j, pair, in1, in2, o1, o2;
        };
        std::vector<Act> plan;
        int cur = 0, prev = -1;  // labels of s_{j-1}, s_{j-2}
        plan.push_back({1, 0, -1, -1, 0, -1});
        plan.push_back({2, 0, 0, -1, 1, -1});
        prev = 0;
        cur = 1;
        int j = 3;
        for (; j + 1 <= k; j += 2) {
            int o[2], c = 0;
            for (int l = 0; l < 4 && c < 2; ++l)
                if (l != cur && l != prev) o[c++] = l;
            plan.push_back({j, 1, cur, prev, o[0], o[1]});
            prev = o[0];
            cur = o[1];
        }
        if (j == k) {
            plan.push_back({k, 0, cur, prev, prev, -1});
            prev = cur;
            cur = plan.back().o1;
        }
        double *phys[4];
        const size_t nn = std::max(op->n_local, 1);
        double *spare[3] = {tmp, P->tmp2.as<double>(), P->tmp2.as<double>() + nn};
        for (int l = 0, q = 0; l < 4; ++l) phys[l] = (l == cur) ? z : spare[q++];
        auto coefs = [&](int jj, StepArgs &st) {
            const double *cf = &P->coef[4 * (jj - 1)];
            st.a = cf[0];
            st.b = cf[1];
            st.c = cf[2];
            st.d = cf[3];
        };
        for (const Act &a : plan) {
            const bool last = a.pair ? (a.j + 1 == k) : (a.j == k);
            if (!a.pair) {
                StepArgs st;
                st.done = done;
                st.out = phys[a.o1];
                const double *cf = &P->coef[4 * (a.j - 1)];
                if (a.j == 1) {
                    st.x = r;
                    st.a = cf[0] / tb;
                    st.b = cf[1] / tb + cf[3];
                } else if (a.j == 2) {
                    st.x = phys[a.in1];
                    st.r = r;
                    st.a = cf[0];
                    st.b = cf[1];
                    st.d = cf[2] / tb + cf[3];
                } else {
                    st.x = phys[a.in1];
                    st.s2 = phys[a.in2];
                    st.r = r;
                    coefs(a.j, st);
                }
                if (last && dotv) {
                    st.dotv = dotv;
                    st.partials = partials;
                    if (nparts) *nparts = op->num_partials();
                }
                TimedScope ts(ctx, T_DEGREE);
                NPC_TRY(op->step(st));
            } else {
                StepArgs s1, s2;
                s1.done = s2.done = done;
                s1.x = phys[a.in1];
                s1.s2 = phys[a.in2];
                s1.r = s2.r = r;
                s1.out = phys[a.o1];
                s2.out = phys[a.o2];
                coefs(a.j, s1);
                coefs(a.j + 1, s2);
                if (last && dotv) {
                    s2.dotv = dotv;
                    s2.partials = partials;
                    if (nparts) *nparts = op->num_partials2();
                }
                TimedScope ts(ctx, T_DEGREE);
                NPC_TRY(op->step2(s1, s2));
            }
        }
        return NPC_SUCCESS;
    }
    auto buf = [&](int j) { return ((k - j) % 2 == 0) ? z : tmp; };
    for (int j = 1; j <= k; ++j) {
        const double *cf = &P->coef[4 * (j - 1)];
        StepArgs s;
        s.done = done;
        s.out = buf(j);
        if (j == 1) {
            s.x = r;
            s.a = cf[0] / tb;
            s.b = cf[1] / tb + cf[3];
        } else if (j == 2) {
            s.x = buf(1);
            s.r = r;
            s.a = cf[0];
            s.b = cf[1];
            s.d = cf[2] / tb + cf[3];
        } else {
            s.x = buf(j - 1);
            s.s2 = buf(j);
            s.r = r;
            s.a = cf[0];
            s.b = cf[1];
            s.c = cf[2];
            s.d = cf[3];
        }
        if (j == k && dotv) {
            s.dotv = dotv;
            s.partials = partials;
            if (nparts) *nparts = op->num_partials();
        }
        TimedScope ts(ctx, T_DEGREE);
        NPC_TRY(op->step(s));
    }
    return NPC_SUCCESS;
}

npc_status apply_poly(npc_poly P, const double *r, double *z) {
    Operator *op = P->op->op.get();
    if (!op->permuted()) return apply_poly_internal(P, r, z, nullptr, nullptr, nullptr, nullptr);
    NPC_TRY(op->to_internal(r, P->rin.as<double>()));
    NPC_TRY(apply_poly_internal(P, P->rin.as<double>(), P->zout.as<double>(), nullptr, nullptr, nullptr, nullptr));
    return op->to_external(P->zout.as<double>(), z);
}

npc_status apply_operator(Operator *op, const double *x, double *y, DevBuf &scratch) {
    StepArgs s;
    s.a = 1.0;
    if (!op->permuted()) {
        s.x = x;
        s.out = y;
        TimedScope ts(op->ctx, T_OPERATOR);
        return op->step(s);
    }
    NPC_TRY(scratch.alloc(sizeof(double) * 2 * std::max(op->n_local, 1)));
    double *xi = scratch.as<double>(), *yi = xi + std::max(op->n_local, 1);
    NPC_TRY(op->to_internal(x, xi));
    s.x = xi;
    s.out = yi;
    {
        TimedScope ts(op->ctx, T_OPERATOR);
        NPC_TRY(op->step(s));
    }
    return op->to_external(yi, y);
}

// ================================================================== PCG
struct CgDev {
    double gamma, gamma_old, delta, alpha, alpha_old, beta;
    double rr, bnorm2, tol2;
    int done, iters, maxit, breakdown, converged, first, multi, pad;
};

// sums[0] = <r, u> (gamma), sums[1] = <u, A u> (delta) -- the one allreduce of the iteration.
// (Distributed contexts reduce ||r_{i+1}||^2 separately, overlapped with the next p_k(A) r:
// k_cg_rrcheck.)  multi == 2 is the north star's single fused allreduce:
// sums[2] = ||r_i||^2 of the previous update rode in the same allreduce, and the exit check
// happens here, one (k+1)-application block late.
__global__ void k_cg_scalars(CgDev *st, const double *sums, double *history) {
    if (st->done) return;
    if (st->multi == 2) {
        const double t = sums[2];
        st->rr = t;
        if (history) history[st->iters] = sqrt(t / st->bnorm2);
        if (t <= st->tol2) {
            st->converged = 1;
            st->done = 1;
            return;
        }
        if (st->iters >= st->maxit) {
            st->done = 1;
            return;
        }
    }
    const double g = sums[0], dl = sums[1];
    if (!(g > 0.0)) {
        st->breakdown = 1;
        st->done = 1;
        return;
    }
    double beta = 0.0, denom = dl;
    if (!st->first) {
        beta = g / st->gamma_old;
        denom = dl - beta * g / st->alpha_old;
    }
    if (!(denom > 0.0)) {
        st->breakdown = 2;
        st->done = 1;
        return;
    }
    const double alpha = g / denom;
    st->gamma = g;
    st->delta = dl;
    st->beta = beta;
    st->alpha = alpha;
    st->gamma_old = g;
    st->alpha_old = alpha;
    st->first = 0;
}

// p = u + beta p; s = w + beta s; x += alpha p; r -= alpha s; partial ||r||^2.
__global__ void __launch_bounds__(256) k_cg_update(const CgDev *st, const double *__restrict__ u,
                                                   const double *__restrict__ w, double *__restrict__ p,
                                                   double *__restrict__ s, double *__restrict__ x,
                                                   double *__restrict__ r, int n, double *partials) {
    if (st->done) return;
    __shared__ double red[8];
    const double alpha = st->alpha, beta = st->beta;
    double acc = 0.0;
    // p, s and x are touched only here, once per iteration: streaming (evict-first) accesses
    // keep them from displacing r, u, w and the polynomial's ping-pong vector in L2, which
    // matters when those fit and the whole PCG working set does not (config 2: 8 x 16.8 MB).
    for (int i = blockIdx.x * 256 + threadIdx.x; i < n; i += gridDim.x * 256) {
#ifndef NPC_CG_NOCS
        const double pi = u[i] + beta * __ldcs(p + i);
        const double si = w[i] + beta * __ldcs(s + i);
        __stcs(p + i, pi);
        __stcs(s + i, si);
        __stcs(x + i, __ldcs(x + i) + alpha * pi);
#else
        const double pi = u[i] + beta * p[i];
        const double si = w[i] + beta * s[i];
        p[i] = pi;
        s[i] = si;
        x[i] += alpha * pi;
#endif
        const double ri = r[i] - alpha * si;
        r[i] = ri;
        acc += ri * ri;
    }
    acc = block_sum<256>(acc, red);
    if (threadIdx.x == 0) partials[blockIdx.x] = acc;
}

__global__ void __launch_bounds__(1024) k_cg_rr(CgDev *st, const double *__restrict__ partials, int np,
                                                double *sums, double *history) {
    if (st->done) return;
    __shared__ double red[32];
    double t = 0.0;
    for (int i = threadIdx.x; i < np; i += 1024) t += partials[i];
    t = block_sum<1024>(t, red);
    if (threadIdx.x == 0) {
        st->iters += 1;
        // multi 1: the local partial, allreduced on the side stream; multi 2: the local partial
        // rides in the next iteration's fused allreduce
        sums[st->multi == 1 ? 4 : 2] = t;
        if (!st->multi) {
            st->rr = t;
            if (history) history[st->iters] = sqrt(t / st->bnorm2);
            if (t <= st->tol2) {
                st->converged = 1;
                st->done = 1;
            } else if (st->iters >= st->maxit) {
                st->done = 1;
            }
        }
    }
}

// Distributed contexts: the global ||r_i||^2 arrives from an allreduce on
// the side stream that overlaps the next p_k(A) r; on convergence the flag is raised while
// that application is in flight, so its remaining degree kernels and w = A u no-op (the
// discarded work is about one allreduce latency, not a whole (k+1)-application block).
__global__ void k_cg_rrcheck(CgDev *st, const double *rr_glob, double *history) {
    if (st->done) return;
    const double t = *rr_glob;
    st->rr = t;
    if (history) history[st->iters] = sqrt(t / st->bnorm2);
    if (t <= st->tol2) {
        st->converged = 1;
        st->done = 1;
    } else if (st->iters >= st->maxit) {
        st->done = 1;
    }
}

// Sets an IF node's condition: run the next PCG iteration only while the device flag is clear.
__global__ void k_set_cond_not_done(cudaGraphConditionalHandle h, const int *done) {
    cudaGraphSetConditional(h, *done ? 0u : 1u);
}

// Stream-captured replay of a fixed work block.  While active, ctx->stream points at the
// library's graph stream (forked from the caller's stream); the destructor joins back.
struct GraphRun {
    static constexpr int ITERS = 4;
    Context *c;
    PcgCache &cache;
    cudaStream_t orig;
    cudaGraphExec_t exec = nullptr;  // owned by the cache
    unsigned long long kernels = 0;
    bool forked = false;
    GraphRun(Context *ctx, PcgCache &pc) : c(ctx), cache(pc), orig(ctx->stream) {}
    // One iteration as the body of a conditional (IF) node: a solve that converges inside a
    // replayed block skips the block's remaining iterations instead of launching them as no-ops
    template <class F>
    npc_status cond_iteration(F &&body, const int *done) {
        cudaStreamCaptureStatus cs;
        cudaGraph_t cg = nullptr;
        const cudaGraphNode_t *deps = nullptr;
        size_t nd = 0;
        NPC_CUDA_TRY(cudaStreamGetCaptureInfo(c->stream, &cs, nullptr, &cg, &deps, &nd));
        cudaGraphConditionalHandle h;
        NPC_CUDA_TRY(cudaGraphConditionalHandleCreate(&h, cg, 0, cudaGraphCondAssignDefault));
        k_set_cond_not_done<<<1, 1, 0, c->stream>>>(h, done);
        NPC_LAUNCH_CHECK();
        NPC_CUDA_TRY(cudaStreamGetCaptureInfo(c->stream, &cs, nullptr, &cg, &deps, &nd));
        cudaGraphNodeParams p = {};
        p.type = cudaGraphNodeTypeConditional;
        p.conditional.handle = h;
        p.conditional.type = cudaGraphCondTypeIf;
        p.conditional.size = 1;
        cudaGraphNode_t node;
        NPC_CUDA_TRY(cudaGraphAddNode(&node, cg, deps, nd, &p));
        NPC_CUDA_TRY(cudaStreamUpdateCaptureDependencies(c->stream, &node, 1, cudaStreamSetCaptureDependencies));
        if (!c->body_stream) NPC_CUDA_TRY(cudaStreamCreateWithFlags(&c->body_stream, cudaStreamNonBlocking));
        cudaStream_t parent = c->stream;
        NPC_CUDA_TRY(cudaStreamBeginCaptureToGraph(c->body_stream, p.conditional.phGraph_out[0], nullptr, nullptr, 0,
                                                   cudaStreamCaptureModeThreadLocal));
        c->stream = c->body_stream;
        npc_status st = body();
        c->stream = parent;
        cudaGraph_t out = nullptr;
        cudaError_t ce = cudaStreamEndCapture(c->body_stream, &out);
        if (st != NPC_SUCCESS) return st;
        NPC_CUDA_TRY(ce);
        return NPC_SUCCESS;
    }
    template <class F>
    npc_status capture(F &&body, const int *cond_done = nullptr) {
        if (!c->graph_stream) {
            NPC_CUDA_TRY(cudaStreamCreateWithFlags(&c->graph_stream, cudaStreamNonBlocking));
            NPC_CUDA_TRY(cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming));
            NPC_CUDA_TRY(cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming));
        }
        NPC_CUDA_TRY(cudaEventRecord(c->ev_fork, orig));
        NPC_CUDA_TRY(cudaStreamWaitEvent(c->graph_stream, c->ev_fork, 0));
        c->stream = c->graph_stream;
        forked = true;
        if (cache.exec) {  // replay the graph captured by an earlier solve
            exec = cache.exec;
            kernels = cache.kernels;
            return NPC_SUCCESS;
        }
        const unsigned long long l0 = g_launches.load();
        NPC_CUDA_TRY(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
        c->capturing = c->timing;
        c->captured.clear();
        npc_status st = NPC_SUCCESS;
        for (int i = 0; i < ITERS && st == NPC_SUCCESS; ++i) st = cond_done ? cond_iteration(body, cond_done) : body();
        c->capturing = false;
        cache.release_events();
        cache.timing_events.swap(c->captured);
        cache.timed = c->timing;
        cudaGraph_t g = nullptr;
        cudaError_t ce = cudaStreamEndCapture(c->stream, &g);
        kernels = g_launches.load() - l0;
        g_launches.fetch_sub(kernels);  // captured, not launched
        if (st != NPC_SUCCESS) {
            if (g) cudaGraphDestroy(g);
            return st;
        }
        if (ce != cudaSuccess) {
            set_error("PCG graph capture failed: %s", cudaGetErrorString(ce));
            return NPC_ERR_CUDA;
        }
        cudaError_t ie = cudaGraphInstantiate(&exec, g, 0);
        cudaGraphDestroy(g);
        if (ie != cudaSuccess) {
            exec = nullptr;
            set_error("PCG graph instantiate failed: %s", cudaGetErrorString(ie));
            return NPC_ERR_CUDA;
        }
        cache.exec = exec;
        cache.kernels = kernels;
        return NPC_SUCCESS;
    }
    npc_status launch() {
        NPC_CUDA_TRY(cudaGraphLaunch(exec, c->stream));
        g_launches.fetch_add(kernels);
        return NPC_SUCCESS;
    }
    ~GraphRun() {
        if (forked) {
            cudaEventRecord(c->ev_join, c->stream);
            cudaStreamWaitEvent(orig, c->ev_join, 0);
            c->stream = orig;
        }
    }
};

static double now_s() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

// Device scalars area layout (ctx->scalars): [CgDev][sums: 8 doubles][history ...]
npc_status pcg(npc_poly P, npc_operator H, const double *b_ext, double *x_ext, double tol, int maxit,
               npc_pcg_stats *stats) {
    const double t0 = now_s();
    Operator *op = H->op.get();
    Context *ctx = op->ctx;
    const int n = op->n_local;
    const int k = P ? P->degree : 0;
    npc_pcg_stats st{};
    st.setup_seconds = P ? P->setup_seconds : 0.0;
    double *host_hist = stats ? stats->history : nullptr;
    // work vectors (internal order): b, x, r, u, w, p, s
    PcgCache &cache = P ? P->pcg : H->pcg;
    if (op->supports_fused_pcg() && !ctx->distributed() && (!P || (P->kind == 0 && P->lr_p == 0 &&
                                                                (P->degree == 0 || P->coef_dev.p)))) {
        // small operator: the whole solve in one cluster launch (csr_cluster.cu)
        if (cache.dev_maxit < maxit) {
            cache.invalidate();
            NPC_TRY(cache.dev.alloc(sizeof(CgDev) + sizeof(double) * (8 + (size_t)maxit + 1)));
            cache.dev_maxit = maxit;
        }
        ClusterPcgOut *dout = reinterpret_cast<ClusterPcgOut *>(cache.dev.p);
        double *dhist = reinterpret_cast<double *>(cache.dev.as<char>() + sizeof(CgDev)) + 8;
        // tol2b = tol^2 ||b||^2 needs ||b||: the kernel forms ||b||^2 itself, so pass tol^2 and
        // let it scale (encoded as a negative number: -tol^2)
        {
            TimedScope ts(ctx, T_DEGREE);
            NPC_TRY(op->pcg_fused(b_ext, x_ext, P ? P->coef_dev.as<double>() : nullptr, k,
                                  P ? P->theta_bar : 1.0, P ? 1 : 0, -tol * tol, maxit, dout,
                                  host_hist ? dhist : nullptr));
        }
        ClusterPcgOut h;
        NPC_CUDA_TRY(cudaMemcpyAsync(&h, dout, sizeof(h), cudaMemcpyDeviceToHost, ctx->stream));
        if (host_hist && h.iters >= 0)
            NPC_CUDA_TRY(cudaMemcpyAsync(host_hist, dhist, sizeof(double) * ((size_t)maxit + 1),
                                         cudaMemcpyDeviceToHost, ctx->stream));
        NPC_TRY(stream_sync(ctx, ctx->stream));
        if (ctx->timing) ctx->t_flush();
        st.iters = h.iters;
        st.converged = h.converged;
        st.op_applications = h.applications;
        st.reductions = h.reductions;
        st.relres_recursive = h.bnorm2 > 0.0 ? sqrt(h.rr / h.bnorm2) : 0.0;
        st.relres_true = h.relres_true;
        st.solve_seconds = now_s() - t0;
        if (stats) {
            double *hh = stats->history;
            *stats = st;
            stats->history = hh;
        }
        if (h.breakdown) {
            set_error("PCG breakdown (%s <= 0) at iteration %d", h.breakdown == 1 ? "<r,z>" : "<p,Ap>", h.iters);
            return NPC_ERR_BREAKDOWN;
        }
        if (!h.converged) {
            set_error("PCG did not converge in %d iterations (true relres %.3e)", maxit, h.relres_true);
            return NPC_ERR_NOT_CONVERGED;
        }
        return NPC_SUCCESS;
    }
    const size_t nn = std::max(n, 1);
    if (cache.work_n != nn) {
        cache.invalidate();
        NPC_TRY(cache.work.alloc(sizeof(double) * nn * 7));
        cache.work_n = nn;
    }
    DevBuf &work = cache.work;
    double *b = work.as<double>(), *x = b + nn, *r = x + nn, *u = r + nn, *w = u + nn, *p = w + nn, *s = p + nn;
    if (op->permuted()) {
        NPC_TRY(op->to_internal(b_ext, b));
        NPC_TRY(op->to_internal(x_ext, x));
    } else {
        NPC_CUDA_TRY(cudaMemcpyAsync(b, b_ext, sizeof(double) * n, cudaMemcpyDeviceToDevice, ctx->stream));
        NPC_CUDA_TRY(cudaMemcpyAsync(x, x_ext, sizeof(double) * n, cudaMemcpyDeviceToDevice, ctx->stream));
    }
    NPC_CUDA_TRY(cudaMemsetAsync(p, 0, sizeof(double) * n, ctx->stream));
    NPC_CUDA_TRY(cudaMemsetAsync(s, 0, sizeof(double) * n, ctx->stream));
    const int np_op = op->num_partials();
    const int np_vec = vec_grid(n);
    NPC_TRY(ctx->ensure_partials(std::max(np_op, np_vec)));
    double *P0 = ctx->partial_slot(0), *P1 = ctx->partial_slot(1), *P2 = ctx->partial_slot(2);
    if (cache.dev_maxit < maxit) {
        cache.invalidate();
        NPC_TRY(cache.dev.alloc(sizeof(CgDev) + sizeof(double) * (8 + (size_t)maxit + 1)));
        cache.dev_maxit = maxit;
    }
    if (cache.key_partials != ctx->partials.p || cache.key_cap != ctx->partial_cap) {
        cache.invalidate();
        cache.key_partials = ctx->partials.p;
        cache.key_cap = ctx->partial_cap;
    }
    DevBuf &dev = cache.dev;
    CgDev *cg = dev.as<CgDev>();
    double *sums = reinterpret_cast<double *>(cg + 1);
    double *dhist = sums + 8;

    // x0 == 0 ?  ||x0||^2 together with ||b||^2
    int npa = 0, npb = 0;
    NPC_TRY(launch_dot(ctx, b, b, n, P0, &npa));
    NPC_TRY(launch_dot(ctx, x, x, n, P1, &npb));
    NPC_TRY(launch_reduce_sum(ctx, P0, npa, sums + 0, 1, P1, npb, sums + 1));
    NPC_TRY(ctx->allreduce_sum(sums, 2));
    double h2[2];
    NPC_CUDA_TRY(cudaMemcpyAsync(h2, sums, sizeof(h2), cudaMemcpyDeviceToHost, ctx->stream));
    NPC_TRY(stream_sync(ctx, ctx->stream));
    st.reductions += 1;
    const double bnorm2 = h2[0];
    const bool x0_nonzero = h2[1] != 0.0;
    auto finish_true_residual = [&](double *relres) -> npc_status {
        // r_true = b - A x  (u as scratch), ||r_true||^2
        StepArgs t;
        t.x = x;
        t.r = b;
        t.out = u;
        t.a = -1.0;
        t.d = 1.0;
        {
            TimedScope ts(ctx, T_OPERATOR);
            NPC_TRY(op->step(t));
        }
        st.op_applications += 1;
        int np = 0;
        NPC_TRY(launch_dot(ctx, u, u, n, P0, &np));
        NPC_TRY(launch_reduce_sum(ctx, P0, np, sums + 3));
        NPC_TRY(ctx->allreduce_sum(sums + 3, 1));
        st.reductions += 1;
        double tr;
        NPC_CUDA_TRY(cudaMemcpyAsync(&tr, sums + 3, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
        NPC_TRY(stream_sync(ctx, ctx->stream));
        *relres = sqrt(tr / bnorm2);
        return NPC_SUCCESS;
    };
    auto export_x = [&]() -> npc_status {
        if (op->permuted()) return op->to_external(x, x_ext);
        NPC_CUDA_TRY(cudaMemcpyAsync(x_ext, x, sizeof(double) * n, cudaMemcpyDeviceToDevice, ctx->stream));
        return NPC_SUCCESS;
    };
    npc_status result = NPC_SUCCESS;
    if (bnorm2 == 0.0) {  // b = 0 -> x = 0
        NPC_CUDA_TRY(cudaMemsetAsync(x_ext, 0, sizeof(double) * n, ctx->stream));
        NPC_TRY(stream_sync(ctx, ctx->stream));
        st.converged = 1;
        st.solve_seconds = now_s() - t0;
        if (stats) {
            double *hh = stats->history;
            *stats = st;
            stats->history = hh;
            if (hh) hh[0] = 0.0;
        }
        return NPC_SUCCESS;
    }
    // r0 = b - A x0 (or b)
    if (x0_nonzero) {
        StepArgs t;
        t.x = x;
        t.r = b;
        t.out = r;
        t.a = -1.0;
        t.d = 1.0;
        {
            TimedScope ts(ctx, T_OPERATOR);
            NPC_TRY(op->step(t));
        }
        st.op_applications += 1;
    } else {
        NPC_CUDA_TRY(cudaMemcpyAsync(r, b, sizeof(double) * n, cudaMemcpyDeviceToDevice, ctx->stream));
    }
    {
        int np = 0;
        NPC_TRY(launch_dot(ctx, r, r, n, P0, &np));
        NPC_TRY(launch_reduce_sum(ctx, P0, np, sums + 2));
        NPC_TRY(ctx->allreduce_sum(sums + 2, 1));
        st.reductions += 1;
    }
    double rr0;
    NPC_CUDA_TRY(cudaMemcpyAsync(&rr0, sums + 2, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    NPC_TRY(stream_sync(ctx, ctx->stream));
    std::vector<double> hist_host;
    if (host_hist) host_hist[0] = sqrt(rr0 / bnorm2);
    CgDev h{};
    h.rr = rr0;
    h.bnorm2 = bnorm2;
    h.tol2 = tol * tol * bnorm2;
    h.maxit = maxit;
    h.first = 1;
    // 1 = side-stream ||r||^2 check (default), 2 = one fused {gamma, delta, ||r||^2} allreduce
    h.multi = ctx->distributed() ? (ctx->fused_allreduce ? 2 : 1) : 0;
    const bool side_rr = h.multi == 1, fused_rr = h.multi == 2;
    // the fused allreduce sums sums[2] over the ranks: a global value is seeded as its 1/P share
    const double rr_share = fused_rr ? 1.0 / ctx->nranks : 1.0;
    bool done = rr0 <= h.tol2;
    st.relres_recursive = sqrt(rr0 / bnorm2);
    if (done) {
        double tr;
        NPC_TRY(finish_true_residual(&tr));
        if (tr <= tol) {
            st.converged = 1;
            st.relres_true = tr;
            NPC_TRY(export_x());
            NPC_TRY(stream_sync(ctx, ctx->stream));
            st.solve_seconds = now_s() - t0;
            if (stats) {
                double *hh = stats->history;
                *stats = st;
                stats->history = hh;
            }
            return NPC_SUCCESS;
        }
        NPC_CUDA_TRY(cudaMemcpyAsync(r, u, sizeof(double) * n, cudaMemcpyDeviceToDevice, ctx->stream));
        h.rr = tr * tr * bnorm2;
    }
    double rr_seed = h.rr * rr_share;
    NPC_CUDA_TRY(cudaMemcpyAsync(cg, &h, sizeof(h), cudaMemcpyHostToDevice, ctx->stream));
    NPC_CUDA_TRY(cudaMemcpyAsync(sums + 2, &rr_seed, sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
    const int *dflag = &cg->done;
    int chunk = 4;
    // Iterations between host checks grow 4, 8, ..., 64 for short iterations; when one chunk of
    // 4 already takes >= 2 ms the host checks after every graph replay instead (a few µs per
    // check), so at most 3 iterations run past convergence -- no-op kernels still stream some
    // data (the CSR kernel issues its tile copy before reading the flag).
    int chunk_max = 64;
    double t_chunk = now_s();
    int true_checks = 0;
    bool rr_pending = false;
    long long iter_calls = 0;
    auto join_rr = [&]() -> npc_status {
        if (rr_pending) {
            NPC_CUDA_TRY(cudaStreamWaitEvent(ctx->stream, ctx->ev_rr1, 0));
            rr_pending = false;
        }
        return NPC_SUCCESS;
    };
    if (side_rr && !ctx->ev_rr0) {
        NPC_CUDA_TRY(cudaEventCreateWithFlags(&ctx->ev_rr0, cudaEventDisableTiming));
        NPC_CUDA_TRY(cudaEventCreateWithFlags(&ctx->ev_rr1, cudaEventDisableTiming));
    }
    // One PCG iteration = k fused degree kernels (+ halo) + A u + reduce (+ allreduce) +
    // scalars + update + ||r||^2; every kernel no-ops once the device flag says done.
    auto iteration = [&]() -> npc_status {
        {
            // u = p_k(A) r  with partials of gamma = <u, r>
            int npg = 0;
            if (P)
                NPC_TRY(apply_poly_internal(P, r, u, r, P0, &npg, dflag));
            else
                NPC_TRY(launch_scale(ctx, r, u, 1.0, n, r, P0, &npg, dflag));
            // w = A u with partials of delta = <w, u>
            StepArgs t;
            t.x = u;
            t.out = w;
            t.a = 1.0;
            t.dotv = u;
            t.partials = P1;
            t.done = dflag;
            {
                TimedScope ts(ctx, T_OPERATOR);
                NPC_TRY(op->step(t));
            }
            {
                TimedScope ts(ctx, T_REDUCE);
                NPC_TRY(launch_reduce_sum(ctx, P0, npg, sums + 0, 1, P1, np_op, sums + 1));
            }
            NPC_TRY(ctx->allreduce_sum(sums, fused_rr ? 3 : 2));  // the single global reduction
            NPC_TRY(join_rr());  // ||r_i||^2 of the previous update is known (and checked)
            {
                TimedScope ts(ctx, T_REDUCE);
                k_cg_scalars<<<1, 1, 0, ctx->stream>>>(cg, sums, dhist);
                NPC_LAUNCH_CHECK();
            }
            {
                TimedScope ts(ctx, T_UPDATE);
                k_cg_update<<<np_vec, 256, 0, ctx->stream>>>(cg, u, w, p, s, x, r, n, P2);
                NPC_LAUNCH_CHECK();
            }
            {
                TimedScope ts(ctx, T_REDUCE);
                k_cg_rr<<<1, 1024, 0, ctx->stream>>>(cg, P2, np_vec, sums, dhist);
                NPC_LAUNCH_CHECK();
            }
            if (side_rr) {  // ||r_{i+1}||^2: allreduce + check on the side stream
                NvtxRange nv("npc:allreduce_rr");
                NPC_CUDA_TRY(cudaEventRecord(ctx->ev_rr0, ctx->stream));
                NPC_CUDA_TRY(cudaStreamWaitEvent(ctx->aux_stream, ctx->ev_rr0, 0));
                NPC_TRY(ctx->tr->allreduce_sum_aux(ctx, sums + 4, 1, ctx->aux_stream));
                k_cg_rrcheck<<<1, 1, 0, ctx->aux_stream>>>(cg, sums + 4, dhist);
                NPC_LAUNCH_CHECK();
                NPC_CUDA_TRY(cudaEventRecord(ctx->ev_rr1, ctx->aux_stream));
                rr_pending = true;
                // a captured block of GraphRun::ITERS iterations ends joined
                if (++iter_calls % GraphRun::ITERS == 0) NPC_TRY(join_rr());
            }
        }
        return NPC_SUCCESS;
    };
    // CUDA Graph of GRAPH_ITERS iterations (all pointers and coefficients are fixed for the
    // solve), replayed on a library stream: one launch per 4 iterations instead of 4(k+5)
    // launches; NCCL calls and the halo fork/join are captured too.  Off while timing.
    // With timing on, the captured graph carries event-record nodes around every launch and is
    // replayed one graph per host sync so that its events can be read after each replay.
    if (cache.exec && (cache.timed != ctx->timing || cache.fused != fused_rr)) cache.invalidate();
    GraphRun gr(ctx, cache);
    const bool graph_ok = op->capture_safe() && (!ctx->tr || ctx->tr->capturable()) && !getenv("NPC_NO_GRAPH");
    // A new graph costs capture + instantiation: milliseconds with NCCL calls in it (16 ms for a
    // DFN block of 4 iterations on a 1-rank communicator) and ~0.1 ms per degree launch for high
    // degrees (config 5, k = 200: ~140 ms for a 1-iteration solve).  So a distributed or k >= 32
    // solve without a cached graph runs its first chunk eagerly -- its kernels are long enough
    // to hide the launches -- and captures only if it needs a second chunk.  (Low degrees
    // capture at once: eager 4-iteration chunks measured slower on configs 2 and 6, k = 30.)
    bool deferred = graph_ok && !cache.exec && (h.multi || k >= 32);
    // Opt-in (NPC_GRAPH_COND=1; single rank, untimed): each captured iteration is the body of a
    // conditional IF node whose condition a one-thread kernel sets from the done flag, so the
    // iterations after convergence inside a replayed block are skipped rather than launched as
    // no-ops.  A/B (phase_times, fresh polynomial): config 6 48.1 -> 47.1 ms, config 4 914 ->
    // 911 ms, config 3 unchanged, config 2 8.8 -> 9.3 ms (the larger graph costs more to build).
    const bool cond = !h.multi && !ctx->timing && getenv("NPC_GRAPH_COND") != nullptr;
    // ... and that eager chunk is ONE iteration: a solve that converges at once (config 5) then
    // stops there -- in a 4-iteration block the no-op iterations still launch every kernel, and
    // the bulk-copy kernels issue their tile loads before they read the done flag
    if (deferred) chunk = 1;
    if (graph_ok && !deferred) {
        iter_calls = 0;
        NPC_TRY(gr.capture(iteration, cond ? dflag : nullptr));
        cache.fused = fused_rr;
    }
    t_chunk = now_s();  // the first chunk's clock starts after the capture
    for (;;) {
        if (gr.exec) {
            if (ctx->timing) {  // read the events after every replay; stop replaying once done
                for (int it = 0; it < chunk; it += GraphRun::ITERS) {
                    NPC_TRY(gr.launch());
                    int dflag_h = 0;
                    NPC_CUDA_TRY(cudaMemcpyAsync(&dflag_h, dflag, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
                    NPC_TRY(stream_sync(ctx, ctx->stream));
                    ctx->t_flush_graph(cache.timing_events);
                    if (dflag_h) break;
                }
            } else {
                for (int it = 0; it < chunk; it += GraphRun::ITERS) NPC_TRY(gr.launch());
            }
        } else {
            for (int it = 0; it < chunk; ++it) NPC_TRY(iteration());
            NPC_TRY(join_rr());
        }
        NPC_CUDA_TRY(cudaMemcpyAsync(&h, cg, sizeof(h), cudaMemcpyDeviceToHost, ctx->stream));
        NPC_TRY(stream_sync(ctx, ctx->stream));
        if (ctx->timing) ctx->t_flush();
        if (!h.done) {
            if (deferred) {
                deferred = false;
                iter_calls = 0;
                NPC_TRY(gr.capture(iteration, cond ? dflag : nullptr));
                cache.fused = fused_rr;
            }
            if (chunk_max == 64 && now_s() - t_chunk >= 2e-3) chunk_max = GraphRun::ITERS;
            chunk = std::min(chunk * 2, chunk_max);
            t_chunk = now_s();
            continue;
        }
        st.iters = h.iters;
        st.relres_recursive = sqrt(h.rr / bnorm2);
        // fused allreduce: the exit was seen after u = p_k(A) r and w = A u of the next iteration
        if (fused_rr && !h.breakdown) st.op_applications += k + 1, st.reductions += 1;
        if (h.breakdown) {
            set_error("PCG breakdown (%s <= 0) at iteration %d", h.breakdown == 1 ? "<r,z>" : "<p,Ap>", h.iters);
            result = NPC_ERR_BREAKDOWN;
            break;
        }
        if (h.converged) {
            double tr;
            NPC_TRY(finish_true_residual(&tr));
            st.relres_true = tr;
            if (tr <= tol || ++true_checks > 50) {
                st.converged = tr <= tol;
                if (!st.converged) {
                    set_error("true residual %.3e stays above tol after %d replacements", tr, true_checks - 1);
                    result = NPC_ERR_NOT_CONVERGED;
                }
                break;
            }
            // residual replacement (reading A23): r = b - A x, and restart the recurrence
            // from the current x (beta = 0: p = u, s = w in the next iteration)
            NPC_CUDA_TRY(cudaMemcpyAsync(r, u, sizeof(double) * n, cudaMemcpyDeviceToDevice, ctx->stream));
            h.rr = tr * tr * bnorm2;
            h.converged = 0;
            h.done = 0;
            h.first = 1;
            rr_seed = h.rr * rr_share;
            NPC_CUDA_TRY(cudaMemcpyAsync(cg, &h, sizeof(h), cudaMemcpyHostToDevice, ctx->stream));
            NPC_CUDA_TRY(cudaMemcpyAsync(sums + 2, &rr_seed, sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
            if (h.iters >= maxit) {
                result = NPC_ERR_NOT_CONVERGED;
                break;
            }
            chunk = 1;
            continue;
        }
        // maxit
        double tr;
        NPC_TRY(finish_true_residual(&tr));
        st.relres_true = tr;
        set_error("PCG did not converge in %d iterations (relres %.3e)", maxit, st.relres_recursive);
        result = NPC_ERR_NOT_CONVERGED;
        break;
    }
    // counters: k+1 applications per x-update (Table tab11 law); distributed contexts reduce
    // ||r||^2 in a second (overlapped) allreduce per iteration.  Not counted: the application
    // in flight when the overlapped check raises the done flag (its remaining kernels no-op).
    st.op_applications += (long long)h.iters * (k + 1);
    st.reductions += h.iters * (side_rr ? 2 : 1);
    if (P && P->lr_p > 0)  // V^T r inside every application of the preconditioner
        st.reductions += h.iters;
    if (host_hist && h.iters > 0)
        NPC_CUDA_TRY(cudaMemcpyAsync(host_hist + 1, dhist + 1, sizeof(double) * h.iters, cudaMemcpyDeviceToHost,
                                     ctx->stream));
    NPC_TRY(export_x());
    NPC_TRY(stream_sync(ctx, ctx->stream));
    st.solve_seconds = now_s() - t0;
    if (stats) {
        double *hh = stats->history;
        *stats = st;
        stats->history = hh;
    }
    return result;
}

// ================================================================== Lanczos
struct LzDev {
    double vn2;
    int steps, stop;
};

__global__ void k_lz_scale_init(const double *v0, double *q, double *qprev, int n, const double *vn2) {
    const double inv = 1.0 / sqrt(*vn2);
    for (int i = blockIdx.x * 256 + threadIdx.x; i < n; i += gridDim.x * 256) {
        q[i] = v0[i] * inv;
        qprev[i] = 0.0;
    }
}

// mode 0: w -= beta_prev q_prev ; partial <q, w>
// mode 1: w -= alpha q          ; partial <w, w>
template <int MODE>
__global__ void __launch_bounds__(256) k_lz_axpy(double *__restrict__ w, const double *__restrict__ v,
                                                 const double *__restrict__ q, const double *coef, int n,
                                                 double *partials, const LzDev *lz) {
    if (lz->stop) return;
    __shared__ double red[8];
    const double cf = coef ? *coef : 0.0;
    double acc = 0.0;
    for (int i = blockIdx.x * 256 + threadIdx.x; i < n; i += gridDim.x * 256) {
        const double wi = w[i] - cf * v[i];
        w[i] = wi;
        acc += (MODE == 0 ? q[i] : wi) * wi;
    }
    acc = block_sum<256>(acc, red);
    if (threadIdx.x == 0) partials[blockIdx.x] = acc;
}

__global__ void k_lz_beta(LzDev *lz, double *betas, int j, const double *sum) {
    if (lz->stop) return;
    const double b = sqrt(*sum);
    betas[j] = b;
    lz->steps = j + 1;
    if (b == 0.0) lz->stop = 1;
}

__global__ void k_lz_next(const LzDev *lz, const double *w, double *q, double *qprev, const double *beta, int n) {
    if (lz->stop) return;
    const double inv = 1.0 / *beta;
    for (int i = blockIdx.x * 256 + threadIdx.x; i < n; i += gridDim.x * 256) {
        qprev[i] = q[i];
        q[i] = w[i] * inv;
    }
}

// Number of eigenvalues of the symmetric tridiagonal T (diag a, offdiag b) below x.
static int sturm_count(const std::vector<double> &a, const std::vector<double> &b, double x) {
    int cnt = 0;
    double d = 1.0;
    for (size_t i = 0; i < a.size(); ++i) {
        const double off2 = i ? b[i - 1] * b[i - 1] : 0.0;
        d = a[i] - x - (i ? off2 / d : 0.0);
        if (d == 0.0) d = -1e-300;
        if (d < 0.0) ++cnt;
    }
    return cnt;
}

static double tridiag_eig(const std::vector<double> &a, const std::vector<double> &b, int idx) {
    double lo = 1e300, hi = -1e300;
    for (size_t i = 0; i < a.size(); ++i) {  // Gershgorin
        double r = (i ? fabs(b[i - 1]) : 0.0) + (i + 1 < a.size() ? fabs(b[i]) : 0.0);
        lo = std::min(lo, a[i] - r);
        hi = std::max(hi, a[i] + r);
    }
    for (int it = 0; it < 200 && hi - lo > 1e-16 * std::max(fabs(lo), fabs(hi)); ++it) {
        const double mid = 0.5 * (lo + hi);
        if (mid <= lo || mid >= hi) break;
        if (sturm_count(a, b, mid) > idx)
            hi = mid;
        else
            lo = mid;
    }
    return 0.5 * (lo + hi);
}

// Solve (T - mu I) x = x (in place) for the symmetric tridiagonal T (diag a, offdiag b) by
// Gaussian elimination with partial pivoting (the dgttrf/dgttrs scheme).
static void tridiag_shift_solve(const std::vector<double> &a, const std::vector<double> &b, double mu,
                                std::vector<double> &x) {
    const int m = (int)a.size();
    std::vector<double> d(m), du(m, 0.0), du2(m, 0.0), dl(m, 0.0);
    std::vector<char> swp(m, 0);
    const double tiny = 1e-300 + 1e-16 * (fabs(mu) + 1e-300);
    for (int i = 0; i < m; ++i) {
        d[i] = a[i] - mu;
        if (i + 1 < m) du[i] = dl[i] = b[i];
    }
    for (int i = 0; i + 1 < m; ++i) {
        if (fabs(d[i]) >= fabs(dl[i])) {
            if (d[i] == 0.0) d[i] = tiny;
            const double f = dl[i] / d[i];
            dl[i] = f;
            d[i + 1] -= f * du[i];
        } else {
            const double f = d[i] / dl[i];
            d[i] = dl[i];
            dl[i] = f;
            const double t = du[i];
            du[i] = d[i + 1];
            d[i + 1] = t - f * d[i + 1];
            if (i + 2 < m) {
                du2[i] = du[i + 1];
                du[i + 1] = -f * du[i + 1];
            }
            swp[i] = 1;
        }
    }
    if (d[m - 1] == 0.0) d[m - 1] = tiny;
    for (int i = 0; i + 1 < m; ++i) {
        if (!swp[i]) {
            x[i + 1] -= dl[i] * x[i];
        } else {
            const double t = x[i];
            x[i] = x[i + 1];
            x[i + 1] = t - dl[i] * x[i];
        }
    }
    x[m - 1] /= d[m - 1];
    if (m > 1) x[m - 2] = (x[m - 2] - du[m - 2] * x[m - 1]) / d[m - 2];
    for (int i = m - 3; i >= 0; --i) x[i] = (x[i] - du[i] * x[i + 1] - du2[i] * x[i + 2]) / d[i];
}

double tridiag_eigenvalue(const std::vector<double> &a, const std::vector<double> &b, int idx) {
    return tridiag_eig(a, b, idx);
}
void tridiag_inverse_iteration(const std::vector<double> &a, const std::vector<double> &b, double mu,
                               std::vector<double> &x) {
    tridiag_shift_solve(a, b, mu, x);
}

npc_status lanczos(Operator *op, int m, const double *v0_ext, unsigned long long seed, double *lmin, double *lmax,
                   double *out_ex) {
    Context *ctx = op->ctx;
    const int n = op->n_local;
    const size_t nn = std::max(n, 1);
    DevBuf work, dev;
    NPC_TRY(work.alloc(sizeof(double) * nn * 4));
    double *q = work.as<double>(), *qp = q + nn, *w = qp + nn, *v0 = w + nn;
    if (v0_ext) {
        if (op->permuted())
            NPC_TRY(op->to_internal(v0_ext, v0));
        else
            NPC_CUDA_TRY(cudaMemcpyAsync(v0, v0_ext, sizeof(double) * n, cudaMemcpyDeviceToDevice, ctx->stream));
    } else {
        NPC_TRY(launch_hash_vector(ctx, w, n, op->row_begin, seed));
        if (op->permuted())
            NPC_TRY(op->to_internal(w, v0));
        else
            NPC_CUDA_TRY(cudaMemcpyAsync(v0, w, sizeof(double) * n, cudaMemcpyDeviceToDevice, ctx->stream));
    }
    NPC_TRY(dev.alloc(sizeof(LzDev) + sizeof(double) * (2 * (size_t)m + 8)));
    LzDev *lz = dev.as<LzDev>();
    double *alphas = reinterpret_cast<double *>(lz + 1), *betas = alphas + m, *sums = betas + m;
    NPC_CUDA_TRY(cudaMemsetAsync(dev.p, 0, dev.bytes, ctx->stream));
    const int npv = vec_grid(n);
    NPC_TRY(ctx->ensure_partials(std::max(npv, op->num_partials())));
    double *P0 = ctx->partial_slot(0);
    int np = 0;
    NPC_TRY(launch_dot(ctx, v0, v0, n, P0, &np));
    NPC_TRY(launch_reduce_sum(ctx, P0, np, &lz->vn2));
    NPC_TRY(ctx->allreduce_sum(&lz->vn2, 1));
    double vn2;
    NPC_CUDA_TRY(cudaMemcpyAsync(&vn2, &lz->vn2, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    NPC_TRY(stream_sync(ctx, ctx->stream));
    if (!(vn2 > 0.0)) {
        set_error("estimate_spectrum: start vector is zero");
        return NPC_ERR_INVALID_ARGUMENT;
    }
    if (op->supports_fused_lanczos() && !ctx->distributed()) {  // small operator: one cluster launch
        TimedScope ts(ctx, T_OPERATOR);
        NPC_TRY(op->lanczos_fused(v0, m, alphas, betas, &lz->steps));
    } else {
    k_lz_scale_init<<<npv, 256, 0, ctx->stream>>>(v0, q, qp, n, &lz->vn2);
    NPC_LAUNCH_CHECK();
    for (int j = 0; j < m; ++j) {
        StepArgs s;
        s.x = q;
        s.out = w;
        s.a = 1.0;
        s.done = &lz->stop;
        {
            TimedScope ts(ctx, T_OPERATOR);
            NPC_TRY(op->step(s));
        }
        {
            TimedScope ts(ctx, T_VECTOR);
            k_lz_axpy<0><<<npv, 256, 0, ctx->stream>>>(w, qp, q, j ? &betas[j - 1] : nullptr, n, P0, lz);
            NPC_LAUNCH_CHECK();
        }
        {
            TimedScope ts(ctx, T_REDUCE);
            NPC_TRY(launch_reduce_sum(ctx, P0, npv, &alphas[j]));
        }
        NPC_TRY(ctx->allreduce_sum(&alphas[j], 1));
        {
            TimedScope ts(ctx, T_VECTOR);
            k_lz_axpy<1><<<npv, 256, 0, ctx->stream>>>(w, q, nullptr, &alphas[j], n, P0, lz);
            NPC_LAUNCH_CHECK();
        }
        {
            TimedScope ts(ctx, T_REDUCE);
            NPC_TRY(launch_reduce_sum(ctx, P0, npv, &sums[0]));
        }
        NPC_TRY(ctx->allreduce_sum(&sums[0], 1));
        {
            TimedScope ts(ctx, T_REDUCE);
            k_lz_beta<<<1, 1, 0, ctx->stream>>>(lz, betas, j, &sums[0]);
            NPC_LAUNCH_CHECK();
        }
        {
            TimedScope ts(ctx, T_VECTOR);
            k_lz_next<<<npv, 256, 0, ctx->stream>>>(lz, w, q, qp, &betas[j], n);
            NPC_LAUNCH_CHECK();
        }
    }
    }
    LzDev hl;
    std::vector<double> ha(m), hb(m);
    NPC_CUDA_TRY(cudaMemcpyAsync(&hl, lz, sizeof(hl), cudaMemcpyDeviceToHost, ctx->stream));
    NPC_CUDA_TRY(cudaMemcpyAsync(ha.data(), alphas, sizeof(double) * m, cudaMemcpyDeviceToHost, ctx->stream));
    NPC_CUDA_TRY(cudaMemcpyAsync(hb.data(), betas, sizeof(double) * m, cudaMemcpyDeviceToHost, ctx->stream));
    NPC_TRY(stream_sync(ctx, ctx->stream));
    if (ctx->timing) ctx->t_flush();
    const int sN = std::max(1, hl.steps);
    const double beta_last = hb[sN - 1];
    ha.resize(sN);
    hb.resize(sN > 1 ? sN - 1 : 0);
    const double th_min = tridiag_eig(ha, hb, 0);
    const double th_max = tridiag_eig(ha, hb, sN - 1);
    // Ritz residual of the top pair: ||A y - theta y|| = beta_s |e_s^T s|, s from inverse
    // iteration on T_s - theta I (tridiagonal LU with partial pivoting).
    double rho = 0.0;
    if (hl.stop == 0 && beta_last > 0.0) {
        std::vector<double> x(sN, 1.0);
        for (int it = 0; it < 3; ++it) {
            tridiag_shift_solve(ha, hb, th_max, x);
            double nrm = 0.0;
            for (double v : x) nrm += v * v;
            nrm = sqrt(nrm);
            if (!(nrm > 0.0) || !std::isfinite(nrm)) break;
            for (double &v : x) v /= nrm;
        }
        rho = beta_last * fabs(x[sN - 1]);
    }
    if (out_ex) {
        out_ex[0] = th_min;
        out_ex[1] = th_max;
        out_ex[2] = rho;
        out_ex[3] = (double)hl.steps;
    }
    *lmin = th_min;
    *lmax = th_max + rho;
    return NPC_SUCCESS;
}

}  // namespace npc
