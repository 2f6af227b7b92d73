// api.cu -- the C ABI (include/npc.h): argument validation, handle lifetime, dispatch.
#include <stdarg.h>
#include <stdio.h>

#include <algorithm>
#include <chrono>
#include <cstring>

#include "npc_internal.cuh"

namespace npc {
std::atomic<unsigned long long> g_launches{0};
static thread_local char g_err[1024] = "";
// The context of the API call in progress on this thread (ErrScope): set_error also records
// the message there, for npc_last_error(ctx).
static thread_local npc_context g_cur = nullptr;
void set_error(const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
    if (g_cur) memcpy(g_cur->err, g_err, sizeof(g_err));
}
struct ErrScope {
    npc_context prev;
    explicit ErrScope(npc_context c) : prev(g_cur) { g_cur = c; }
    ~ErrScope() { g_cur = prev; }
};
static double wall_s() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}
npc_status poly_coefficients(int k, double lmin, double lmax, double xi, double *theta_bar, double *delta,
                             double *sigma, double *coef);
npc_status apply_poly(npc_poly P, const double *r, double *z);
npc_status apply_operator(Operator *op, const double *x, double *y, DevBuf &scratch);
npc_status pcg(npc_poly P, npc_operator H, const double *b, double *x, double tol, int maxit, npc_pcg_stats *stats);
npc_status lanczos(Operator *op, int m, const double *v0, unsigned long long seed, double *lmin, double *lmax,
                   double *out_ex);
npc_status newton_zetas(int nlev, double lmin, double lmax, double xi, std::vector<double> &zeta);
}  // namespace npc

using namespace npc;

#define NPC_GUARD(cond, code, ...)      \
    do {                                \
        if (!(cond)) {                  \
            npc::set_error(__VA_ARGS__); \
            return code;                \
        }                               \
    } while (0)

// Select the device of the handle for the duration of a call.
struct DeviceScope {
    int prev = -1;
    explicit DeviceScope(int dev) {
        if (cudaGetDevice(&prev) == cudaSuccess && prev != dev) cudaSetDevice(dev);
    }
    ~DeviceScope() {
        int cur;
        if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
    }
};

extern "C" {

const char *npc_last_error(npc_context ctx) { return ctx ? ctx->err : g_err; }
unsigned long long npc_launch_count(void) { return g_launches.load(); }
const char *npc_version(void) { return "npc 0.2 sm_100a (fp64, CSR/SELL/stencil/Schur/DFN/callback)"; }

npc_status npc_get_unique_id(void *out128) {
    NPC_GUARD(out128, NPC_ERR_INVALID_ARGUMENT, "npc_get_unique_id: null output");
    ncclUniqueId id;
    NPC_NCCL_TRY(ncclGetUniqueId(&id));
    static_assert(sizeof(id) == 128, "ncclUniqueId is 128 bytes");
    memcpy(out128, &id, sizeof(id));
    return NPC_SUCCESS;
}

}  // extern "C"

static npc_status context_create(int device, int nranks, int rank, const void *nccl_unique_id,
                                 const char *local_group, void *cuda_stream, npc_context *out) {
    NPC_GUARD(out, NPC_ERR_INVALID_ARGUMENT, "npc_context_create: null output");
    *out = nullptr;
    NPC_GUARD(nranks >= 1 && rank >= 0 && rank < nranks, NPC_ERR_INVALID_ARGUMENT, "npc_context_create: bad rank %d/%d",
              rank, nranks);
    int ndev = 0;
    NPC_CUDA_TRY(cudaGetDeviceCount(&ndev));
    NPC_GUARD(device >= 0 && device < ndev, NPC_ERR_INVALID_ARGUMENT, "npc_context_create: device %d of %d", device, ndev);
    cudaDeviceProp prop;
    NPC_CUDA_TRY(cudaGetDeviceProperties(&prop, device));
    NPC_GUARD(prop.major == 10 && prop.minor == 0, NPC_ERR_UNSUPPORTED,
              "libnpc is built for sm_100a (B200); device %d is sm_%d%d", device, prop.major, prop.minor);
    DeviceScope ds(device);
    NPC_CUDA_TRY(cudaSetDevice(device));
    auto h = std::make_unique<npc_context_s>();
    Context &c = h->ctx;
    c.device = device;
    c.nranks = nranks;
    c.rank = rank;
    c.num_sms = prop.multiProcessorCount;
    if (cuda_stream) {
        c.stream = (cudaStream_t)cuda_stream;
    } else {
        NPC_CUDA_TRY(cudaStreamCreateWithFlags(&c.stream, cudaStreamNonBlocking));
        c.own_stream = true;
    }
    if (nranks > 1 || local_group || nccl_unique_id) {
        NPC_CUDA_TRY(cudaStreamCreateWithFlags(&c.comm_stream, cudaStreamNonBlocking));
        NPC_CUDA_TRY(cudaStreamCreateWithFlags(&c.aux_stream, cudaStreamNonBlocking));
        if (local_group)
            NPC_TRY(make_local_transport(&c, local_group, c.tr));
        else
            NPC_TRY(make_nccl_transport(&c, nccl_unique_id, c.tr));
        const char *e = getenv("NPC_PCG_FUSED_ALLREDUCE");
        c.fused_allreduce = e && atoi(e) != 0;
    }
    NPC_TRY(c.ensure_partials(4096));
    *out = h.release();
    return NPC_SUCCESS;
}

extern "C" {

npc_status npc_context_create(int device, int nranks, int rank, const void *nccl_unique_id, void *cuda_stream,
                              npc_context *out) {
    NPC_GUARD(nranks == 1 || nccl_unique_id, NPC_ERR_INVALID_ARGUMENT,
              "npc_context_create: nranks > 1 needs an NCCL unique id");
    return context_create(device, nranks, rank, nccl_unique_id, nullptr, cuda_stream, out);
}

npc_status npc_context_create_local(int device, int nranks, int rank, const char *group, void *cuda_stream,
                                    npc_context *out) {
    NPC_GUARD(group && group[0], NPC_ERR_INVALID_ARGUMENT, "npc_context_create_local: empty group name");
    return context_create(device, nranks, rank, nullptr, group, cuda_stream, out);
}

npc_status npc_context_set_timing(npc_context ctx, int enable) {
    NPC_GUARD(ctx, NPC_ERR_INVALID_ARGUMENT, "npc_context_set_timing: null context");
    ErrScope es(ctx);
    ctx->ctx.timing = enable != 0;
    return NPC_SUCCESS;
}

npc_status npc_context_set_fused_allreduce(npc_context ctx, int enable) {
    NPC_GUARD(ctx, NPC_ERR_INVALID_ARGUMENT, "npc_context_set_fused_allreduce: null context");
    ErrScope es(ctx);
    ctx->ctx.fused_allreduce = enable != 0;
    return NPC_SUCCESS;
}

npc_status npc_context_get_timing(npc_context ctx, double *ms_out, long long *launches_out) {
    NPC_GUARD(ctx, NPC_ERR_INVALID_ARGUMENT, "npc_context_get_timing: null context");
    ErrScope es(ctx);
    DeviceScope ds(ctx->ctx.device);
    NPC_CUDA_TRY(cudaStreamSynchronize(ctx->ctx.stream));
    ctx->ctx.t_flush();
    for (int i = 0; i < NPC_TIMING_CLASSES; ++i) {
        if (ms_out) ms_out[i] = ctx->ctx.t_ms[i];
        if (launches_out) launches_out[i] = ctx->ctx.t_cnt[i];
        ctx->ctx.t_ms[i] = 0.0;
        ctx->ctx.t_cnt[i] = 0;
    }
    return NPC_SUCCESS;
}

npc_status npc_context_destroy(npc_context ctx) {
    if (!ctx) return NPC_SUCCESS;
    {
        DeviceScope ds(ctx->ctx.device);
        Context &c = ctx->ctx;
        if (c.stream) cudaStreamSynchronize(c.stream);
        c.tr.reset();
        if (c.comm_stream) cudaStreamDestroy(c.comm_stream);
        if (c.aux_stream) cudaStreamDestroy(c.aux_stream);
        c.partials.release();
        c.scalars.release();
        if (c.own_stream && c.stream) cudaStreamDestroy(c.stream);
    }
    delete ctx;
    return NPC_SUCCESS;
}

npc_status npc_create_operator(npc_context ctx, const npc_operator_desc *desc, npc_operator *out) {
    NPC_GUARD(ctx && desc && out, NPC_ERR_INVALID_ARGUMENT, "npc_create_operator: null argument");
    ErrScope es(ctx);
    *out = nullptr;
    NPC_GUARD(desc->n_local >= 0 && desc->row_begin >= 0, NPC_ERR_DIMENSION, "npc_create_operator: negative size");
    if (!ctx->ctx.distributed())
        NPC_GUARD(desc->row_begin == 0 && (desc->n_global == 0 || desc->n_global == desc->n_local), NPC_ERR_DIMENSION,
                  "npc_create_operator: single rank must own all rows");
    else
        NPC_GUARD(desc->row_begin + desc->n_local <= desc->n_global, NPC_ERR_DIMENSION,
                  "npc_create_operator: rows beyond n_global");
    DeviceScope ds(ctx->ctx.device);
    npc_operator_desc d = *desc;
    if (d.n_global == 0) d.n_global = d.n_local;
    std::unique_ptr<Operator> op;
    switch (d.kind) {
        case NPC_OP_CSR: NPC_TRY(make_csr_operator(&ctx->ctx, &d, op)); break;
        case NPC_OP_SELL: NPC_TRY(make_sell_operator(&ctx->ctx, &d, op)); break;
        case NPC_OP_STENCIL: NPC_TRY(make_stencil_operator(&ctx->ctx, &d, op)); break;
        case NPC_OP_SCHUR: NPC_TRY(make_schur_operator(&ctx->ctx, &d, op)); break;
        case NPC_OP_CALLBACK: NPC_TRY(make_callback_operator(&ctx->ctx, &d, op)); break;
        case NPC_OP_DFN: NPC_TRY(make_dfn_operator(&ctx->ctx, &d, op)); break;
        default: NPC_GUARD(false, NPC_ERR_INVALID_ARGUMENT, "npc_create_operator: unknown kind %d", (int)d.kind);
    }
    NPC_TRY(ctx->ctx.ensure_partials(op->num_partials()));
    NPC_CUDA_TRY(cudaDeviceSynchronize());
    auto h = std::make_unique<npc_operator_s>();
    h->owner = ctx;
    h->device = ctx->ctx.device;
    h->op = std::move(op);
    *out = h.release();
    return NPC_SUCCESS;
}

npc_status npc_operator_matrix_bytes(npc_operator op, double *bytes) {
    NPC_GUARD(op && bytes, NPC_ERR_INVALID_ARGUMENT, "npc_operator_matrix_bytes: null argument");
    ErrScope es(op->owner);
    *bytes = op->op->matrix_bytes();
    return NPC_SUCCESS;
}

npc_status npc_destroy_operator(npc_operator op) {
    if (!op) return NPC_SUCCESS;
    {
        DeviceScope ds(op->device);
        cudaDeviceSynchronize();
        op->op.reset();
    }
    delete op;
    return NPC_SUCCESS;
}

npc_status npc_apply_operator(npc_operator op, const double *x_dev, double *y_dev) {
    ErrScope es(op ? op->owner : nullptr);
    NPC_GUARD(op && (x_dev || op->op->n_local == 0) && (y_dev || op->op->n_local == 0), NPC_ERR_INVALID_ARGUMENT,
              "npc_apply_operator: null argument");
    NPC_GUARD(x_dev != y_dev || op->op->n_local == 0, NPC_ERR_INVALID_ARGUMENT, "npc_apply_operator: x aliases y");
    DeviceScope ds(op->owner->ctx.device);
    static thread_local DevBuf scratch;
    return apply_operator(op->op.get(), x_dev, y_dev, scratch);
}

npc_status npc_estimate_spectrum(npc_operator op, int nsteps, const double *v0_dev, unsigned long long seed,
                                 double *lmin, double *lmax) {
    ErrScope es(op ? op->owner : nullptr);
    NPC_GUARD(op && lmin && lmax, NPC_ERR_INVALID_ARGUMENT, "npc_estimate_spectrum: null argument");
    NPC_GUARD(nsteps >= 1 && nsteps <= 100000, NPC_ERR_INVALID_ARGUMENT, "npc_estimate_spectrum: nsteps %d", nsteps);
    NPC_GUARD(op->op->n_global >= 1, NPC_ERR_DIMENSION, "npc_estimate_spectrum: empty operator");
    DeviceScope ds(op->owner->ctx.device);
    const double t0 = wall_s();
    const npc_status st = lanczos(op->op.get(), nsteps, v0_dev, seed, lmin, lmax, nullptr);
    op->estimate_seconds = wall_s() - t0;
    return st;
}

npc_status npc_estimate_spectrum_ex(npc_operator op, int nsteps, const double *v0_dev, unsigned long long seed,
                                    double *out4) {
    ErrScope es(op ? op->owner : nullptr);
    NPC_GUARD(op && out4, NPC_ERR_INVALID_ARGUMENT, "npc_estimate_spectrum_ex: null argument");
    NPC_GUARD(nsteps >= 1 && nsteps <= 100000, NPC_ERR_INVALID_ARGUMENT, "npc_estimate_spectrum_ex: nsteps %d", nsteps);
    NPC_GUARD(op->op->n_global >= 1, NPC_ERR_DIMENSION, "npc_estimate_spectrum_ex: empty operator");
    DeviceScope ds(op->owner->ctx.device);
    double lo, hi;
    const double t0 = wall_s();
    const npc_status st = lanczos(op->op.get(), nsteps, v0_dev, seed, &lo, &hi, out4);
    op->estimate_seconds = wall_s() - t0;
    return st;
}

npc_status npc_poly_coefficients(int degree, double lmin, double lmax, double xi, double *theta_bar, double *delta,
                                 double *sigma, double *coef) {
    NPC_GUARD(theta_bar && delta && sigma, NPC_ERR_INVALID_ARGUMENT, "npc_poly_coefficients: null output");
    return poly_coefficients(degree, lmin, lmax, xi, theta_bar, delta, sigma, coef);
}

npc_status npc_set_poly(npc_operator op, int degree, double lmin, double lmax, double xi, npc_poly *out) {
    ErrScope es(op ? op->owner : nullptr);
    NPC_GUARD(op && out, NPC_ERR_INVALID_ARGUMENT, "npc_set_poly: null argument");
    const double t0 = wall_s();
    *out = nullptr;
    NPC_GUARD(degree <= 100000, NPC_ERR_INVALID_ARGUMENT, "npc_set_poly: degree %d too large", degree);
    auto P = std::make_unique<npc_poly_s>();
    P->op = op;
    P->device = op->device;
    P->degree = degree;
    P->lmin = lmin;
    P->lmax = lmax;
    P->xi = xi;
    P->coef.assign(4 * (size_t)std::max(degree, 0) + 4, 0.0);
    NPC_TRY(poly_coefficients(degree, lmin, lmax, xi, &P->theta_bar, &P->delta, &P->sigma, P->coef.data()));
    DeviceScope ds(op->owner->ctx.device);
    const size_t n = std::max(op->op->n_local, 1);
    NPC_TRY(P->tmp.alloc(sizeof(double) * n));
    if (degree >= 4 && op->op->supports_step2()) NPC_TRY(P->tmp2.alloc(sizeof(double) * n * 2));
    if (degree >= 1 && op->op->supports_fused_poly()) {
        NPC_TRY(P->coef_dev.alloc(sizeof(double) * 4 * (size_t)degree));
        NPC_CUDA_TRY(cudaMemcpy(P->coef_dev.p, P->coef.data(), sizeof(double) * 4 * (size_t)degree,
                                cudaMemcpyHostToDevice));
    }
    if (op->op->permuted()) {
        NPC_TRY(P->rin.alloc(sizeof(double) * n));
        NPC_TRY(P->zout.alloc(sizeof(double) * n));
    }
    P->setup_seconds = op->estimate_seconds + (wall_s() - t0);
    *out = P.release();
    return NPC_SUCCESS;
}

npc_status npc_set_poly_newton(npc_operator op, int nlev, double lmin, double lmax, double xi, npc_poly *out) {
    ErrScope es(op ? op->owner : nullptr);
    NPC_GUARD(op && out, NPC_ERR_INVALID_ARGUMENT, "npc_set_poly_newton: null argument");
    const double t0 = wall_s();
    *out = nullptr;
    NPC_GUARD(nlev >= 0 && nlev <= 16, NPC_ERR_INVALID_ARGUMENT, "npc_set_poly_newton: nlev %d not in [0, 16]", nlev);
    auto P = std::make_unique<npc_poly_s>();
    P->op = op;
    P->device = op->device;
    P->kind = 1;
    P->nlev = nlev;
    P->degree = (1 << nlev) - 1;
    P->lmin = lmin;
    P->lmax = lmax;
    P->xi = xi;
    NPC_TRY(newton_zetas(nlev, lmin, lmax, xi, P->zeta));
    NPC_TRY(poly_coefficients(0, lmin, lmax, xi, &P->theta_bar, &P->delta, &P->sigma, nullptr));
    DeviceScope ds(op->device);
    const size_t n = std::max(op->op->n_local, 1);
    NPC_TRY(P->tmp.alloc(sizeof(double) * n));
    if (nlev >= 2) NPC_TRY(P->nbuf.alloc(sizeof(double) * n * 2 * (nlev - 1)));
    if (op->op->permuted()) {
        NPC_TRY(P->rin.alloc(sizeof(double) * n));
        NPC_TRY(P->zout.alloc(sizeof(double) * n));
    }
    P->setup_seconds = op->estimate_seconds + (wall_s() - t0);
    *out = P.release();
    return NPC_SUCCESS;
}

npc_status npc_poly_set_lowrank(npc_poly poly, int p, const double *V_dev) {
    NPC_GUARD(poly, NPC_ERR_INVALID_ARGUMENT, "npc_poly_set_lowrank: null poly");
    ErrScope es(poly->op->owner);
    NPC_GUARD(p >= 0 && p <= NPC_LOWRANK_MAX, NPC_ERR_INVALID_ARGUMENT, "npc_poly_set_lowrank: p %d not in [0, %d]", p,
              NPC_LOWRANK_MAX);
    NPC_GUARD(p == 0 || poly->op->op->n_local == 0 || V_dev, NPC_ERR_INVALID_ARGUMENT, "npc_poly_set_lowrank: null V");
    NPC_GUARD(p <= poly->op->op->n_global, NPC_ERR_DIMENSION, "npc_poly_set_lowrank: p > n");
    DeviceScope ds(poly->op->owner->ctx.device);
    return set_lowrank(poly, p, V_dev);
}

npc_status npc_ritz_vectors(npc_operator op, int nsteps, int p, const double *v0_dev, double *V_dev,
                            double *theta_out) {
    NPC_GUARD(op && theta_out, NPC_ERR_INVALID_ARGUMENT, "npc_ritz_vectors: null argument");
    ErrScope es(op->owner);
    NPC_GUARD(p >= 1 && p <= NPC_LOWRANK_MAX, NPC_ERR_INVALID_ARGUMENT, "npc_ritz_vectors: p %d not in [1, %d]", p,
              NPC_LOWRANK_MAX);
    NPC_GUARD(nsteps >= p && nsteps <= 4096, NPC_ERR_INVALID_ARGUMENT, "npc_ritz_vectors: nsteps %d not in [p, 4096]",
              nsteps);
    NPC_GUARD(op->op->n_local == 0 || V_dev, NPC_ERR_INVALID_ARGUMENT, "npc_ritz_vectors: null V");
    NPC_GUARD(op->op->n_global >= nsteps, NPC_ERR_DIMENSION, "npc_ritz_vectors: nsteps > n");
    DeviceScope ds(op->owner->ctx.device);
    return ritz_vectors(op->op.get(), nsteps, p, v0_dev, V_dev, theta_out);
}

npc_status npc_destroy_poly(npc_poly poly) {
    if (!poly) return NPC_SUCCESS;
    {
        DeviceScope ds(poly->device);
        cudaDeviceSynchronize();
        poly->tmp.release();
        poly->tmp2.release();
        poly->coef_dev.release();
        poly->rin.release();
        poly->zout.release();
        poly->lr_V.release();
        poly->lr_Ginv.release();
        poly->lr_scratch.release();
    }
    delete poly;
    return NPC_SUCCESS;
}

npc_status npc_apply_poly(npc_poly poly, const double *r_dev, double *z_dev) {
    NPC_GUARD(poly, NPC_ERR_INVALID_ARGUMENT, "npc_apply_poly: null poly");
    ErrScope es(poly->op->owner);
    const int n = poly->op->op->n_local;
    NPC_GUARD(n == 0 || (r_dev && z_dev), NPC_ERR_INVALID_ARGUMENT, "npc_apply_poly: null vector");
    NPC_GUARD(n == 0 || r_dev != z_dev, NPC_ERR_INVALID_ARGUMENT, "npc_apply_poly: z must not alias r");
    DeviceScope ds(poly->op->owner->ctx.device);
    return apply_poly(poly, r_dev, z_dev);
}

npc_status npc_pcg_solve(npc_poly poly, npc_operator op, const double *b_dev, double *x_dev, double tol, int maxit,
                         npc_pcg_stats *stats) {
    NPC_GUARD(op, NPC_ERR_INVALID_ARGUMENT, "npc_pcg_solve: null operator");
    ErrScope es(op->owner);
    NPC_GUARD(!poly || poly->op == op, NPC_ERR_INVALID_ARGUMENT, "npc_pcg_solve: poly built for another operator");
    NPC_GUARD(tol > 0.0 && tol < 1.0, NPC_ERR_INVALID_ARGUMENT, "npc_pcg_solve: tol %g not in (0,1)", tol);
    NPC_GUARD(maxit >= 1, NPC_ERR_INVALID_ARGUMENT, "npc_pcg_solve: maxit %d < 1", maxit);
    NPC_GUARD(op->op->n_local == 0 || (b_dev && x_dev), NPC_ERR_INVALID_ARGUMENT, "npc_pcg_solve: null vector");
    NPC_GUARD(op->op->n_local == 0 || b_dev != x_dev, NPC_ERR_INVALID_ARGUMENT, "npc_pcg_solve: x aliases b");
    DeviceScope ds(op->owner->ctx.device);
    return pcg(poly, op, b_dev, x_dev, tol, maxit, stats);
}

npc_status npc_halo_plan(int n_local, const int *rowptr, const int *colidx, int nranks, const long long *row_starts,
                         int rank, int *n_ghost, long long *ghost_ids, int *recv_counts) {
    NPC_GUARD(rowptr && n_ghost && row_starts && (colidx || rowptr[n_local] == 0), NPC_ERR_INVALID_ARGUMENT,
              "npc_halo_plan: null argument");
    HaloPlan plan;
    NPC_TRY(halo_plan_local(n_local, rowptr, colidx, nranks, row_starts, rank, plan));
    const int cap = *n_ghost;
    *n_ghost = plan.n_ghost;
    if (ghost_ids) {
        NPC_GUARD(cap >= plan.n_ghost, NPC_ERR_INVALID_ARGUMENT, "npc_halo_plan: ghost_ids capacity %d < %d", cap,
                  plan.n_ghost);
        std::copy(plan.ghost_ids.begin(), plan.ghost_ids.end(), ghost_ids);
    }
    if (recv_counts) std::copy(plan.recv_count.begin(), plan.recv_count.end(), recv_counts);
    return NPC_SUCCESS;
}

}  // extern "C"
