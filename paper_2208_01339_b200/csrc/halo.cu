// halo.cu -- row-block partition halo plan and per-application ghost exchange.
//
// The paper's DSMat (Fig. DSMat) stripes consecutive rows over MPI
// ranks and receives "the components of the distributed vector r that correspond to the
// column indices of the extra diagonal CSR blocks", overlapping the transfer with the local
// block product.  Here: one GPU per rank, ghosts sorted by global id
// (so the ghosts owned by one peer are contiguous in the ghost buffer and arrive with one
// receive), send lists fixed at create time, transfers on a dedicated comm stream through
// the context's transport (NCCL; or the local thread-group transport used for testing).
#include <algorithm>

#include "npc_internal.cuh"

namespace npc {

npc_status halo_plan_local(int n_local, const int *rowptr, const int *colidx, int nranks, const long long *row_starts,
                           int rank, HaloPlan &plan) {
    if (n_local < 0 || nranks < 1 || rank < 0 || rank >= nranks || !rowptr || !row_starts) {
        set_error("halo_plan: invalid arguments");
        return NPC_ERR_INVALID_ARGUMENT;
    }
    for (int q = 0; q < nranks; ++q)
        if (row_starts[q + 1] < row_starts[q]) {
            set_error("halo_plan: row_starts not monotone");
            return NPC_ERR_DIMENSION;
        }
    const long long r0 = row_starts[rank], r1 = row_starts[rank + 1];
    if (r1 - r0 != n_local) {
        set_error("halo_plan: row_starts disagree with n_local");
        return NPC_ERR_DIMENSION;
    }
    const long long nglob = row_starts[nranks];
    std::vector<long long> g;
    const long long nnz = rowptr[n_local];
    for (long long p = 0; p < nnz; ++p) {
        long long c = colidx[p];
        if (c < 0 || c >= nglob) {
            set_error("halo_plan: column %lld out of range", c);
            return NPC_ERR_DIMENSION;
        }
        if (c < r0 || c >= r1) g.push_back(c);
    }
    std::sort(g.begin(), g.end());
    g.erase(std::unique(g.begin(), g.end()), g.end());
    plan.ghost_ids = g;
    plan.n_ghost = (int)g.size();
    plan.recv_count.assign(nranks, 0);
    plan.recv_off.assign(nranks, 0);
    int q = 0;
    for (size_t i = 0; i < g.size(); ++i) {
        while (g[i] >= row_starts[q + 1]) ++q;
        plan.recv_count[q]++;
    }
    for (int k = 1; k < nranks; ++k) plan.recv_off[k] = plan.recv_off[k - 1] + plan.recv_count[k - 1];
    return NPC_SUCCESS;
}

// Plan from an arbitrary list of referenced global ids (any row space; duplicates and owned
// ids allowed): ghosts = the sorted distinct ids outside [row_starts[rank], row_starts[rank+1]).
npc_status halo_plan_from_ids(std::vector<long long> ids, int nranks, const long long *row_starts, int rank,
                              HaloPlan &plan) {
    const long long r0 = row_starts[rank], r1 = row_starts[rank + 1], nglob = row_starts[nranks];
    std::vector<long long> g;
    for (long long c : ids) {
        if (c < 0 || c >= nglob) {
            set_error("halo_plan: id %lld out of range", c);
            return NPC_ERR_DIMENSION;
        }
        if (c < r0 || c >= r1) g.push_back(c);
    }
    std::sort(g.begin(), g.end());
    g.erase(std::unique(g.begin(), g.end()), g.end());
    plan.ghost_ids = g;
    plan.n_ghost = (int)g.size();
    plan.recv_count.assign(nranks, 0);
    plan.recv_off.assign(nranks, 0);
    int q = 0;
    for (size_t i = 0; i < g.size(); ++i) {
        while (g[i] >= row_starts[q + 1]) ++q;
        plan.recv_count[q]++;
    }
    for (int k = 1; k < nranks; ++k) plan.recv_off[k] = plan.recv_off[k - 1] + plan.recv_count[k - 1];
    return NPC_SUCCESS;
}

// Turn every rank's recv lists (ghost ids, by owner) into the owners' send lists.
npc_status halo_plan_exchange(Context *ctx, long long row_begin, HaloPlan &plan) {
    const int P = ctx->nranks;
    std::vector<int> all;
    NPC_TRY(ctx->tr->allgather_i32v(ctx, plan.recv_count, all));
    plan.send_count.assign(P, 0);
    plan.send_off.assign(P, 0);
    for (int q = 0; q < P; ++q) plan.send_count[q] = all[(size_t)q * P + ctx->rank];
    for (int q = 1; q < P; ++q) plan.send_off[q] = plan.send_off[q - 1] + plan.send_count[q - 1];
    const int nsend = plan.send_off[P - 1] + plan.send_count[P - 1];
    // my ghost ids go to their owners; I receive the ids the peers need from me
    std::vector<long long> ids(nsend);
    std::vector<long long> mine(plan.ghost_ids);
    std::vector<int> rc(plan.recv_count), ro(plan.recv_off);
    rc[ctx->rank] = 0;
    NPC_TRY(ctx->tr->alltoallv_i64(ctx, mine, rc, ro, ids, plan.send_count, plan.send_off));
    plan.send_idx.resize(nsend);
    for (int i = 0; i < nsend; ++i) {
        const long long li = ids[i] - row_begin;
        if (li < 0 || li >= (1LL << 31)) {
            set_error("halo plan: peer asked for row %lld not owned here", ids[i]);
            return NPC_ERR_DIMENSION;
        }
        plan.send_idx[i] = (int)li;
    }
    return NPC_SUCCESS;
}

HaloRuntime::~HaloRuntime() {
    if (packed) cudaEventDestroy(packed);
    if (ready) cudaEventDestroy(ready);
}

npc_status halo_setup(Context *ctx, const HaloPlan &plan, HaloRuntime &rt) {
    (void)ctx;
    const size_t ns = plan.send_idx.size();
    NPC_TRY(rt.send_idx.alloc(sizeof(int) * std::max<size_t>(ns, 1)));
    NPC_TRY(rt.send_buf.alloc(sizeof(double) * std::max<size_t>(ns, 1)));
    NPC_TRY(rt.ghost_buf.alloc(sizeof(double) * std::max(plan.n_ghost, 1)));
    if (ns) NPC_CUDA_TRY(cudaMemcpy(rt.send_idx.p, plan.send_idx.data(), sizeof(int) * ns, cudaMemcpyHostToDevice));
    NPC_CUDA_TRY(cudaEventCreateWithFlags(&rt.packed, cudaEventDisableTiming));
    NPC_CUDA_TRY(cudaEventCreateWithFlags(&rt.ready, cudaEventDisableTiming));
    return NPC_SUCCESS;
}

// Pack x[send_idx] on the compute stream, then send/recv on the comm stream (overlapping the
// interior kernels the caller enqueues next); halo_wait joins before the boundary kernels.
// Both transports (NCCL, and the local thread group used for testing) run this same
// choreography.
npc_status halo_start(Context *ctx, const HaloPlan &plan, HaloRuntime &rt, const double *x, double *recv) {
    NvtxRange nv("npc:halo");
    NPC_TRY(ctx->tr->before_pack(ctx, ctx->stream));
    NPC_TRY(launch_gather(ctx, x, rt.send_idx.as<int>(), rt.send_buf.as<double>(), (int)plan.send_idx.size()));
    NPC_CUDA_TRY(cudaEventRecord(rt.packed, ctx->stream));
    NPC_CUDA_TRY(cudaStreamWaitEvent(ctx->comm_stream, rt.packed, 0));
    NPC_TRY(ctx->tr->exchange(ctx, rt.send_buf.as<double>(), plan.send_count, plan.send_off,
                              recv ? recv : rt.ghost_buf.as<double>(),
                              plan.recv_count, plan.recv_off, ctx->comm_stream));
    NPC_CUDA_TRY(cudaEventRecord(rt.ready, ctx->comm_stream));
    return NPC_SUCCESS;
}

npc_status halo_wait(Context *ctx, HaloRuntime &rt) {
    NPC_CUDA_TRY(cudaStreamWaitEvent(ctx->stream, rt.ready, 0));
    return NPC_SUCCESS;
}

}  // namespace npc
