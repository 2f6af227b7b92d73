// halo.cu -- row-block partition halo plan and per-application ghost exchange.
//
// The paper's DSMat (Fig. DSMat) stripes consecutive rows over MPI
// ranks and receives "the components of the distributed vector r that correspond to the
// column indices of the extra diagonal CSR blocks", overlapping the transfer with the local
// block product.  Here: one GPU per rank, ghosts sorted by global id
// (so the ghosts owned by one peer are contiguous in the ghost buffer and arrive with one
// ncclRecv), send lists fixed at create time, transfers on a dedicated comm stream.
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

npc_status halo_plan_exchange(Context *ctx, long long row_begin, HaloPlan &plan) {
    const int P = ctx->nranks;
    // 1) counts: all-to-all of recv_count -> send_count (via allgather of the full matrix)
    DevBuf cnt;
    NPC_TRY(cnt.alloc(sizeof(int) * P * P));
    NPC_CUDA_TRY(cudaMemcpyAsync(cnt.as<int>() + (size_t)ctx->rank * P, plan.recv_count.data(), sizeof(int) * P,
                                 cudaMemcpyHostToDevice, ctx->stream));
    NPC_NCCL_TRY(ncclAllGather(cnt.as<int>() + (size_t)ctx->rank * P, cnt.as<int>(), P, ncclInt32, ctx->comm, ctx->stream));
    std::vector<int> all((size_t)P * P);
    NPC_CUDA_TRY(cudaMemcpyAsync(all.data(), cnt.p, sizeof(int) * P * P, cudaMemcpyDeviceToHost, ctx->stream));
    NPC_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    plan.send_count.assign(P, 0);
    plan.send_off.assign(P, 0);
    for (int q = 0; q < P; ++q) plan.send_count[q] = all[(size_t)q * P + ctx->rank];
    for (int q = 1; q < P; ++q) plan.send_off[q] = plan.send_off[q - 1] + plan.send_count[q - 1];
    const int nsend = plan.send_off[P - 1] + plan.send_count[P - 1];
    // 2) ids: send my ghost ids to their owners, receive the ids peers need from me
    DevBuf gid, sid;
    NPC_TRY(gid.alloc(sizeof(long long) * std::max(plan.n_ghost, 1)));
    NPC_TRY(sid.alloc(sizeof(long long) * std::max(nsend, 1)));
    if (plan.n_ghost)
        NPC_CUDA_TRY(cudaMemcpyAsync(gid.p, plan.ghost_ids.data(), sizeof(long long) * plan.n_ghost,
                                     cudaMemcpyHostToDevice, ctx->stream));
    NPC_NCCL_TRY(ncclGroupStart());
    for (int q = 0; q < P; ++q) {
        if (q == ctx->rank) continue;
        if (plan.recv_count[q])
            NPC_NCCL_TRY(ncclSend(gid.as<long long>() + plan.recv_off[q], plan.recv_count[q], ncclInt64, q, ctx->comm,
                                  ctx->stream));
        if (plan.send_count[q])
            NPC_NCCL_TRY(ncclRecv(sid.as<long long>() + plan.send_off[q], plan.send_count[q], ncclInt64, q, ctx->comm,
                                  ctx->stream));
    }
    NPC_NCCL_TRY(ncclGroupEnd());
    std::vector<long long> ids(std::max(nsend, 1));
    NPC_CUDA_TRY(cudaMemcpyAsync(ids.data(), sid.p, sizeof(long long) * nsend, cudaMemcpyDeviceToHost, ctx->stream));
    NPC_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    plan.send_idx.resize(nsend);
    for (int i = 0; i < nsend; ++i) plan.send_idx[i] = (int)(ids[i] - row_begin);
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

npc_status halo_start(Context *ctx, const HaloPlan &plan, HaloRuntime &rt, const double *x) {
    const int P = ctx->nranks;
    NPC_TRY(launch_gather(ctx, x, rt.send_idx.as<int>(), rt.send_buf.as<double>(), (int)plan.send_idx.size()));
    NPC_CUDA_TRY(cudaEventRecord(rt.packed, ctx->stream));
    NPC_CUDA_TRY(cudaStreamWaitEvent(ctx->comm_stream, rt.packed, 0));
    NPC_NCCL_TRY(ncclGroupStart());
    for (int q = 0; q < P; ++q) {
        if (q == ctx->rank) continue;
        if (plan.send_count[q])
            NPC_NCCL_TRY(ncclSend(rt.send_buf.as<double>() + plan.send_off[q], plan.send_count[q], ncclDouble, q,
                                  ctx->comm, ctx->comm_stream));
        if (plan.recv_count[q])
            NPC_NCCL_TRY(ncclRecv(rt.ghost_buf.as<double>() + plan.recv_off[q], plan.recv_count[q], ncclDouble, q,
                                  ctx->comm, ctx->comm_stream));
    }
    NPC_NCCL_TRY(ncclGroupEnd());
    NPC_CUDA_TRY(cudaEventRecord(rt.ready, ctx->comm_stream));
    return NPC_SUCCESS;
}

npc_status halo_wait(Context *ctx, HaloRuntime &rt) {
    NPC_CUDA_TRY(cudaStreamWaitEvent(ctx->stream, rt.ready, 0));
    return NPC_SUCCESS;
}

}  // namespace npc
