// transport.cu -- the collectives the multi-rank path needs, behind one interface:
//   * NcclTransport: one process per GPU, NCCL over NVLink/NVSwitch (the product path);
//   * LocalTransport: ranks are host threads of ONE process (any GPUs, including one GPU
//     shared by all ranks), exchanging through host barriers and device-to-device copies.
//     It exists so the multi-rank code (partition, ghost remap, interior/boundary tiles,
//     distributed Lanczos and PCG) can be run and checked on a single B200; ranks never wait
//     on one another on the device (every wait is a host barrier after a stream sync), so it
//     is safe to run several ranks on one GPU.  It is not captured into CUDA graphs.
#include <chrono>
#include <condition_variable>
#include <cstdlib>
#include <map>
#include <mutex>

#include "npc_internal.cuh"

namespace npc {

npc_status Transport::sync(Context *c, cudaStream_t s) {
    (void)c;
    NPC_CUDA_TRY(cudaStreamSynchronize(s));
    return NPC_SUCCESS;
}

npc_status stream_sync(Context *c, cudaStream_t s) {
    if (c->tr) return c->tr->sync(c, s);
    NPC_CUDA_TRY(cudaStreamSynchronize(s));
    return NPC_SUCCESS;
}

static double nccl_timeout_s() {
    static const double t = [] {
        const char *e = getenv("NPC_NCCL_TIMEOUT_S");
        const double v = e ? atof(e) : 600.0;
        return v > 0 ? v : 600.0;
    }();
    return t;
}

// ================================================================== NCCL
class NcclTransport : public Transport {
  public:
    ncclComm_t comm = nullptr;
    ncclComm_t comm_aux = nullptr;  // split of comm: the PCG ||r||^2 allreduce on the side stream
    ~NcclTransport() override {
        if (comm_aux) ncclCommDestroy(comm_aux);
        if (comm) ncclCommDestroy(comm);
    }
    npc_status live() const {
        if (comm) return NPC_SUCCESS;
        set_error("NCCL communicator was aborted by an earlier error");
        return NPC_ERR_NCCL;
    }
    bool capturable() const override { return true; }
    bool aborted = false;

    // Wait for s while polling both communicators' asynchronous error state (NCCL reports a
    // failed peer, network error or internal error there, while the stream would otherwise never
    // drain); on an error or after the timeout the communicators are aborted -- their pending
    // operations are cancelled so the stream drains -- and the call fails with NPC_ERR_NCCL.
    npc_status sync(Context *c, cudaStream_t s) override {
        (void)c;
        if (aborted) {
            set_error("NCCL communicator was aborted by an earlier error");
            return NPC_ERR_NCCL;
        }
        const auto t0 = std::chrono::steady_clock::now();
        for (int spin = 0;; ++spin) {
            const cudaError_t e = cudaStreamQuery(s);
            if (e == cudaSuccess) return NPC_SUCCESS;
            if (e != cudaErrorNotReady) {
                set_error("stream wait: %s", cudaGetErrorString(e));
                return NPC_ERR_CUDA;
            }
            ncclResult_t r1 = ncclSuccess, r2 = ncclSuccess;
            ncclCommGetAsyncError(comm, &r1);
            if (comm_aux) ncclCommGetAsyncError(comm_aux, &r2);
            const double dt = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
            const bool bad = (r1 != ncclSuccess && r1 != ncclInProgress) || (r2 != ncclSuccess && r2 != ncclInProgress);
            if (bad || dt > nccl_timeout_s()) {
                aborted = true;
                if (comm_aux) ncclCommAbort(comm_aux);
                ncclCommAbort(comm);
                comm_aux = nullptr;
                comm = nullptr;
                if (bad)
                    set_error("NCCL asynchronous error: %s (communicators aborted)",
                              ncclGetErrorString(r1 != ncclSuccess ? r1 : r2));
                else
                    set_error("NCCL wait exceeded NPC_NCCL_TIMEOUT_S = %.0f s (communicators aborted)",
                              nccl_timeout_s());
                return NPC_ERR_NCCL;
            }
            if (spin > 64) std::this_thread::sleep_for(std::chrono::microseconds(20));
        }
    }

    npc_status allgather_i64(Context *c, long long mine, std::vector<long long> &all) override {
        const int P = c->nranks;
        DevBuf d;
        NPC_TRY(d.alloc(sizeof(long long) * P));
        NPC_CUDA_TRY(cudaMemcpyAsync(d.as<long long>() + c->rank, &mine, sizeof(long long), cudaMemcpyHostToDevice,
                                     c->stream));
        NPC_NCCL_TRY(ncclAllGather(d.as<long long>() + c->rank, d.as<long long>(), 1, ncclInt64, comm, c->stream));
        all.resize(P);
        NPC_CUDA_TRY(cudaMemcpyAsync(all.data(), d.p, sizeof(long long) * P, cudaMemcpyDeviceToHost, c->stream));
        NPC_TRY(sync(c, c->stream));
        return NPC_SUCCESS;
    }
    npc_status allgather_i32v(Context *c, const std::vector<int> &mine, std::vector<int> &all) override {
        const int P = c->nranks, m = (int)mine.size();
        DevBuf d;
        NPC_TRY(d.alloc(sizeof(int) * (size_t)P * m));
        NPC_CUDA_TRY(cudaMemcpyAsync(d.as<int>() + (size_t)c->rank * m, mine.data(), sizeof(int) * m,
                                     cudaMemcpyHostToDevice, c->stream));
        NPC_NCCL_TRY(ncclAllGather(d.as<int>() + (size_t)c->rank * m, d.as<int>(), m, ncclInt32, comm, c->stream));
        all.resize((size_t)P * m);
        NPC_CUDA_TRY(cudaMemcpyAsync(all.data(), d.p, sizeof(int) * P * m, cudaMemcpyDeviceToHost, c->stream));
        NPC_TRY(sync(c, c->stream));
        return NPC_SUCCESS;
    }
    npc_status alltoallv_i64(Context *c, const std::vector<long long> &sbuf, const std::vector<int> &scount,
                             const std::vector<int> &soff, std::vector<long long> &rbuf,
                             const std::vector<int> &rcount, const std::vector<int> &roff) override {
        const int P = c->nranks;
        DevBuf ds, dr;
        NPC_TRY(ds.alloc(sizeof(long long) * std::max<size_t>(sbuf.size(), 1)));
        NPC_TRY(dr.alloc(sizeof(long long) * std::max<size_t>(rbuf.size(), 1)));
        if (!sbuf.empty())
            NPC_CUDA_TRY(cudaMemcpyAsync(ds.p, sbuf.data(), sizeof(long long) * sbuf.size(), cudaMemcpyHostToDevice,
                                         c->stream));
        NPC_NCCL_TRY(ncclGroupStart());
        for (int q = 0; q < P; ++q) {
            if (q == c->rank) continue;
            if (scount[q])
                NPC_NCCL_TRY(ncclSend(ds.as<long long>() + soff[q], scount[q], ncclInt64, q, comm, c->stream));
            if (rcount[q])
                NPC_NCCL_TRY(ncclRecv(dr.as<long long>() + roff[q], rcount[q], ncclInt64, q, comm, c->stream));
        }
        NPC_NCCL_TRY(ncclGroupEnd());
        if (!rbuf.empty())
            NPC_CUDA_TRY(cudaMemcpyAsync(rbuf.data(), dr.p, sizeof(long long) * rbuf.size(), cudaMemcpyDeviceToHost,
                                         c->stream));
        NPC_TRY(sync(c, c->stream));
        return NPC_SUCCESS;
    }
    npc_status exchange(Context *c, const double *sbuf, const std::vector<int> &scount, const std::vector<int> &soff,
                        double *rbuf, const std::vector<int> &rcount, const std::vector<int> &roff,
                        cudaStream_t s) override {
        NPC_TRY(live());
        NPC_NCCL_TRY(ncclGroupStart());
        for (int q = 0; q < c->nranks; ++q) {
            if (q == c->rank) continue;
            if (scount[q]) NPC_NCCL_TRY(ncclSend(sbuf + soff[q], scount[q], ncclDouble, q, comm, s));
            if (rcount[q]) NPC_NCCL_TRY(ncclRecv(rbuf + roff[q], rcount[q], ncclDouble, q, comm, s));
        }
        NPC_NCCL_TRY(ncclGroupEnd());
        return NPC_SUCCESS;
    }
    npc_status allreduce_sum(Context *c, double *dev, int count, cudaStream_t s) override {
        (void)c;
        NPC_TRY(live());
        NvtxRange nv("npc:allreduce");
        NPC_NCCL_TRY(ncclAllReduce(dev, dev, count, ncclDouble, ncclSum, comm, s));
        return NPC_SUCCESS;
    }
    npc_status allreduce_sum_aux(Context *c, double *dev, int count, cudaStream_t s) override {
        (void)c;
        NPC_TRY(live());
        NPC_NCCL_TRY(ncclAllReduce(dev, dev, count, ncclDouble, ncclSum, comm_aux, s));
        return NPC_SUCCESS;
    }
    npc_status allgather_slots(Context *c, double *full, int m, const std::vector<int> &counts,
                               cudaStream_t s) override {
        (void)counts;
        NPC_TRY(live());
        NPC_NCCL_TRY(ncclAllGather(full + (size_t)c->rank * m, full, m, ncclDouble, comm, s));
        return NPC_SUCCESS;
    }
    npc_status reduce_scatter_slots(Context *c, const double *full, double *mine, int m, cudaStream_t s) override {
        (void)c;
        NPC_TRY(live());
        NPC_NCCL_TRY(ncclReduceScatter(full, mine, m, ncclDouble, ncclSum, comm, s));
        return NPC_SUCCESS;
    }
};

npc_status make_nccl_transport(Context *c, const void *uid, std::unique_ptr<Transport> &out) {
    auto t = std::make_unique<NcclTransport>();
    ncclUniqueId id;
    memcpy(&id, uid, sizeof(id));
    NPC_NCCL_TRY(ncclCommInitRank(&t->comm, c->nranks, id, c->rank));
    NPC_NCCL_TRY(ncclCommSplit(t->comm, 0, c->rank, &t->comm_aux, nullptr));
    out = std::move(t);
    return NPC_SUCCESS;
}

// ================================================================== local thread group
struct LocalGroup {
    int nranks;
    std::mutex mu;
    std::condition_variable cv;
    int arrived = 0;
    long long generation = 0;
    std::vector<const void *> slot;     // per-rank published pointer (host or device)
    std::vector<const void *> slot2;    // second pointer (offsets / counts)
    std::vector<int> slot_device;
    std::vector<cudaEvent_t> ev_packed, ev_copied;  // per rank (exchange ordering, see below)
    bool aborted = false;
    explicit LocalGroup(int n)
        : nranks(n), slot(n, nullptr), slot2(n, nullptr), slot_device(n, 0), ev_packed(n, nullptr),
          ev_copied(n, nullptr) {}
    // false if the group was aborted (a rank left) or the wait timed out
    bool barrier() {
        std::unique_lock<std::mutex> lk(mu);
        if (aborted) return false;
        const long long gen = generation;
        if (++arrived == nranks) {
            arrived = 0;
            ++generation;
            cv.notify_all();
            return true;
        }
        const bool ok = cv.wait_for(lk, std::chrono::seconds(90), [&] { return generation != gen || aborted; });
        if (generation != gen) return true;  // released normally (even if aborted since)
        if (!ok) aborted = true;
        if (aborted) cv.notify_all();
        return !aborted;
    }
    void abort() {
        std::lock_guard<std::mutex> lk(mu);
        aborted = true;
        cv.notify_all();
    }
};

#define NPC_BARRIER(g)                                                                   \
    do {                                                                                 \
        if (!(g)->barrier()) {                                                           \
            set_error("local group aborted (a rank failed, left, or timed out)");        \
            return NPC_ERR_INVALID_ARGUMENT;                                             \
        }                                                                                \
    } while (0)

static std::mutex g_groups_mu;
static std::map<std::string, std::weak_ptr<LocalGroup>> g_groups;

// A failing rank aborts the group so that its peers leave their barriers with an error.
#define LT_CUDA_TRY(expr)                                                                          \
    do {                                                                                           \
        cudaError_t e_ = (expr);                                                                   \
        if (e_ != cudaSuccess) {                                                                   \
            g->abort();                                                                            \
            npc::set_error("%s:%d: %s -> %s", __FILE__, __LINE__, #expr, cudaGetErrorString(e_));    \
            return NPC_ERR_CUDA;                                                                   \
        }                                                                                          \
    } while (0)

class LocalTransport : public Transport {
  public:
    std::shared_ptr<LocalGroup> g;
    DevBuf stage;  // reduce_scatter_slots: the P contributions to this rank's slot
    int rank = 0;
    cudaEvent_t ev_packed = nullptr, ev_copied = nullptr;
    bool exchanged = false;  // a previous exchange's copies may still read my send buffer
    ~LocalTransport() override {
        if (g) g->abort();  // a rank leaving releases peers still waiting for it
        if (ev_packed) cudaEventDestroy(ev_packed);
        if (ev_copied) cudaEventDestroy(ev_copied);
    }
    bool capturable() const override { return false; }

    // The next pack overwrites my send buffer: wait (on the device) for every peer's copies of
    // the previous exchange.  Those events were recorded before that exchange's second host
    // barrier, and no peer can re-record them before I reach the next exchange.
    npc_status before_pack(Context *c, cudaStream_t s) override {
        if (!exchanged) return NPC_SUCCESS;
        for (int q = 0; q < c->nranks; ++q)
            if (q != c->rank && g->ev_copied[q]) LT_CUDA_TRY(cudaStreamWaitEvent(s, g->ev_copied[q], 0));
        return NPC_SUCCESS;
    }

    npc_status allgather_i64(Context *c, long long mine, std::vector<long long> &all) override {
        g->slot[c->rank] = &mine;
        NPC_BARRIER(g);
        all.resize(c->nranks);
        for (int q = 0; q < c->nranks; ++q) all[q] = *static_cast<const long long *>(g->slot[q]);
        NPC_BARRIER(g);
        return NPC_SUCCESS;
    }
    npc_status allgather_i32v(Context *c, const std::vector<int> &mine, std::vector<int> &all) override {
        g->slot[c->rank] = mine.data();
        NPC_BARRIER(g);
        const size_t m = mine.size();
        all.resize((size_t)c->nranks * m);
        for (int q = 0; q < c->nranks; ++q)
            memcpy(all.data() + (size_t)q * m, g->slot[q], sizeof(int) * m);
        NPC_BARRIER(g);
        return NPC_SUCCESS;
    }
    npc_status alltoallv_i64(Context *c, const std::vector<long long> &sbuf, const std::vector<int> &scount,
                             const std::vector<int> &soff, std::vector<long long> &rbuf,
                             const std::vector<int> &rcount, const std::vector<int> &roff) override {
        (void)scount;
        g->slot[c->rank] = sbuf.data();
        g->slot2[c->rank] = soff.data();
        NPC_BARRIER(g);
        for (int q = 0; q < c->nranks; ++q) {
            if (q == c->rank || !rcount[q]) continue;
            const long long *src = static_cast<const long long *>(g->slot[q]);
            const int *qoff = static_cast<const int *>(g->slot2[q]);
            memcpy(rbuf.data() + roff[q], src + qoff[c->rank], sizeof(long long) * rcount[q]);
        }
        NPC_BARRIER(g);
        return NPC_SUCCESS;
    }
    // Asynchronous, like NCCL send/recv on the comm stream: the host threads meet at two
    // barriers only to publish pointers and events; on the device every copy waits for its
    // source rank's "packed" event, and each rank's "copied" event orders its peers' next pack
    // (before_pack).  No stream of any rank is synchronised and no kernel waits for another
    // rank's kernel (stream-ordered event waits only), so several ranks may share one GPU and
    // the interior tiles of every rank overlap the exchange as they do over NCCL.
    npc_status exchange(Context *c, const double *sbuf, const std::vector<int> &scount, const std::vector<int> &soff,
                        double *rbuf, const std::vector<int> &rcount, const std::vector<int> &roff,
                        cudaStream_t s) override {
        (void)scount;
        NvtxRange nv("npc:halo");
        LT_CUDA_TRY(cudaEventRecord(ev_packed, s));  // s already waits for the pack
        g->slot[c->rank] = sbuf;
        g->slot2[c->rank] = soff.data();
        g->slot_device[c->rank] = c->device;
        NPC_BARRIER(g);
        for (int q = 0; q < c->nranks; ++q) {
            if (q == c->rank || !rcount[q]) continue;
            const double *src = static_cast<const double *>(g->slot[q]);
            const int *qoff = static_cast<const int *>(g->slot2[q]);
            LT_CUDA_TRY(cudaStreamWaitEvent(s, g->ev_packed[q], 0));
            if (g->slot_device[q] == c->device)
                LT_CUDA_TRY(cudaMemcpyAsync(rbuf + roff[q], src + qoff[c->rank], sizeof(double) * rcount[q],
                                             cudaMemcpyDeviceToDevice, s));
            else
                LT_CUDA_TRY(cudaMemcpyPeerAsync(rbuf + roff[q], c->device, src + qoff[c->rank], g->slot_device[q],
                                                 sizeof(double) * rcount[q], s));
        }
        LT_CUDA_TRY(cudaEventRecord(ev_copied, s));
        exchanged = true;
        NPC_BARRIER(g);  // every rank has enqueued its copies (the soff arrays may go)
        return NPC_SUCCESS;
    }
    npc_status allgather_slots(Context *c, double *full, int m, const std::vector<int> &counts,
                               cudaStream_t s) override {
        LT_CUDA_TRY(cudaStreamSynchronize(s));  // my slot is complete
        g->slot[c->rank] = full;
        g->slot_device[c->rank] = c->device;
        NPC_BARRIER(g);
        for (int q = 0; q < c->nranks; ++q) {
            if (q == c->rank || !counts[q]) continue;
            const double *src = static_cast<const double *>(g->slot[q]) + (size_t)q * m;
            if (g->slot_device[q] == c->device)
                LT_CUDA_TRY(cudaMemcpyAsync(full + (size_t)q * m, src, sizeof(double) * counts[q],
                                            cudaMemcpyDeviceToDevice, s));
            else
                LT_CUDA_TRY(cudaMemcpyPeerAsync(full + (size_t)q * m, c->device, src, g->slot_device[q],
                                                sizeof(double) * counts[q], s));
        }
        LT_CUDA_TRY(cudaStreamSynchronize(s));
        NPC_BARRIER(g);  // peers may now overwrite their buffers
        return NPC_SUCCESS;
    }
    npc_status reduce_scatter_slots(Context *c, const double *full, double *mine, int m, cudaStream_t s) override {
        const int P = c->nranks;
        if (stage.bytes < sizeof(double) * (size_t)P * m) NPC_TRY(stage.alloc(sizeof(double) * (size_t)P * m));
        LT_CUDA_TRY(cudaStreamSynchronize(s));
        g->slot[c->rank] = full;
        g->slot_device[c->rank] = c->device;
        NPC_BARRIER(g);
        double *st = stage.as<double>();
        for (int q = 0; q < P; ++q) {  // rank q's contribution to my slot -> stage row q
            const double *src = static_cast<const double *>(g->slot[q]) + (size_t)c->rank * m;
            if (g->slot_device[q] == c->device)
                LT_CUDA_TRY(cudaMemcpyAsync(st + (size_t)q * m, src, sizeof(double) * m, cudaMemcpyDeviceToDevice, s));
            else
                LT_CUDA_TRY(cudaMemcpyPeerAsync(st + (size_t)q * m, c->device, src, g->slot_device[q],
                                                sizeof(double) * m, s));
        }
        NPC_TRY(launch_sum_rows(c, st, P, m, mine, s));  // fixed rank order
        LT_CUDA_TRY(cudaStreamSynchronize(s));
        NPC_BARRIER(g);
        return NPC_SUCCESS;
    }
    npc_status allreduce_sum(Context *c, double *dev, int count, cudaStream_t s) override {
        std::vector<double> mine(count), sum(count, 0.0);
        LT_CUDA_TRY(cudaMemcpyAsync(mine.data(), dev, sizeof(double) * count, cudaMemcpyDeviceToHost, s));
        LT_CUDA_TRY(cudaStreamSynchronize(s));
        g->slot[c->rank] = mine.data();
        NPC_BARRIER(g);
        for (int q = 0; q < c->nranks; ++q) {  // fixed rank order: identical bits on every rank
            const double *v = static_cast<const double *>(g->slot[q]);
            for (int i = 0; i < count; ++i) sum[i] += v[i];
        }
        NPC_BARRIER(g);
        LT_CUDA_TRY(cudaMemcpyAsync(dev, sum.data(), sizeof(double) * count, cudaMemcpyHostToDevice, s));
        LT_CUDA_TRY(cudaStreamSynchronize(s));
        return NPC_SUCCESS;
    }
};

npc_status make_local_transport(Context *c, const char *group, std::unique_ptr<Transport> &out) {
    auto t = std::make_unique<LocalTransport>();
    t->rank = c->rank;
    NPC_CUDA_TRY(cudaEventCreateWithFlags(&t->ev_packed, cudaEventDisableTiming));
    NPC_CUDA_TRY(cudaEventCreateWithFlags(&t->ev_copied, cudaEventDisableTiming));
    {
        std::lock_guard<std::mutex> lk(g_groups_mu);
        auto &w = g_groups[group];
        t->g = w.lock();
        if (!t->g) {
            t->g = std::make_shared<LocalGroup>(c->nranks);
            w = t->g;
        } else if (t->g->nranks != c->nranks) {
            set_error("local group '%s' has %d ranks, not %d", group, t->g->nranks, c->nranks);
            return NPC_ERR_INVALID_ARGUMENT;
        }
        t->g->ev_packed[c->rank] = t->ev_packed;
        t->g->ev_copied[c->rank] = t->ev_copied;
    }
    out = std::move(t);
    return NPC_SUCCESS;
}

}  // namespace npc
