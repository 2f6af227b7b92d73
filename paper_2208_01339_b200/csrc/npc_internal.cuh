// npc_internal.cuh -- internal types of libnpc (not part of the C ABI).
//
// Layering: kernels (op_*.cu, vec_kernels.cu) <- operators (Operator
// subclasses) <- drivers (solvers.cu: apply_poly, PCG, Lanczos) <- C ABI (api.cu).
#pragma once

#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>
#include <nccl.h>
#include <stdint.h>

#include <algorithm>
#include <atomic>
#include <memory>
#include <thread>
#include <mutex>
#include <string>
#include <vector>

#include "npc.h"

namespace npc {

// ------------------------------------------------------------------ errors
void set_error(const char *fmt, ...);

#define NPC_CUDA_TRY(expr)                                                                     \
    do {                                                                                       \
        cudaError_t e_ = (expr);                                                               \
        if (e_ != cudaSuccess) {                                                               \
            npc::set_error("%s:%d: %s -> %s", __FILE__, __LINE__, #expr, cudaGetErrorString(e_)); \
            return e_ == cudaErrorMemoryAllocation ? NPC_ERR_OUT_OF_MEMORY : NPC_ERR_CUDA;     \
        }                                                                                      \
    } while (0)

#define NPC_NCCL_TRY(expr)                                                                     \
    do {                                                                                       \
        ncclResult_t e_ = (expr);                                                              \
        if (e_ != ncclSuccess) {                                                               \
            npc::set_error("%s:%d: %s -> %s", __FILE__, __LINE__, #expr, ncclGetErrorString(e_)); \
            return NPC_ERR_NCCL;                                                               \
        }                                                                                      \
    } while (0)

#define NPC_TRY(expr)                       \
    do {                                    \
        npc_status s_ = (expr);             \
        if (s_ != NPC_SUCCESS) return s_;   \
    } while (0)

// Count every kernel launch of the library (npc_launch_count) and check the launch.
extern std::atomic<unsigned long long> g_launches;
#define NPC_LAUNCH_CHECK()                                            \
    do {                                                              \
        npc::g_launches.fetch_add(1, std::memory_order_relaxed);      \
        NPC_CUDA_TRY(cudaGetLastError());                             \
    } while (0)

// ------------------------------------------------------------------ device buffers
// Device memory pool (pool.cu): blocks of >= 1 MiB are, when released, kept per device
// (keyed by their exact size) for reuse instead of being unmapped -- cudaMalloc/cudaFree of the PCG work vectors and Lanczos bases cost ~1 ms per
// solve on the bench configs.  A release first waits for the device (as cudaFree does), so a
// block is never handed out while a kernel may still touch it.  The cache is bounded
// (NPC_POOL_MB, default 16384) and flushed when cudaMalloc reports out-of-memory.
cudaError_t pool_alloc(void **p, size_t bytes);
void pool_free(void *p, size_t bytes);  // bytes as passed to pool_alloc

struct DevBuf {
    void *p = nullptr;
    size_t bytes = 0;
    DevBuf() = default;
    DevBuf(const DevBuf &) = delete;
    DevBuf &operator=(const DevBuf &) = delete;
    ~DevBuf() { release(); }
    void release() {
        if (p) pool_free(p, bytes);
        p = nullptr;
        bytes = 0;
    }
    npc_status alloc(size_t nbytes) {
        release();
        if (nbytes == 0) nbytes = 16;
        cudaError_t e = pool_alloc(&p, nbytes);
        if (e != cudaSuccess) {
            p = nullptr;
            set_error("cudaMalloc(%zu) failed: %s", nbytes, cudaGetErrorString(e));
            return e == cudaErrorMemoryAllocation ? NPC_ERR_OUT_OF_MEMORY : NPC_ERR_CUDA;
        }
        bytes = nbytes;
        return NPC_SUCCESS;
    }
    template <class T>
    T *as() const { return static_cast<T *>(p); }
};

// ------------------------------------------------------------------ the fused step
// One call = one application of A fused with the Chebyshev three-term update
// (PAPER.md:253-295):
//     out = a * (A x) + b * x + c * s2 + d * r
// optionally emitting per-block partials of <out, dotv> (the PCG inner products fused
// into the producing kernel).  s2 may alias out (in-place over s_{j-2}).
struct StepArgs {
    const double *x = nullptr;   // input of A: this rank's owned entries (internal order)
    const double *s2 = nullptr;  // nullable
    const double *r = nullptr;   // nullable
    double *out = nullptr;
    const double *dotv = nullptr;  // nullable -> no dot partials
    double *partials = nullptr;    // >= Operator::num_partials() doubles when dotv != null
    const int *done = nullptr;     // nullable device flag: when *done != 0 the kernels no-op
    double a = 1.0, b = 0.0, c = 0.0, d = 0.0;
};

// Fused degree-step epilogue o = a*y + b*x (+ c*s_{j-2}) (+ d*r) in ONE rounding order --
// a*y rounded, then one FMA per term in this order -- for every kernel of an operator family,
// whose storage forms are compared bitwise (the compiler's own contraction choice differs
// between kernels).
template <bool HAS_S2, bool HAS_R>
__device__ __forceinline__ double degree_epilogue(const StepArgs &s, double y, double x, double s2v, double rv) {
    double o = fma(s.b, x, __dmul_rn(s.a, y));
    if (HAS_S2) o = fma(s.c, s2v, o);
    if (HAS_R) o = fma(s.d, rv, o);
    return o;
}

struct Context;
struct ClusterPcgOut;

class Operator {
  public:
    virtual ~Operator() = default;
    // Enqueue one fused step on ctx->stream (including any halo exchange).
    virtual npc_status step(const StepArgs &s) = 0;
    // Number of per-block dot partials a step writes (grid of the last kernel).
    virtual int num_partials() const = 0;
    // Algorithmic bytes of one application + recurrence, for reporting.
    virtual double bytes_per_step(bool has_s2, bool has_r) const = 0;
    // Operator-data part of it, in the stored format (bytes_per_step minus x read + out write).
    virtual double matrix_bytes() const { return bytes_per_step(false, false) - 16.0 * n_local; }
    // Two consecutive degrees in one pass (temporal blocking, stencils): s1 produces s_j from
    // s_{j-1} = s1.x, s_{j-2} = s1.s2, r = s1.r into s1.out; s2 produces s_{j+1} into s2.out
    // (s2.x = s1.out, s2.s2 = s1.x implied) with the optional dot of s2.  Outputs must not
    // alias the inputs.
    virtual bool supports_step2() const { return false; }
    virtual npc_status step2(const StepArgs &s1, const StepArgs &s2) {
        (void)s1; (void)s2;
        return NPC_ERR_UNSUPPORTED;
    }
    virtual int num_partials2() const { return num_partials(); }
    // The whole polynomial in one launch (small CSR operators: csr_cluster.cu).  coef_dev is the
    // 4k table of npc_poly_coefficients; writes nparts partials of <z, dotv> when dotv != null.
    virtual bool supports_fused_poly() const { return false; }
    // All steps of the Lanczos estimate in one launch (small CSR operators, single rank);
    // v0 in internal order; writes alphas[m], betas[m] and the steps taken (device).
    virtual bool supports_fused_lanczos() const { return false; }
    virtual npc_status lanczos_fused(const double *v0, int m, double *alphas, double *betas, int *steps) {
        (void)v0; (void)m; (void)alphas; (void)betas; (void)steps;
        return NPC_ERR_UNSUPPORTED;
    }
    // The whole PCG solve in one launch (small CSR operators, single rank).
    virtual bool supports_fused_pcg() const { return false; }
    virtual npc_status pcg_fused(const double *b, double *x, const double *coef_dev, int k, double tb, int use_poly,
                                 double tol2b, int maxit, ClusterPcgOut *out, double *history) {
        (void)b; (void)x; (void)coef_dev; (void)k; (void)tb; (void)use_poly; (void)tol2b; (void)maxit; (void)out;
        (void)history;
        return NPC_ERR_UNSUPPORTED;
    }
    virtual npc_status apply_poly_fused(const double *r, double *z, const double *coef_dev, int k, double tb,
                                        const double *dotv, double *partials, int *nparts, const int *done) {
        (void)r; (void)z; (void)coef_dev; (void)k; (void)tb; (void)dotv; (void)partials; (void)nparts; (void)done;
        return NPC_ERR_UNSUPPORTED;
    }
    virtual double bytes_per_step2() const { return 0.0; }
    // Internal vector order differs from the caller's (SELL sigma-sort)?
    virtual bool permuted() const { return false; }
    // May its steps be stream-captured into a CUDA graph? (user callbacks: no)
    virtual bool capture_safe() const { return true; }
    // out[i] = in[perm[i]] (to internal) / out[perm[i]] = in[i] (to caller order).
    virtual npc_status to_internal(const double *in, double *out) { (void)in; (void)out; return NPC_SUCCESS; }
    virtual npc_status to_external(const double *in, double *out) { (void)in; (void)out; return NPC_SUCCESS; }

    Context *ctx = nullptr;
    npc_op_kind kind = NPC_OP_CSR;
    int n_local = 0;
    long long n_global = 0;
    long long row_begin = 0;
};

// ------------------------------------------------------------------ transport (transport.cu)
struct Context;
class Transport {
  public:
    virtual ~Transport() = default;
    virtual bool capturable() const = 0;  // may its calls be captured into a CUDA graph?
    // setup-time collectives on host data
    virtual npc_status allgather_i64(Context *c, long long mine, std::vector<long long> &all) = 0;
    virtual npc_status allgather_i32v(Context *c, const std::vector<int> &mine, std::vector<int> &all) = 0;
    virtual npc_status alltoallv_i64(Context *c, const std::vector<long long> &sbuf, const std::vector<int> &scount,
                                     const std::vector<int> &soff, std::vector<long long> &rbuf,
                                     const std::vector<int> &rcount, const std::vector<int> &roff) = 0;
    // per-application / per-iteration traffic on device buffers, enqueued on stream s
    virtual npc_status exchange(Context *c, const double *sbuf, const std::vector<int> &scount,
                                const std::vector<int> &soff, double *rbuf, const std::vector<int> &rcount,
                                const std::vector<int> &roff, cudaStream_t s) = 0;
    virtual npc_status allreduce_sum(Context *c, double *dev, int count, cudaStream_t s) = 0;
    // Same sum on an auxiliary channel that may run CONCURRENTLY with the transport's other
    // calls (NCCL: a split communicator); issued in the same order on every rank.
    virtual npc_status allreduce_sum_aux(Context *c, double *dev, int count, cudaStream_t s) {
        return allreduce_sum(c, dev, count, s);
    }
    // Padded-slot collectives of the Schur operator (slot q = [q m, q m + m) of a P*m buffer;
    // rank q's valid entries are the first counts[q] of its slot):
    //   allgather_slots: in place, every rank's slot is copied into every rank's buffer;
    //   reduce_scatter_slots: mine[0..m) = sum over ranks of their full[rank*m .. +m).
    virtual npc_status allgather_slots(Context *c, double *full, int m, const std::vector<int> &counts,
                                       cudaStream_t s) = 0;
    virtual npc_status reduce_scatter_slots(Context *c, const double *full, double *mine, int m,
                                            cudaStream_t s) = 0;
    // Host wait for stream s.  NCCL: polls the communicators' asynchronous error state while
    // waiting and aborts them (NPC_ERR_NCCL) on an error or after NPC_NCCL_TIMEOUT_S seconds
    // (default 600) -- a dead or wedged peer ends the call instead of hanging it.
    virtual npc_status sync(Context *c, cudaStream_t s);
    // Called on the compute stream before a halo pack overwrites the send buffer that peers
    // may still be reading (local transport: waits for their copies; NCCL: nothing).
    virtual npc_status before_pack(Context *c, cudaStream_t s) {
        (void)c, (void)s;
        return NPC_SUCCESS;
    }
};
// Host wait for stream s of context c (through the transport when distributed).
npc_status stream_sync(Context *c, cudaStream_t s);
npc_status make_nccl_transport(Context *c, const void *uid, std::unique_ptr<Transport> &out);
npc_status make_local_transport(Context *c, const char *group, std::unique_ptr<Transport> &out);

// ------------------------------------------------------------------ context
struct Context {
    int device = 0;
    int nranks = 1, rank = 0;
    cudaStream_t stream = nullptr;       // compute stream
    cudaStream_t comm_stream = nullptr;  // halo traffic (distributed contexts)
    cudaStream_t aux_stream = nullptr;   // PCG side ||r||^2 allreduce (distributed): never queues
                                         // behind (or holds up) the halo traffic on comm_stream
    bool own_stream = false;
    cudaStream_t graph_stream = nullptr;  // CUDA-graph replay of PCG iterations
    cudaStream_t body_stream = nullptr;   // capture of conditional iteration bodies
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    cudaEvent_t ev_rr0 = nullptr, ev_rr1 = nullptr;  // PCG side-stream ||r||^2 allreduce (distributed)
    std::unique_ptr<Transport> tr;       // distributed contexts: NCCL or a local thread group
    // Distributed context: created with a transport (any nranks >= 1, see include/npc.h). Every
    // operator and solver takes its multi-rank path (halo plans, collectives) iff this holds; a
    // 1-rank distributed context runs that path with empty halos and 1-rank collectives.
    bool distributed() const { return tr != nullptr; }
    int num_sms = 148;
    // scratch for reductions: partial arrays + scalar slots
    DevBuf partials;        // 4 slots of partial_cap doubles
    size_t partial_cap = 0;
    DevBuf scalars;         // small device scalar area (see solvers.cu)
    double *host_pinned = nullptr;  // pinned host mirror for small readbacks

    npc_status ensure_partials(size_t n);
    double *partial_slot(int i) { return partials.as<double>() + (size_t)i * partial_cap; }
    // Sum 'count' doubles at dev (in place) over all ranks (no-op on one rank).
    npc_status allreduce_sum(double *dev, int count);

    // ---- optional event timing (npc_context_set_timing)
    struct Pending {
        int cls;
        cudaEvent_t e0, e1;
        int count;  // launches (degree applications) the interval covers
    };
    // PCG on a distributed context: false (default) = {gamma, delta} on the critical path +
    // ||r||^2 on the side stream; true = ONE allreduce of {gamma, delta, ||r||^2} per iteration
    // (npc_context_set_fused_allreduce / NPC_PCG_FUSED_ALLREDUCE=1; solvers.cu).
    bool fused_allreduce = false;
    bool timing = false;
    int timing_suppress = 0;         // > 0: inside a scope that times a whole group of launches
    bool capturing = false;          // a PCG iteration is being stream-captured (timing on)
    std::vector<cudaEvent_t> ev_free;
    std::vector<Pending> pending;
    std::vector<Pending> captured;   // events recorded as graph nodes during the capture
    double t_ms[NPC_TIMING_CLASSES] = {0};
    long long t_cnt[NPC_TIMING_CLASSES] = {0};
    int t_begin(int cls, int count = 1);
    void t_end(int idx);
    void t_flush();  // caller has synchronised the stream
    void t_flush_graph(const std::vector<Pending> &ev);  // a timed graph replay has completed
    ~Context();
};

// RAII bracket of a launch (or a multi-kernel step) for the timing classes above.
// A scope nested inside a group scope (timing_suppress > 0) records nothing; a group scope
// (count > 1) brackets several launches with one event pair and credits them all.
// NVTX range (host side, header-only NVTX3: free unless a profiler is attached) for nsys /
// ncu range filtering: npc:degree, npc:operator, npc:update, npc:reduce, npc:vector (every
// TimedScope), npc:halo, npc:allreduce(_rr), npc:pcg, npc:lanczos.
struct NvtxRange {
    explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange &) = delete;
    NvtxRange &operator=(const NvtxRange &) = delete;
};
inline const char *timing_class_name(int cls) {
    static const char *names[] = {"npc:degree", "npc:operator", "npc:update", "npc:reduce", "npc:vector"};
    return cls >= 0 && cls < 5 ? names[cls] : "npc:other";
}
struct TimedScope {
    Context *c;
    int idx;
    NvtxRange nv;
    TimedScope(Context *ctx, int cls, int count = 1)
        : c(ctx), idx(ctx->timing && ctx->timing_suppress == 0 ? ctx->t_begin(cls, count) : -1),
          nv(timing_class_name(cls)) {}
    ~TimedScope() {
        if (idx >= 0) c->t_end(idx);
    }
};
struct TimingGroup {  // suppresses the per-launch scopes inside a group scope
    Context *c;
    explicit TimingGroup(Context *ctx) : c(ctx) { ++c->timing_suppress; }
    ~TimingGroup() { --c->timing_suppress; }
};
enum { T_DEGREE = 0, T_OPERATOR = 1, T_UPDATE = 2, T_REDUCE = 3, T_VECTOR = 4 };

// ------------------------------------------------------------------ launch helpers
// vec_kernels.cu
npc_status launch_reduce_sum(Context *ctx, const double *partials, int n, double *out, int nvec = 1,
                             const double *partials2 = nullptr, int n2 = 0, double *out2 = nullptr);
npc_status launch_scale(Context *ctx, const double *in, double *out, double alpha, int n,
                        const double *dotv, double *partials, int *nparts, const int *done);
npc_status launch_axpby_step(Context *ctx, const double *y, const StepArgs &s, int n);
npc_status launch_dot(Context *ctx, const double *a, const double *b, int n, double *partials, int *nparts);
npc_status launch_gather(Context *ctx, const double *in, const int *idx, double *out, int n);
npc_status launch_scatter(Context *ctx, const double *in, const int *idx, double *out, int n);
npc_status launch_fill(Context *ctx, double *out, double v, int n);
npc_status launch_hash_vector(Context *ctx, double *out, int n, long long offset, unsigned long long seed);
// out[i] = sum_{q=0..P-1} rows[q*m + i] in q order (i < m), on stream s
npc_status launch_sum_rows(Context *ctx, const double *rows, int P, int m, double *out, cudaStream_t s);

// Grid size of the plain vector kernels for n entries (fixed: partial counts are static).
int vec_grid(int n);

// Cluster-resident polynomial for small CSR operators (csr_cluster.cu)
struct SmallCsrDev {
    const int *rowptr;
    const int *cols;
    const double *vals;
    int n, R, nnz_cta;
};
struct SmallCsrPlan {
    int cl_size = 0, R = 0, nnz_cta = 0, threads = 0;
    size_t smem = 0;      // polynomial kernel
    size_t smem_pcg = 0;  // whole-PCG kernel (0: does not fit)
};
struct ClusterPcgOut {
    int iters, converged, breakdown, pad;
    long long applications, reductions;
    double rr, relres_true, bnorm2;
};
npc_status launch_csr_lanczos_cluster(Context *ctx, const SmallCsrDev &A, const SmallCsrPlan &pl, const double *v0,
                                      int m, double *alphas, double *betas, int *steps);
npc_status launch_csr_pcg_cluster(Context *ctx, const SmallCsrDev &A, const SmallCsrPlan &pl, const double *b,
                                  double *x, const double *coef, int k, double tb, int use_poly, double tol2b,
                                  int maxit, ClusterPcgOut *out, double *history);
bool plan_csr_poly_cluster(int n, const int *rowptr, SmallCsrPlan &pl);
npc_status launch_csr_poly_cluster(Context *ctx, const SmallCsrDev &A, int cl_size, int threads, size_t smem,
                                   const double *r, double *z, const double *coef, int k, double tb,
                                   const double *dotv, double *partials, const int *done);

// Low-rank correction and Ritz vectors (lowrank.cu)
#define NPC_LOWRANK_MAX 16

// Operator factories (op_*.cu)
npc_status make_csr_operator(Context *ctx, const npc_operator_desc *d, std::unique_ptr<Operator> &out);
npc_status make_sell_operator(Context *ctx, const npc_operator_desc *d, std::unique_ptr<Operator> &out);
npc_status make_stencil_operator(Context *ctx, const npc_operator_desc *d, std::unique_ptr<Operator> &out);
npc_status make_schur_operator(Context *ctx, const npc_operator_desc *d, std::unique_ptr<Operator> &out);
npc_status make_callback_operator(Context *ctx, const npc_operator_desc *d, std::unique_ptr<Operator> &out);
npc_status make_dfn_operator(Context *ctx, const npc_operator_desc *d, std::unique_ptr<Operator> &out);

// Host halo plan (halo.cu)
struct HaloPlan {
    int n_ghost = 0;
    std::vector<long long> ghost_ids;     // ascending global ids
    std::vector<int> recv_count, recv_off;  // per rank, into the ghost buffer
    std::vector<int> send_count, send_off;  // per rank, into the send buffer
    std::vector<int> send_idx;            // local owned indices to pack (by destination)
    bool empty() const { return n_ghost == 0 && send_idx.empty(); }
};
npc_status halo_plan_local(int n_local, const int *rowptr, const int *colidx, int nranks,
                           const long long *row_starts, int rank, HaloPlan &plan);
npc_status halo_plan_from_ids(std::vector<long long> ids, int nranks, const long long *row_starts, int rank,
                              HaloPlan &plan);
// Exchange ghost-id lists with the owners (NCCL, collective) to fill send lists.
npc_status halo_plan_exchange(Context *ctx, long long row_begin, HaloPlan &plan);
// Per-step exchange: pack x[send_idx] -> send buffer, ncclSend/Recv to the ghost buffer,
// on ctx->comm_stream after an event on ctx->stream; records 'ready' on comm_stream.
struct HaloRuntime {
    DevBuf send_idx, send_buf, ghost_buf;
    cudaEvent_t packed = nullptr, ready = nullptr;
    ~HaloRuntime();
};
npc_status halo_setup(Context *ctx, const HaloPlan &plan, HaloRuntime &rt);
// recv: where the ghosts land (default rt.ghost_buf), e.g. the tail of a local+ghost vector.
npc_status halo_start(Context *ctx, const HaloPlan &plan, HaloRuntime &rt, const double *x,
                      double *recv = nullptr);
npc_status halo_wait(Context *ctx, HaloRuntime &rt);

// Raise a kernel's dynamic shared memory limit to the device maximum once (thread-safe).
// Setting it per launch to the launch's own size races when several host threads launch the
// same kernel with different sizes; the limit does not change occupancy, the launch size does.
npc_status allow_max_dynamic_smem_ptr(const void *kern);  // vec_kernels.cu
template <class K>
npc_status allow_max_dynamic_smem(K kern) {
    return allow_max_dynamic_smem_ptr(reinterpret_cast<const void *>(kern));
}

// Host-side parallel loop over [0, n) in contiguous chunks (operator setup: validation and
// format conversion of 10^7-10^8 entries).  fn(begin, end, thread_index).
template <class F>
void host_parallel_for(long long n, F &&fn, long long grain = 200000) {
    const int hw = (int)std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
    const int nt = n < grain ? 1 : (int)std::min<long long>(hw, n / std::max(grain / 8, 1LL) + 1);
    if (nt == 1) {
        fn(0LL, n, 0);
        return;
    }
    std::vector<std::thread> th;
    for (int t = 0; t < nt; ++t) {
        const long long b = n * t / nt, e = n * (t + 1) / nt;
        th.emplace_back([&fn, b, e, t]() { fn(b, e, t); });
    }
    for (auto &x : th) x.join();
}

// Device-side bit helpers
__host__ __device__ inline int ceil_div(long long a, long long b) { return (int)((a + b - 1) / b); }

// Per-(operator, poly) PCG state kept across solves: work vectors, device scalars and the
// captured CUDA graph of the iteration (valid while none of the pointers it bakes in move).
struct PcgCache {
    DevBuf work, dev;
    size_t work_n = 0;
    long long dev_maxit = -1;
    cudaGraphExec_t exec = nullptr;
    unsigned long long kernels = 0;  // kernels per graph launch
    const void *key_partials = nullptr;
    size_t key_cap = 0;
    bool timed = false;                         // captured with timing event nodes
    bool fused = false;                         // captured with the single fused allreduce
    std::vector<Context::Pending> timing_events;  // owned by the graph (re-recorded per replay)
    void release_events() {
        for (auto &p : timing_events) {
            if (p.e0) cudaEventDestroy(p.e0);
            if (p.e1) cudaEventDestroy(p.e1);
        }
        timing_events.clear();
    }
    void invalidate() {
        if (exec) cudaGraphExecDestroy(exec);
        exec = nullptr;
        release_events();
        timed = false;
    }
    ~PcgCache() { invalidate(); }
};

}  // namespace npc

// Opaque handle structs of the C ABI.
struct npc_context_s {
    npc::Context ctx;
    char err[1024] = "";  // last failing call on this context (npc_last_error(ctx))
};
// Handles record their device so that destroy never dereferences another handle: Python's
// cyclic GC may destroy a context before its operators, or an operator before its polys.
struct npc_operator_s {
    npc_context owner = nullptr;
    int device = 0;
    std::unique_ptr<npc::Operator> op;
    npc::PcgCache pcg;  // plain CG (poly == NULL)
    double estimate_seconds = 0.0;  // wall time of the last npc_estimate_spectrum on it
};
struct npc_poly_s {
    npc_operator op = nullptr;
    int device = 0;
    int kind = 0;              // 0 = Chebyshev (Alg. 2), 1 = Newton (Alg. 1)
    int nlev = 0;              // Newton: number of levels (degree 2^nlev - 1)
    std::vector<double> zeta;  // Newton: zeta_0 .. zeta_nlev
    npc::DevBuf nbuf;          // Newton: 2 work vectors per level >= 2
    int degree = 0;
    double lmin = 0, lmax = 0, xi = 0;
    double theta_bar = 0, delta = 0, sigma = 0;
    double setup_seconds = 0;  // the operator's last spectrum estimate + this set_poly
    std::vector<double> coef;  // 4 * degree: a_j, b_j, c_j, d_j (j = 1..k)
    npc::DevBuf coef_dev;      // the same table on the device (cluster-resident polynomial)
    npc::DevBuf tmp;           // second recurrence buffer (internal order)
    npc::DevBuf tmp2;          // two more buffers when the operator fuses two degrees (step2)
    npc::DevBuf rin, zout;     // internal-order copies when the operator is permuted
    npc::PcgCache pcg;         // PCG work vectors + captured iteration graph
    // low-rank spectral correction P = p_k(A) + V (V^T A V)^{-1} V^T (lowrank.cu)
    int lr_p = 0;
    npc::DevBuf lr_V;          // n_local x lr_p, internal order, column-major
    npc::DevBuf lr_Ginv;       // lr_p x lr_p row-major
    npc::DevBuf lr_scratch;    // multi-dot partials | sums | coefficients
};

namespace npc {
npc_status set_lowrank(npc_poly P, int p, const double *V_ext);
npc_status lowrank_pre(npc_poly P, const double *r, const int *done);
npc_status lowrank_post(npc_poly P, double *z, const double *dotv, double *partials, int *nparts, const int *done);
npc_status ritz_vectors(Operator *op, int m, int p, const double *v0_ext, double *V_ext, double *theta);
}  // namespace npc
