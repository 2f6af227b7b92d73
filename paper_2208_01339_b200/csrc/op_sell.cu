// op_sell.cu -- general sparse operator stored as SELL-C-sigma (C = 32), BASELINE config 4
// (unstructured kNN graph Laplacian), with the Chebyshev recurrence fused in.
//
// Layout: rows are sorted by descending length inside windows of sigma rows (stable), which
// defines a symmetric permutation of the rank's rows; every internal vector lives in that
// order (the caller's vectors are permuted once on entry/exit of apply_poly / pcg_solve,
// never per degree).  Chunks of 32 consecutive internal rows are stored column-major,
// padded to the chunk's longest row (padding: value 0, column = the row itself).  One warp
// per chunk: lane = row, each slot is one fully coalesced 256 B value + 128 B index load.
// Entries keep their original (ascending original-column) order inside a row, so the
// summation order equals the CSR oracle's.
#include <algorithm>
#include <numeric>

#include "device_util.cuh"
#include "npc_internal.cuh"

namespace npc {

npc_status validate_csr_desc(Context *ctx, const npc_operator_desc *d);
npc_status localize_columns(Context *ctx, const npc_operator_desc *d, HaloPlan &plan, std::vector<int> &local_cols);

static constexpr int SELL_C = 32;
static constexpr int SELL_WARPS = 8;

struct SellDev {
    const int *chunk_off;  // slot offset of each chunk (in units of entries)
    const int *chunk_len;  // slots per row of each chunk
    const int *cols;
    const double *vals;
    int n, nchunks;
    const double *ghost;
};

template <bool HAS_S2, bool HAS_R, bool DOT, bool GHOST>
__global__ void __launch_bounds__(SELL_C *SELL_WARPS) k_sell_step(SellDev A, StepArgs s, const int *__restrict__ chunks,
                                                                  int nlist) {
    if (s.done && *s.done) return;
    __shared__ double red[SELL_WARPS];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int li = blockIdx.x * SELL_WARPS + warp;
    double acc = 0.0;
    if (li < nlist) {
        const int ch = chunks ? chunks[li] : li;
        const int row = ch * SELL_C + lane;
        const int len = A.chunk_len[ch];
        const long long base = (long long)A.chunk_off[ch] + lane;
        const double *__restrict__ X = s.x;
        double y = 0.0;
        int j = 0;
        for (; j + 4 <= len; j += 4) {
            int c[4];
            double v[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                c[u] = __ldcs(A.cols + base + (long long)(j + u) * SELL_C);
                v[u] = __ldcs(A.vals + base + (long long)(j + u) * SELL_C);
            }
            double xv[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) xv[u] = (GHOST && c[u] >= A.n) ? A.ghost[c[u] - A.n] : __ldg(X + c[u]);
#pragma unroll
            for (int u = 0; u < 4; ++u) y += v[u] * xv[u];
        }
        for (; j < len; ++j) {
            int c = __ldcs(A.cols + base + (long long)j * SELL_C);
            double v = __ldcs(A.vals + base + (long long)j * SELL_C);
            double xv = (GHOST && c >= A.n) ? A.ghost[c - A.n] : __ldg(X + c);
            y += v * xv;
        }
        if (row < A.n) {
            double o = s.a * y + s.b * X[row];
            if (HAS_S2) o += s.c * s.s2[row];
            if (HAS_R) o += s.d * s.r[row];
            s.out[row] = o;
            if (DOT) acc = o * s.dotv[row];
        }
    }
    if (DOT) {
        acc = block_sum<SELL_C * SELL_WARPS>(acc, red);
        if (threadIdx.x == 0) s.partials[blockIdx.x] = acc;
    }
}

class SellOperator : public Operator {
  public:
    DevBuf chunk_off, chunk_len, cols, vals, perm;
    DevBuf chunks_interior, chunks_boundary;
    int nchunks = 0, n_interior = 0, n_boundary = 0;
    long long nslots = 0, nnz = 0;
    bool multi = false;
    HaloPlan plan;
    HaloRuntime halo;

    bool permuted() const override { return true; }
    npc_status to_internal(const double *in, double *out) override {
        return launch_gather(ctx, in, perm.as<int>(), out, n_local);
    }
    npc_status to_external(const double *in, double *out) override {
        return launch_scatter(ctx, in, perm.as<int>(), out, n_local);
    }
    static int blocks(int nch) { return std::max(1, ceil_div(nch, SELL_WARPS)); }
    int num_partials() const override {
        return multi ? blocks(n_interior) + blocks(n_boundary) : blocks(nchunks);
    }
    double bytes_per_step(bool has_s2, bool has_r) const override {
        // stored slots (values + indices, padding included) + per-chunk metadata + vectors
        double b = (double)nslots * 12.0 + (double)nchunks * 8.0 + 2.0 * 8.0 * n_local;
        if (has_s2) b += 8.0 * n_local;
        if (has_r) b += 8.0 * n_local;
        return b;
    }

    template <bool H2, bool HR, bool DT, bool GH>
    npc_status launch_t(const StepArgs &s, const int *list, int nlist, double *partials) {
        if (nlist <= 0) {
            if (partials && DT) NPC_TRY(launch_fill(ctx, partials, 0.0, 1));
            return NPC_SUCCESS;
        }
        SellDev A{chunk_off.as<int>(), chunk_len.as<int>(), cols.as<int>(), vals.as<double>(), n_local, nchunks,
                  GH ? halo.ghost_buf.as<double>() : nullptr};
        StepArgs a = s;
        a.partials = partials;
        k_sell_step<H2, HR, DT, GH><<<blocks(nlist), SELL_C * SELL_WARPS, 0, ctx->stream>>>(A, a, list, nlist);
        NPC_LAUNCH_CHECK();
        return NPC_SUCCESS;
    }
    template <bool GH>
    npc_status launch_g(const StepArgs &s, const int *list, int nlist, double *p) {
        const bool h2 = s.s2 != nullptr, hr = s.r != nullptr, dt = s.dotv != nullptr;
        if (h2 && hr && dt) return launch_t<true, true, true, GH>(s, list, nlist, p);
        if (h2 && hr) return launch_t<true, true, false, GH>(s, list, nlist, p);
        if (h2 && dt) return launch_t<true, false, true, GH>(s, list, nlist, p);
        if (h2) return launch_t<true, false, false, GH>(s, list, nlist, p);
        if (hr && dt) return launch_t<false, true, true, GH>(s, list, nlist, p);
        if (hr) return launch_t<false, true, false, GH>(s, list, nlist, p);
        if (dt) return launch_t<false, false, true, GH>(s, list, nlist, p);
        return launch_t<false, false, false, GH>(s, list, nlist, p);
    }
    npc_status step(const StepArgs &s) override {
        if (n_local == 0 && !multi) return NPC_SUCCESS;
        if (!multi) return launch_g<false>(s, nullptr, nchunks, s.partials);
        NPC_TRY(halo_start(ctx, plan, halo, s.x));
        NPC_TRY(launch_g<false>(s, chunks_interior.as<int>(), n_interior, s.partials));
        NPC_TRY(halo_wait(ctx, halo));
        return launch_g<true>(s, chunks_boundary.as<int>(), n_boundary,
                              s.partials ? s.partials + blocks(n_interior) : nullptr);
    }
};

npc_status make_sell_operator(Context *ctx, const npc_operator_desc *d, std::unique_ptr<Operator> &out) {
    NPC_TRY(validate_csr_desc(ctx, d));
    if (d->sell_C != 0 && d->sell_C != SELL_C) {
        set_error("SELL: only C = 32 is supported");
        return NPC_ERR_UNSUPPORTED;
    }
    const int sigma = d->sell_sigma == 0 ? 256 : d->sell_sigma;
    if (sigma < 1) {
        set_error("SELL: sigma must be >= 1");
        return NPC_ERR_INVALID_ARGUMENT;
    }
    auto op = std::make_unique<SellOperator>();
    op->ctx = ctx;
    op->kind = NPC_OP_SELL;
    const int n = d->n_local;
    op->n_local = n;
    op->n_global = d->n_global;
    op->row_begin = d->row_begin;
    op->multi = ctx->nranks > 1;
    std::vector<int> lcols;
    NPC_TRY(localize_columns(ctx, d, op->plan, lcols));
    op->nnz = d->rowptr[n];
    // sigma-sort: perm[internal] = local row, inv[local row] = internal
    std::vector<int> perm(n), inv(n);
    std::iota(perm.begin(), perm.end(), 0);
    auto len = [&](int i) { return d->rowptr[i + 1] - d->rowptr[i]; };
    for (int w0 = 0; w0 < n; w0 += sigma) {
        int w1 = std::min(n, w0 + sigma);
        std::stable_sort(perm.begin() + w0, perm.begin() + w1, [&](int a, int b) { return len(a) > len(b); });
    }
    for (int i = 0; i < n; ++i) inv[perm[i]] = i;
    op->nchunks = ceil_div(n, SELL_C);
    std::vector<int> coff(op->nchunks + 1, 0), clen(op->nchunks, 0);
    for (int ch = 0; ch < op->nchunks; ++ch) {
        int m = 0;
        for (int l = 0; l < SELL_C; ++l) {
            int ir = ch * SELL_C + l;
            if (ir < n) m = std::max(m, len(perm[ir]));
        }
        clen[ch] = m;
        long long next = (long long)coff[ch] + (long long)m * SELL_C;
        if (next >= (1LL << 31)) {
            set_error("SELL: more than 2^31 slots");
            return NPC_ERR_UNSUPPORTED;
        }
        coff[ch + 1] = (int)next;
    }
    op->nslots = coff[op->nchunks];
    std::vector<int> scols((size_t)op->nslots);
    std::vector<double> svals((size_t)op->nslots, 0.0);
    std::vector<int> ti, tb;
    for (int ch = 0; ch < op->nchunks; ++ch) {
        bool ghost = false;
        for (int l = 0; l < SELL_C; ++l) {
            int ir = ch * SELL_C + l;
            int orow = ir < n ? perm[ir] : -1;
            int L = orow >= 0 ? len(orow) : 0;
            for (int j = 0; j < clen[ch]; ++j) {
                size_t slot = (size_t)coff[ch] + (size_t)j * SELL_C + l;
                if (j < L) {
                    int p = d->rowptr[orow] + j;
                    int c = lcols[p];
                    if (c >= n) ghost = true;
                    scols[slot] = c < n ? inv[c] : c;
                    svals[slot] = d->vals[p];
                } else {
                    scols[slot] = ir < n ? ir : 0;
                    svals[slot] = 0.0;
                }
            }
        }
        (ghost ? tb : ti).push_back(ch);
    }
    op->n_interior = (int)ti.size();
    op->n_boundary = (int)tb.size();
    NPC_TRY(op->chunk_off.alloc(sizeof(int) * (op->nchunks + 1)));
    NPC_TRY(op->chunk_len.alloc(sizeof(int) * std::max(op->nchunks, 1)));
    NPC_TRY(op->cols.alloc(sizeof(int) * std::max<long long>(op->nslots, 1)));
    NPC_TRY(op->vals.alloc(sizeof(double) * std::max<long long>(op->nslots, 1)));
    NPC_TRY(op->perm.alloc(sizeof(int) * std::max(n, 1)));
    NPC_CUDA_TRY(cudaMemcpy(op->chunk_off.p, coff.data(), sizeof(int) * (op->nchunks + 1), cudaMemcpyHostToDevice));
    if (op->nchunks) NPC_CUDA_TRY(cudaMemcpy(op->chunk_len.p, clen.data(), sizeof(int) * op->nchunks, cudaMemcpyHostToDevice));
    if (op->nslots) {
        NPC_CUDA_TRY(cudaMemcpy(op->cols.p, scols.data(), sizeof(int) * op->nslots, cudaMemcpyHostToDevice));
        NPC_CUDA_TRY(cudaMemcpy(op->vals.p, svals.data(), sizeof(double) * op->nslots, cudaMemcpyHostToDevice));
    }
    if (n) NPC_CUDA_TRY(cudaMemcpy(op->perm.p, perm.data(), sizeof(int) * n, cudaMemcpyHostToDevice));
    if (op->multi) {
        // pack list in internal order
        for (auto &i : op->plan.send_idx) i = inv[i];
        NPC_TRY(op->chunks_interior.alloc(sizeof(int) * std::max<size_t>(ti.size(), 1)));
        NPC_TRY(op->chunks_boundary.alloc(sizeof(int) * std::max<size_t>(tb.size(), 1)));
        if (!ti.empty())
            NPC_CUDA_TRY(cudaMemcpy(op->chunks_interior.p, ti.data(), sizeof(int) * ti.size(), cudaMemcpyHostToDevice));
        if (!tb.empty())
            NPC_CUDA_TRY(cudaMemcpy(op->chunks_boundary.p, tb.data(), sizeof(int) * tb.size(), cudaMemcpyHostToDevice));
        NPC_TRY(halo_setup(ctx, op->plan, op->halo));
    }
    out = std::move(op);
    return NPC_SUCCESS;
}

}  // namespace npc
