// op_sell.cu -- general sparse operator stored as SELL-C-sigma (C = 32), BASELINE config 4
// (unstructured kNN graph Laplacian), with the Chebyshev recurrence fused in.
//
// Layout: rows are sorted by descending length inside windows of sigma rows (stable), which
// defines a symmetric permutation of the rank's rows; every internal vector lives in that
// order (the caller's vectors are permuted once on entry/exit of apply_poly / pcg_solve,
// never per degree).  Chunks of 32 consecutive internal rows are stored column-major,
// padded to the chunk's longest row (padding: value 0, column = the row itself).  Entries
// keep their original (ascending original-column) order inside a row, so the summation
// order equals the CSR oracle's.
//
// Kernel: one CTA (4 warps) per tile of 4 consecutive chunks = 128 rows.  The tile's slots
// are one contiguous, 256 B-aligned segment of the value and index arrays; thread 0 moves
// both with 1D bulk TMA (cp.async.bulk + mbarrier, L2 evict-first) while the warps load
// s_{j-2} and r, then warp w reads slot j of chunk w from shared memory (lane = row,
// conflict-free) and gathers x through L1/L2.  Tiles too large for shared memory fall back
// to direct coalesced loads.  Multi-rank: tiles touching a ghost column run after the halo.
#include <algorithm>
#include <numeric>

#include "device_util.cuh"
#include "npc_internal.cuh"

namespace npc {

npc_status validate_csr_desc(Context *ctx, const npc_operator_desc *d);
npc_status localize_columns(Context *ctx, const npc_operator_desc *d, HaloPlan &plan, std::vector<int> &local_cols);

static constexpr int SELL_C = 32;
static constexpr int SELL_TW = 8;  // chunks (warps) per tile
static constexpr int SELL_MAX_SMEM = 160 * 1024;

struct SellDev {
    const int *chunk_off;  // slot offset of each chunk (entries); chunk_off[nchunks] = total
    const int *chunk_len;  // slots per row of each chunk
    const int *cols;
    const double *vals;
    int n, nchunks;
    const double *ghost;
};

#ifndef NPC_SELL_MINB
#define NPC_SELL_MINB 8  // min resident CTAs per SM for the register allocator (A/B-tuned)
#endif
#ifndef NPC_SELL_U
#define NPC_SELL_U 4  // slots per load group of the direct path (A/B-tuned)
#endif
static constexpr int SELL_U = NPC_SELL_U;

template <bool STAGED, bool HAS_S2, bool HAS_R, bool DOT, bool GHOST>
__global__ void __launch_bounds__(SELL_C *SELL_TW, NPC_SELL_MINB)
    k_sell_step(SellDev A, StepArgs s, const int *__restrict__ tiles, int span_max) {
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ uint64_t bar;
    __shared__ double red[SELL_TW];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int tile = tiles ? tiles[blockIdx.x] : blockIdx.x;
    const int ch0 = tile * SELL_TW;
    const int ch1 = min(ch0 + SELL_TW, A.nchunks);
    const int seg0 = A.chunk_off[ch0];
    double *sv = reinterpret_cast<double *>(smem);
    int *sc = reinterpret_cast<int *>(smem + (size_t)span_max * 8);
    if (STAGED) {
        if (threadIdx.x == 0) {
            mbar_init(&bar, 1);
            fence_mbar_init();
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            const int seg1 = A.chunk_off[ch1];
            const uint32_t nb = (uint32_t)(seg1 - seg0);
            mbar_arrive_expect_tx(&bar, nb * 12u);
            if (nb) {
                const uint64_t pol = policy_evict_first();
                bulk_g2s_evict_first(sv, A.vals + seg0, nb * 8u, &bar, pol);
                bulk_g2s_evict_first(sc, A.cols + seg0, nb * 4u, &bar, pol);
            }
        }
    }
    const int ch = ch0 + warp;
    const int row = ch * SELL_C + lane;
    const bool active = ch < ch1 && row < A.n;
    const double *__restrict__ X = s.x;
    double acc = 0.0;
    if (STAGED) {
        double xs = 0.0, s2v = 0.0, rv = 0.0;
        int len = 0, off = 0;
        if (ch < ch1) {
            len = A.chunk_len[ch];
            off = A.chunk_off[ch] - seg0 + lane;
        }
        if (active) {
            xs = X[row];
            if (HAS_S2) s2v = s.s2[row];
            if (HAS_R) rv = s.r[row];
        }
        const bool is_done = s.done && *s.done;  // read while the bulk copy is in flight
        mbar_wait(&bar, 0);
        if (is_done) return;
        if (ch < ch1) {
            double y = 0.0;
            for (int j = 0; j < len; ++j) {
                const int c = sc[off + j * SELL_C];
                const double v = sv[off + j * SELL_C];
                y += v * ((GHOST && c >= A.n) ? A.ghost[c - A.n] : __ldg(X + c));
            }
            if (active) {
                double o = s.a * y + s.b * xs;
                if (HAS_S2) o += s.c * s2v;
                if (HAS_R) o += s.d * rv;
                s.out[row] = o;
                if (DOT) acc = o * s.dotv[row];
            }
        }
    } else {
        // Direct coalesced slot loads (each slot of a warp is one 256 B value + 128 B index
        // line), SELL_U slots per group.  The kernel is bound by memory latency (the x gathers
        // depend on the index loads), so it is tuned for occupancy: few live registers, the
        // epilogue operands loaded after the loop (A/B: profiles/r01_sell_ab.md).
        const bool is_done = s.done && *s.done;  // the PCG's flag, read beside the chunk metadata
        int len = 0;
        long long gbase = lane;
        if (ch < ch1) {
            len = A.chunk_len[ch];
            gbase += A.chunk_off[ch];
        }
        if (is_done) return;  // uniform over the CTA (before the block reduction)
        const int *__restrict__ cp = A.cols + gbase;
        const double *__restrict__ vp = A.vals + gbase;
        double y = 0.0;
        int j = 0;
        for (; j + SELL_U <= len; j += SELL_U) {
            int c[SELL_U];
            double v[SELL_U];
#pragma unroll
            for (int u = 0; u < SELL_U; ++u) {
                c[u] = __ldcs(cp + (j + u) * SELL_C);
                v[u] = __ldcs(vp + (j + u) * SELL_C);
            }
#pragma unroll
            for (int u = 0; u < SELL_U; ++u)
                y += v[u] * ((GHOST && c[u] >= A.n) ? A.ghost[c[u] - A.n] : __ldg(X + c[u]));
        }
        for (; j < len; ++j) {
            const int c = __ldcs(cp + j * SELL_C);
            const double v = __ldcs(vp + j * SELL_C);
            y += v * ((GHOST && c >= A.n) ? A.ghost[c - A.n] : __ldg(X + c));
        }
        if (active) {
            double o = s.a * y + s.b * X[row];
            if (HAS_S2) o += s.c * s.s2[row];
            if (HAS_R) o += s.d * s.r[row];
            s.out[row] = o;
            if (DOT) acc = o * s.dotv[row];
        }
    }
    if (DOT) {
        acc = block_sum<SELL_C * SELL_TW>(acc, red);
        if (threadIdx.x == 0) s.partials[blockIdx.x] = acc;
    }
}

class SellOperator : public Operator {
  public:
    DevBuf chunk_off, chunk_len, cols, vals, perm;
    DevBuf tiles_interior, tiles_boundary;
    int nchunks = 0, ntiles = 0, n_interior = 0, n_boundary = 0;
    long long nslots = 0, nnz = 0;
    int span_max = 0;
    size_t smem_bytes = 0;
    bool staged = true;
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
    int num_partials() const override {
        return multi && ctx->nranks > 1 ? std::max(n_interior, 1) + std::max(n_boundary, 1) : std::max(ntiles, 1);
    }
    double bytes_per_step(bool has_s2, bool has_r) const override {
        // stored slots (values + indices, padding included) + per-chunk metadata + vectors
        double b = (double)nslots * 12.0 + (double)nchunks * 8.0 + 2.0 * 8.0 * n_local;
        if (has_s2) b += 8.0 * n_local;
        if (has_r) b += 8.0 * n_local;
        return b;
    }

    template <bool ST, bool H2, bool HR, bool DT, bool GH>
    npc_status launch_t(const StepArgs &s, const int *list, int nlist, double *partials) {
        if (nlist <= 0) {
            if (partials && DT) NPC_TRY(launch_fill(ctx, partials, 0.0, 1));
            return NPC_SUCCESS;
        }
        SellDev A{chunk_off.as<int>(), chunk_len.as<int>(), cols.as<int>(), vals.as<double>(), n_local, nchunks,
                  GH ? halo.ghost_buf.as<double>() : nullptr};
        StepArgs a = s;
        a.partials = partials;
        auto kern = k_sell_step<ST, H2, HR, DT, GH>;
        const size_t sm = ST ? smem_bytes : 0;
        if (sm > 48 * 1024) NPC_TRY(allow_max_dynamic_smem(kern));
        kern<<<nlist, SELL_C * SELL_TW, sm, ctx->stream>>>(A, a, list, span_max);
        NPC_LAUNCH_CHECK();
        return NPC_SUCCESS;
    }
    template <bool H2, bool HR, bool DT>
    npc_status launch_s(const StepArgs &s, const int *list, int nlist, double *p, bool ghost) {
        if (staged) {
            if (ghost) return launch_t<true, H2, HR, DT, true>(s, list, nlist, p);
            return launch_t<true, H2, HR, DT, false>(s, list, nlist, p);
        }
        if (ghost) return launch_t<false, H2, HR, DT, true>(s, list, nlist, p);
        return launch_t<false, H2, HR, DT, false>(s, list, nlist, p);
    }
    npc_status launch(const StepArgs &s, const int *list, int nlist, double *p, bool ghost) {
        const bool h2 = s.s2 != nullptr, hr = s.r != nullptr, dt = s.dotv != nullptr;
        if (h2 && hr && dt) return launch_s<true, true, true>(s, list, nlist, p, ghost);
        if (h2 && hr) return launch_s<true, true, false>(s, list, nlist, p, ghost);
        if (h2 && dt) return launch_s<true, false, true>(s, list, nlist, p, ghost);
        if (h2) return launch_s<true, false, false>(s, list, nlist, p, ghost);
        if (hr && dt) return launch_s<false, true, true>(s, list, nlist, p, ghost);
        if (hr) return launch_s<false, true, false>(s, list, nlist, p, ghost);
        if (dt) return launch_s<false, false, true>(s, list, nlist, p, ghost);
        return launch_s<false, false, false>(s, list, nlist, p, ghost);
    }
    npc_status step(const StepArgs &s) override {
        if (n_local == 0 && !multi) return NPC_SUCCESS;
        // single rank, or a 1-rank distributed context (no halo; with more ranks the exchange
        // is collective for the local transport even when this rank's plan is empty)
        if (!multi || ctx->nranks == 1) return launch(s, nullptr, ntiles, s.partials, false);
        NPC_TRY(halo_start(ctx, plan, halo, s.x));
        NPC_TRY(launch(s, tiles_interior.as<int>(), n_interior, s.partials, false));
        NPC_TRY(halo_wait(ctx, halo));
        return launch(s, tiles_boundary.as<int>(), n_boundary, s.partials ? s.partials + std::max(n_interior, 1) : nullptr,
                      true);
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
    op->multi = ctx->distributed();
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
    std::vector<char> chunk_ghost(op->nchunks, 0);
    host_parallel_for(op->nchunks, [&](long long cb, long long ce, int) {
    for (int ch = (int)cb; ch < (int)ce; ++ch) {
        for (int l = 0; l < SELL_C; ++l) {
            int ir = ch * SELL_C + l;
            int orow = ir < n ? perm[ir] : -1;
            int L = orow >= 0 ? len(orow) : 0;
            for (int j = 0; j < clen[ch]; ++j) {
                size_t slot = (size_t)coff[ch] + (size_t)j * SELL_C + l;
                if (j < L) {
                    int p = d->rowptr[orow] + j;
                    int c = lcols[p];
                    if (c >= n) chunk_ghost[ch] = 1;
                    scols[slot] = c < n ? inv[c] : c;
                    svals[slot] = d->vals[p];
                } else {
                    scols[slot] = ir < n ? ir : 0;
                    svals[slot] = 0.0;
                }
            }
        }
    }
    });
    // tiles of SELL_TW chunks: largest contiguous slot segment -> shared memory size
    op->ntiles = ceil_div(op->nchunks, SELL_TW);
    std::vector<int> ti, tb;
    for (int t = 0; t < op->ntiles; ++t) {
        const int c0 = t * SELL_TW, c1 = std::min(op->nchunks, c0 + SELL_TW);
        op->span_max = std::max(op->span_max, coff[c1] - coff[c0]);
        bool ghost = false;
        for (int c = c0; c < c1; ++c) ghost = ghost || chunk_ghost[c];
        (ghost ? tb : ti).push_back(t);
    }
    op->smem_bytes = (size_t)op->span_max * 12 + 16;
    // Direct coalesced loads by default: SELL slots are already full 128 B lines per warp, and
    // staging limits occupancy (the x gather needs many warps in flight).  NPC_SELL_STAGED=1
    // selects the bulk-TMA staged variant (measured slower on config 4: profiles/).
    op->staged = getenv("NPC_SELL_STAGED") && op->smem_bytes <= (size_t)SELL_MAX_SMEM;
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
        NPC_TRY(op->tiles_interior.alloc(sizeof(int) * std::max<size_t>(ti.size(), 1)));
        NPC_TRY(op->tiles_boundary.alloc(sizeof(int) * std::max<size_t>(tb.size(), 1)));
        if (!ti.empty())
            NPC_CUDA_TRY(cudaMemcpy(op->tiles_interior.p, ti.data(), sizeof(int) * ti.size(), cudaMemcpyHostToDevice));
        if (!tb.empty())
            NPC_CUDA_TRY(cudaMemcpy(op->tiles_boundary.p, tb.data(), sizeof(int) * tb.size(), cudaMemcpyHostToDevice));
        NPC_TRY(halo_setup(ctx, op->plan, op->halo));
    }
    out = std::move(op);
    return NPC_SUCCESS;
}

}  // namespace npc
