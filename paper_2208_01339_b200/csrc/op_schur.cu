// op_schur.cu -- matrix-free Schur-complement operator S = C + B^T D^{-1} B (BASELINE
// config 5), never assembled, with the Chebyshev recurrence fused into the second pass.
//
// This is the "global sparse product - local inverse - transposed product" shape of the
// paper's S_u application (Alg. 3), with D standing in for
// the block-diagonal A^{-1} and C = tridiag(-1, 2 + c, -1) for G^u.
//   create: Bt = D^{-1/2} B, so S = C + Bt^T Bt and D is never read per application.  The
//           rows of Bt are reordered by length (4, 3, 2, 1 entries; the order of B's rows is
//           free since t = Bt v is internal) and stored SELL-32 column-major (no padding but
//           the tail chunk of each length class).
// Atomic form (NPC_SCHUR_ATOMIC=1; always across ranks), two kernels per application:
//   k_schur_bpass_atomic:    t_q = (Bt v)_q in registers; y[col] += Bt_qj t_q (fp64 RED into
//                            y, L2-resident: the random traffic -- v gather, y scatter --
//                            stays in a 2 x 8n-byte L2 working set)
//   k_schur_tstep:           (S v)_i = (2 + c_i) v_i - v_{i-1} - v_{i+1} + y_i ; y_i = 0 ;
//                            out = a (S v) + b v + c s2 + d r   (+ dot partial)
// Deterministic form (default on one rank): Bt^T is also stored, as CSR over the trace rows
// (column ids = positions of t, ascending), split into K position ranges, and
//   pass 1 (k_schur_bpass):  t = Bt v written out (12 B x rows of B);
//   pass 2 (k_schur_tpass):  (Bt^T t)_i gathered per trace row, tile-staged by bulk TMA, one
//                            launch per t range carrying the row sums, the last fused with C
//                            and the epilogue.  Same bits every run; each launch gathers from a
//                            t range small enough to stay L2-resident (unsplit, the 96 MB t
//                            spills beside the 432 MB Bt^T stream and the pass is 2x slower).
#include <algorithm>
#include <numeric>

#include "device_util.cuh"
#include "npc_internal.cuh"

namespace npc {

static constexpr int SB_WARPS = 8;
static constexpr int ST_TILE = 256;
static constexpr int ST_MAX_SMEM = 200 * 1024;

__global__ void __launch_bounds__(32 * SB_WARPS) k_schur_bpass(const int *__restrict__ chunk_off,
                                                               const int *__restrict__ chunk_len, int nchunks,
                                                               const int *__restrict__ cols,
                                                               const double *__restrict__ vals,
                                                               const double *__restrict__ v, double *__restrict__ t,
                                                               const int *done) {
    if (done && *done) return;
    const int lane = threadIdx.x & 31;
    const int ch = blockIdx.x * SB_WARPS + (threadIdx.x >> 5);
    if (ch >= nchunks) return;
    const int len = chunk_len[ch];
    const long long base = (long long)chunk_off[ch] + lane;
    int c[4];
    double b[4];
#pragma unroll
    for (int j = 0; j < 4; ++j)
        if (j < len) {
            c[j] = __ldcs(cols + base + 32LL * j);
            b[j] = __ldcs(vals + base + 32LL * j);
        }
    double acc = 0.0;
#pragma unroll
    for (int j = 0; j < 4; ++j)
        if (j < len) acc += b[j] * __ldg(v + c[j]);
    t[ch * 32 + lane] = acc;
}

// Atomic form (default): t_q stays in a register and is scattered straight into y with fp64
// reductions (RED.ADD.F64); y (8 n bytes) stays L2-resident, so the only random traffic is
// the v gather and the y scatter, both inside L2.
__global__ void __launch_bounds__(32 * SB_WARPS) k_schur_bpass_atomic(const int *__restrict__ chunk_off,
                                                                      const int *__restrict__ chunk_len, int nchunks,
                                                                      const int *__restrict__ cols,
                                                                      const double *__restrict__ vals,
                                                                      const double *__restrict__ v, double *y,
                                                                      const int *done) {
    if (done && *done) return;
    const int lane = threadIdx.x & 31;
    const int ch = blockIdx.x * SB_WARPS + (threadIdx.x >> 5);
    if (ch >= nchunks) return;
    const int len = chunk_len[ch];
    const long long base = (long long)chunk_off[ch] + lane;
    int c[4];
    double b[4];
#pragma unroll
    for (int j = 0; j < 4; ++j)
        if (j < len) {
            c[j] = __ldcs(cols + base + 32LL * j);
            b[j] = __ldcs(vals + base + 32LL * j);
        }
    double acc = 0.0;
#pragma unroll
    for (int j = 0; j < 4; ++j)
        if (j < len) acc += b[j] * __ldg(v + c[j]);
    // First entries: the chunk's rows are sorted by their first column, so lanes with equal
    // c[0] are contiguous.  Sum their contributions with a segmented warp scan and issue one
    // RED per distinct column (the L2 RED rate bounds this kernel: profiles/).
    const unsigned full = 0xffffffffu;
    // (padding lanes of a class tail carry column 0 and value 0: they add 0 to any segment)
    const bool has0 = len > 0;
    const int c0 = has0 ? c[0] : -1;
    double part = has0 ? b[0] * acc : 0.0;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const double o = __shfl_up_sync(full, part, d);
        const int oc = __shfl_up_sync(full, c0, d);
        // lanes lane-d .. lane all share c0 iff the lane d below does (contiguous segments)
        if (lane >= d && oc == c0) part += o;
    }
    const int next_c0 = __shfl_down_sync(full, c0, 1);
    if (has0 && (lane == 31 || next_c0 != c0) && part != 0.0) atomicAdd(y + c0, part);
    if (acc != 0.0) {
#pragma unroll
        for (int j = 1; j < 4; ++j)
            if (j < len) atomicAdd(y + c[j], b[j] * acc);
    }
}

template <bool HAS_S2, bool HAS_R, bool DOT>
__global__ void __launch_bounds__(ST_TILE) k_schur_tstep(const double *__restrict__ cshift, double *y, int n,
                                                         StepArgs s, const double *xl, const double *xr) {
    if (s.done && *s.done) return;
    __shared__ double red[ST_TILE / 32];
    double acc = 0.0;
    const double *__restrict__ X = s.x;
    // one element per thread (grid = ceil(n / 256)): all loads of a thread are independent,
    // so the whole grid's memory-level parallelism hides the HBM latency
    const int i = blockIdx.x * ST_TILE + threadIdx.x;
    if (i < n) {
        const double xi = X[i];
        double sv = (2.0 + cshift[i]) * xi;
        if (i > 0) sv -= X[i - 1];
        else if (xl) sv -= *xl;  // multi-rank: last row of the previous rank
        if (i < n - 1) sv -= X[i + 1];
        else if (xr) sv -= *xr;  // first row of the next rank
        sv += y[i];
        y[i] = 0.0;
        double o = s.a * sv + s.b * xi;
        if (HAS_S2) o += s.c * s.s2[i];
        if (HAS_R) o += s.d * s.r[i];
        s.out[i] = o;
        if (DOT) acc += o * s.dotv[i];
    }
    if (DOT) {
        acc = block_sum<ST_TILE>(acc, red);
        if (threadIdx.x == 0) s.partials[blockIdx.x] = acc;
    }
}

struct SchurTDev {
    const int *rowptr;
    const int *cols;  // positions in t
    const double *vals;
    const double *cshift;
    const double *t;
    int n;
};

// PARTIAL: the t-position range of this pass is one of several (see SchurOperator::parts):
// yout = yin + the partial row sums, no epilogue.  The last pass adds yin and finishes.  The
// per-row summation sequence is the same as one unsplit pass (bitwise).
template <bool STAGED, bool HAS_S2, bool HAS_R, bool DOT, bool PARTIAL>
__global__ void __launch_bounds__(ST_TILE) k_schur_tpass(SchurTDev T, StepArgs s, int vspan_max,
                                                         const double *__restrict__ yin, double *__restrict__ yout) {
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ uint64_t bar;
    __shared__ double red[ST_TILE / 32];
    const int row0 = blockIdx.x * ST_TILE;
    const int nrows = min(ST_TILE, T.n - row0);
    const int pb = T.rowptr[row0];
    const int v0 = pb & ~1, c0 = pb & ~3;
    double *sv = reinterpret_cast<double *>(smem);
    int *sc = reinterpret_cast<int *>(smem + (size_t)vspan_max * 8);
    if (STAGED) {
        if (threadIdx.x == 0) {
            mbar_init(&bar, 1);
            fence_mbar_init();
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            const int pe = T.rowptr[row0 + nrows];
            const int v1 = (pe + 1) & ~1, c1 = (pe + 3) & ~3;
            const uint32_t bv = (uint32_t)(v1 - v0) * 8u, bc = (uint32_t)(c1 - c0) * 4u;
            // an empty tile (pe == pb) may still have bv or bc != 0 from the alignment
            // rounding: expect exactly the bytes issued, none for an empty tile
            const bool any = pe > pb;
            mbar_arrive_expect_tx(&bar, any ? bv + bc : 0u);
            if (any) {
                const uint64_t pol = policy_evict_first();
                bulk_g2s_evict_first(sv, T.vals + v0, bv, &bar, pol);
                bulk_g2s_evict_first(sc, T.cols + c0, bc, &bar, pol);
            }
        }
    }
    const int i = row0 + threadIdx.x;
    const bool active = threadIdx.x < nrows;
    const double *__restrict__ X = s.x;
    int rb = 0, re = 0;
    double xi = 0.0, cv = 0.0, xl = 0.0, xr = 0.0, s2v = 0.0, rv = 0.0;
    if (active) {
        rb = T.rowptr[i];
        re = T.rowptr[i + 1];
        xi = X[i];
        cv = T.cshift[i];
        if (i > 0) xl = X[i - 1];
        if (i < T.n - 1) xr = X[i + 1];
        if (HAS_S2) s2v = s.s2[i];
        if (HAS_R) rv = s.r[i];
    }
    const bool is_done = s.done && *s.done;  // the PCG's flag, read while the bulk copy is in flight
    if (STAGED) mbar_wait(&bar, 0);
    if (is_done) return;
    double acc = 0.0;
    if (active) {
        double y = yin ? yin[i] : 0.0;
        for (int p = rb; p < re; ++p) {
            int c;
            double v;
            if (STAGED) {
                c = sc[p - c0];
                v = sv[p - v0];
            } else {
                c = __ldcs(T.cols + p);
                v = __ldcs(T.vals + p);
            }
            y += v * __ldg(T.t + c);
        }
        if (PARTIAL) {
            yout[i] = y;
            return;  // no block reduction in partial passes
        }
        const double svv = ((2.0 + cv) * xi - xl - xr) + y;
        double o = s.a * svv + s.b * xi;
        if (HAS_S2) o += s.c * s2v;
        if (HAS_R) o += s.d * rv;
        s.out[i] = o;
        if (DOT) acc = o * s.dotv[i];
    }
    if (DOT) {
        acc = block_sum<ST_TILE>(acc, red);
        if (threadIdx.x == 0) s.partials[blockIdx.x] = acc;
    }
}

class SchurOperator : public Operator {
  public:
    DevBuf cshift, chunk_off, chunk_len, bcols, bvals, t;
    DevBuf trowptr, tcols, tvals;
    // Deterministic form, t split into K position ranges (NPC_SCHUR_SPLIT, default 3) so the
    // t range each pass gathers (96 MB / K) stays L2-resident beside its entry stream; pass k
    // carries the row sums of passes < k in yacc.
    struct Part {
        DevBuf rowptr, cols, vals;
        int vspan = 0, cspan = 0;
        size_t smem = 0;
        bool staged = true;
    };
    std::vector<std::unique_ptr<Part>> parts;
    DevBuf yacc;
    int nbp = 0, nchunks = 0, ntiles = 0;
    long long nnz = 0, nslots = 0;
    int vspan_max = 0, cspan_max = 0;
    size_t smem_bytes = 0;
    bool staged = true;
    bool deterministic = false;  // split two-pass form (default on one rank; NPC_SCHUR_ATOMIC=1 off)
    int grid2 = 1;               // atomic form: grid of k_schur_tstep
    // multi-rank (nranks > 1, atomic form): P slots of m entries; B column ids are remapped to
    // slot positions.  Per application: own x -> my slot of xfull, allgather the slots, B pass
    // of the rank's B rows into yfull, reduce-scatter yfull -> yown, reset yfull, C + epilogue.
    bool multi = false;
    int m = 0, xl_pos = -1, xr_pos = -1;
    std::vector<int> counts;
    DevBuf xfull, yfull, yown;

    int num_partials() const override { return deterministic ? std::max(ntiles, 1) : grid2; }
    double bytes_per_step(bool has_s2, bool has_r) const override {
        if (!deterministic) {
            // Bt slots once, c once, x read + out written, y scattered (L2) then read and reset
            double b = (double)nslots * 12.0 + 8.0 * n_local + 2.0 * 8.0 * n_local + 2.0 * 8.0 * n_local;
            if (has_s2) b += 8.0 * n_local;
            if (has_r) b += 8.0 * n_local;
            return b;
        }
        // pass 1: Bt slots (12 B) + t written; pass 2: Bt^T (12 B/nnz + rowptr) + t read once +
        // c + x + out (+ s_{j-2}, r).  v is gathered from L2 in pass 1 (read once in pass 2).
        const double K = (double)std::max<size_t>(parts.size(), 1);
        double b = (double)nslots * 12.0 + 8.0 * nbp + (double)nnz * 12.0 + 4.0 * K * (n_local + 1) + 8.0 * nbp +
                   3.0 * 8.0 * n_local + (K - 1.0) * 2.0 * 8.0 * n_local;
        if (has_s2) b += 8.0 * n_local;
        if (has_r) b += 8.0 * n_local;
        return b;
    }
    template <bool ST, bool H2, bool HR, bool DT, bool PA>
    npc_status launch_part(const StepArgs &s, const Part &pt, const double *yin, double *yout) {
        SchurTDev T{pt.rowptr.as<int>(), pt.cols.as<int>(), pt.vals.as<double>(), cshift.as<double>(),
                    t.as<double>(), n_local};
        auto kern = k_schur_tpass<ST, H2, HR, DT, PA>;
        const size_t sm = ST ? pt.smem : 0;
        if (sm > 48 * 1024) NPC_TRY(allow_max_dynamic_smem(kern));
        kern<<<ntiles, ST_TILE, sm, ctx->stream>>>(T, s, pt.vspan, yin, yout);
        NPC_LAUNCH_CHECK();
        return NPC_SUCCESS;
    }
    template <bool H2, bool HR, bool DT>
    npc_status launch2s(const StepArgs &s) {
        const int K = (int)parts.size();
        double *ya = yacc.as<double>();
        for (int k = 0; k + 1 < K; ++k) {
            const Part &pt = *parts[k];
            const double *yin = k ? ya : nullptr;
            if (pt.staged)
                NPC_TRY((launch_part<true, false, false, false, true>(s, pt, yin, ya)));
            else
                NPC_TRY((launch_part<false, false, false, false, true>(s, pt, yin, ya)));
        }
        const Part &pl = *parts[K - 1];
        const double *yin = K > 1 ? ya : nullptr;
        return pl.staged ? launch_part<true, H2, HR, DT, false>(s, pl, yin, nullptr)
                         : launch_part<false, H2, HR, DT, false>(s, pl, yin, nullptr);
    }
    template <bool H2, bool HR, bool DT>
    npc_status launch_t(const StepArgs &s) {
        const double *xl = multi && xl_pos >= 0 ? xfull.as<double>() + xl_pos : nullptr;
        const double *xr = multi && xr_pos >= 0 ? xfull.as<double>() + xr_pos : nullptr;
        double *y = multi ? yown.as<double>() : t.as<double>();
        k_schur_tstep<H2, HR, DT><<<grid2, ST_TILE, 0, ctx->stream>>>(cshift.as<double>(), y, n_local, s, xl, xr);
        NPC_LAUNCH_CHECK();
        return NPC_SUCCESS;
    }
    npc_status step_atomic(const StepArgs &s) {
        const double *v = s.x;
        double *y = t.as<double>();
        if (multi) {
            double *xf = xfull.as<double>();
            if (n_local)
                NPC_CUDA_TRY(cudaMemcpyAsync(xf + (size_t)ctx->rank * m, s.x, sizeof(double) * n_local,
                                             cudaMemcpyDeviceToDevice, ctx->stream));
            NPC_TRY(ctx->tr->allgather_slots(ctx, xf, m, counts, ctx->stream));
            v = xf;
            y = yfull.as<double>();
        }
        if (nchunks) {
            k_schur_bpass_atomic<<<ceil_div(nchunks, SB_WARPS), 32 * SB_WARPS, 0, ctx->stream>>>(
                chunk_off.as<int>(), chunk_len.as<int>(), nchunks, bcols.as<int>(), bvals.as<double>(), v, y,
                s.done);
            NPC_LAUNCH_CHECK();
        }
        if (multi) {
            NPC_TRY(ctx->tr->reduce_scatter_slots(ctx, yfull.as<double>(), yown.as<double>(), m, ctx->stream));
            NPC_CUDA_TRY(cudaMemsetAsync(yfull.p, 0, yfull.bytes, ctx->stream));
        }
        const bool h2 = s.s2 != nullptr, hr = s.r != nullptr, dt = s.dotv != nullptr;
        if (h2 && hr && dt) return launch_t<true, true, true>(s);
        if (h2 && hr) return launch_t<true, true, false>(s);
        if (h2 && dt) return launch_t<true, false, true>(s);
        if (h2) return launch_t<true, false, false>(s);
        if (hr && dt) return launch_t<false, true, true>(s);
        if (hr) return launch_t<false, true, false>(s);
        if (dt) return launch_t<false, false, true>(s);
        return launch_t<false, false, false>(s);
    }
    npc_status step(const StepArgs &s) override {
        if (n_local == 0 && !multi) return NPC_SUCCESS;
        if (!deterministic) return step_atomic(s);
        if (nchunks) {
            k_schur_bpass<<<ceil_div(nchunks, SB_WARPS), 32 * SB_WARPS, 0, ctx->stream>>>(
                chunk_off.as<int>(), chunk_len.as<int>(), nchunks, bcols.as<int>(), bvals.as<double>(), s.x,
                t.as<double>(), s.done);
            NPC_LAUNCH_CHECK();
        }
        const bool h2 = s.s2 != nullptr, hr = s.r != nullptr, dt = s.dotv != nullptr;
        if (h2 && hr && dt) return launch2s<true, true, true>(s);
        if (h2 && hr) return launch2s<true, true, false>(s);
        if (h2 && dt) return launch2s<true, false, true>(s);
        if (h2) return launch2s<true, false, false>(s);
        if (hr && dt) return launch2s<false, true, true>(s);
        if (hr) return launch2s<false, true, false>(s);
        if (dt) return launch2s<false, false, true>(s);
        return launch2s<false, false, false>(s);
    }
};

npc_status make_schur_operator(Context *ctx, const npc_operator_desc *d, std::unique_ptr<Operator> &out) {
    const int n = d->n_local, nb = d->b_n_local;
    const bool multi = ctx->distributed();
    if (n < 0 || nb < 0 || (n > 0 && !d->c) || (nb > 0 && (!d->b_rowptr || !d->b_colidx || !d->b_vals || !d->d))) {
        set_error("SCHUR: invalid arrays");
        return NPC_ERR_INVALID_ARGUMENT;
    }

    // trace-row partition: every rank's (row_begin, n_local) -> slot layout
    std::vector<long long> starts{0}, all_n;
    long long n_global = n;
    if (multi) {
        NPC_TRY(ctx->tr->allgather_i64(ctx, n, all_n));
        for (long long c : all_n) starts.push_back(starts.back() + c);
        n_global = starts.back();
        if (d->row_begin != starts[ctx->rank] || (d->n_global && d->n_global != n_global)) {
            set_error("SCHUR: rank %d row_begin %lld / n_global %lld disagree with the partition", ctx->rank,
                      d->row_begin, d->n_global);
            return NPC_ERR_DIMENSION;
        }
        long long nbg = 0;
        std::vector<long long> all_nb;
        NPC_TRY(ctx->tr->allgather_i64(ctx, nb, all_nb));
        for (long long c : all_nb) nbg += c;
        if (d->b_rows_global && d->b_rows_global != nbg) {
            set_error("SCHUR: b_rows_global disagrees with the sum of b_n_local");
            return NPC_ERR_DIMENSION;
        }
    } else if ((d->n_global && d->n_global != n) || (d->b_rows_global && d->b_rows_global != nb)) {
        set_error("SCHUR: sizes disagree");
        return NPC_ERR_DIMENSION;
    }
    if (nb > 0 && d->b_rowptr[0] != 0) {
        set_error("SCHUR: b_rowptr[0] != 0");
        return NPC_ERR_DIMENSION;
    }
    for (int i = 0; i < n; ++i)
        if (!std::isfinite(d->c[i])) {
            set_error("SCHUR: non-finite c");
            return NPC_ERR_DIMENSION;
        }
    // validation in parallel row chunks (first offending row reported)
    {
        std::vector<long long> bad(64, -1);
        std::vector<int> why(64, 0);
        host_parallel_for(nb, [&](long long b, long long e, int t) {
            for (long long q = b; q < e; ++q) {
                const int L = d->b_rowptr[q + 1] - d->b_rowptr[q];
                int w = 0;
                if (L < 0) w = 1;
                else if (L > 4) w = 2;
                else if (!(d->d[q] > 0.0) || !std::isfinite(d->d[q])) w = 3;
                else
                    for (int p = d->b_rowptr[q]; p < d->b_rowptr[q + 1] && !w; ++p)
                        if (d->b_colidx[p] < 0 || d->b_colidx[p] >= n_global || !std::isfinite(d->b_vals[p])) w = 4;
                if (w) {
                    bad[t] = q;
                    why[t] = w;
                    return;
                }
            }
        });
        for (int t = 0; t < 64; ++t)
            if (bad[t] >= 0) {
                const long long q = bad[t];
                if (why[t] <= 2) {
                    set_error("SCHUR: B rows must have 0..4 entries (row %lld has %d)", q,
                              d->b_rowptr[q + 1] - d->b_rowptr[q]);
                    return why[t] == 1 ? NPC_ERR_DIMENSION : NPC_ERR_UNSUPPORTED;
                }
                set_error(why[t] == 3 ? "SCHUR: D must be positive and finite (row %lld)"
                                      : "SCHUR: bad B entry in row %lld", q);
                return NPC_ERR_DIMENSION;
            }
    }
    // Rows grouped by length; within a length class ordered by their first (smallest) column
    // (stable counting sort): the first-column gathers of v and scatters into y of a warp then
    // fall on a few adjacent sectors, cutting the random L2 sector count for one entry per row.
    std::vector<int> byl[5];
    {
        std::vector<int> key(std::max(nb, 1));
        std::vector<long long> cnt((size_t)5 * ((size_t)n_global + 1) + 1, 0);
        auto slot = [&](int L, long long c) { return (size_t)L * ((size_t)n_global + 1) + (size_t)c; };
        for (int q = 0; q < nb; ++q) {
            const int L = d->b_rowptr[q + 1] - d->b_rowptr[q];
            const long long c = L ? d->b_colidx[d->b_rowptr[q]] : 0;
            key[q] = L;
            cnt[slot(L, c) + 1]++;
        }
        for (size_t i = 1; i < cnt.size(); ++i) cnt[i] += cnt[i - 1];
        std::vector<int> sorted(std::max(nb, 1));
        for (int q = 0; q < nb; ++q) {
            const int L = key[q];
            const long long c = L ? d->b_colidx[d->b_rowptr[q]] : 0;
            sorted[cnt[slot(L, c)]++] = q;
        }
        // sorted is ordered by (L, first column, q); split into the length classes
        long long at = 0;
        for (int L = 0; L <= 4; ++L) {
            long long len = 0;
            for (int q = 0; q < nb; ++q) len += key[q] == L;  // class sizes
            byl[L].assign(sorted.begin() + at, sorted.begin() + at + len);
            at += len;
        }
    }
    auto op = std::make_unique<SchurOperator>();
    op->ctx = ctx;
    op->kind = NPC_OP_SCHUR;
    op->n_local = n;
    op->n_global = n_global;
    op->row_begin = d->row_begin;
    op->nnz = nb ? d->b_rowptr[nb] : 0;
    // global column id -> position in the slot layout (identity on one rank)
    int m = n;
    if (multi) {
        m = 1;
        for (long long c : all_n) m = std::max<long long>(m, c);
    }
    auto colpos = [&](int c) -> int {
        if (!multi) return c;
        const int q = (int)(std::upper_bound(starts.begin(), starts.end(), (long long)c) - starts.begin()) - 1;
        return q * m + (int)(c - starts[q]);
    };
    // ---- Bt = D^{-1/2} B, rows ordered by length, SELL-32
    std::vector<int> order;
    std::vector<int> coff{0}, clen;
    for (int L = 4; L >= 1; --L) {
        for (size_t k = 0; k < byl[L].size(); k += 32) {
            clen.push_back(L);
            coff.push_back(coff.back() + 32 * L);
        }
        order.insert(order.end(), byl[L].begin(), byl[L].end());
        while (order.size() % 32) order.push_back(-1);  // pad the class tail
    }
    op->nchunks = (int)clen.size();
    op->nbp = (int)order.size();
    op->nslots = coff.back();
    std::vector<int> scols((size_t)op->nslots, 0);
    std::vector<double> svals((size_t)op->nslots, 0.0);
    std::vector<int> tcount(n + 1, 0);
    host_parallel_for(op->nchunks, [&](long long cb, long long ce, int) {
        for (long long ch = cb; ch < ce; ++ch)
            for (int l = 0; l < 32; ++l) {
                const int q = order[(size_t)ch * 32 + l];
                if (q < 0) continue;
                const double sc = 1.0 / std::sqrt(d->d[q]);
                for (int j = 0; j < clen[ch]; ++j) {
                    const size_t slot = (size_t)coff[ch] + (size_t)j * 32 + l;
                    const int p = d->b_rowptr[q] + j;
                    scols[slot] = colpos(d->b_colidx[p]);
                    svals[slot] = d->b_vals[p] * sc;
                }
            }
    });
    if (!multi)
        for (long long p = 0; p < op->nnz; ++p) tcount[d->b_colidx[p] + 1]++;
    // Single rank: the deterministic split two-pass form (faster, and bitwise reproducible;
    // profiles/r01_schur_scatter_microbench.md).  NPC_SCHUR_ATOMIC=1 selects the fp64-RED form,
    // which is also the form used across ranks (its partial B^T t is reduce-scattered).
    op->deterministic = !multi && getenv("NPC_SCHUR_ATOMIC") == nullptr;
    op->grid2 = std::max(1, ceil_div(n, ST_TILE));
    if (!op->deterministic) {
        NPC_TRY(op->cshift.alloc(sizeof(double) * std::max(n, 1)));
        NPC_TRY(op->t.alloc(sizeof(double) * std::max(n, 1)));  // y accumulator
        NPC_TRY(op->chunk_off.alloc(sizeof(int) * (op->nchunks + 1)));
        NPC_TRY(op->chunk_len.alloc(sizeof(int) * std::max(op->nchunks, 1)));
        NPC_TRY(op->bcols.alloc(sizeof(int) * std::max<long long>(op->nslots, 1)));
        NPC_TRY(op->bvals.alloc(sizeof(double) * std::max<long long>(op->nslots, 1)));
        if (n) NPC_CUDA_TRY(cudaMemcpy(op->cshift.p, d->c, sizeof(double) * n, cudaMemcpyHostToDevice));
        NPC_CUDA_TRY(cudaMemset(op->t.p, 0, op->t.bytes));
        NPC_CUDA_TRY(cudaMemcpy(op->chunk_off.p, coff.data(), sizeof(int) * coff.size(), cudaMemcpyHostToDevice));
        if (op->nchunks) {
            NPC_CUDA_TRY(cudaMemcpy(op->chunk_len.p, clen.data(), sizeof(int) * clen.size(), cudaMemcpyHostToDevice));
            NPC_CUDA_TRY(cudaMemcpy(op->bcols.p, scols.data(), sizeof(int) * scols.size(), cudaMemcpyHostToDevice));
            NPC_CUDA_TRY(cudaMemcpy(op->bvals.p, svals.data(), sizeof(double) * svals.size(), cudaMemcpyHostToDevice));
        }
        if (multi) {
            const int P = ctx->nranks, r = ctx->rank;
            op->multi = true;
            op->m = m;
            op->counts.assign(all_n.begin(), all_n.end());
            // neighbours of the rank's end rows in the tridiagonal block: last row of the
            // nearest non-empty rank below, first row of the nearest non-empty rank above
            for (int q = r - 1; q >= 0 && n > 0; --q)
                if (all_n[q] > 0) {
                    op->xl_pos = q * m + (int)all_n[q] - 1;
                    break;
                }
            for (int q = r + 1; q < P && n > 0; ++q)
                if (all_n[q] > 0) {
                    op->xr_pos = q * m;
                    break;
                }
            NPC_TRY(op->xfull.alloc(sizeof(double) * (size_t)P * m));
            NPC_TRY(op->yfull.alloc(sizeof(double) * (size_t)P * m));
            NPC_TRY(op->yown.alloc(sizeof(double) * (size_t)m));
            NPC_CUDA_TRY(cudaMemset(op->xfull.p, 0, op->xfull.bytes));
            NPC_CUDA_TRY(cudaMemset(op->yfull.p, 0, op->yfull.bytes));
        }
        out = std::move(op);
        return NPC_SUCCESS;
    }
    // ---- Bt^T as CSR over trace rows: column ids = positions in t (ascending)
    std::vector<int> trp(n + 1, 0);
    for (int i = 0; i < n; ++i) trp[i + 1] = trp[i] + tcount[i + 1];
    std::vector<int> fill(trp.begin(), trp.end() - 1);
    std::vector<int> tc((size_t)op->nnz + 8, 0);
    std::vector<double> tv((size_t)op->nnz + 8, 0.0);
    for (int pos = 0; pos < op->nbp; ++pos) {
        const int q = order[pos];
        if (q < 0) continue;
        const int ch = pos / 32, l = pos % 32;
        for (int j = 0; j < clen[ch]; ++j) {
            const size_t slot = (size_t)coff[ch] + (size_t)j * 32 + l;
            const int i = scols[slot];
            tc[fill[i]] = pos;
            tv[fill[i]] = svals[slot];
            fill[i]++;
        }
    }
    op->ntiles = std::max(1, ceil_div(n, ST_TILE));
    // split the t positions into K ranges; part k keeps each row's entries with positions in
    // range k (rows' entries are in ascending position order, so parts are row sub-ranges)
    int K = 2;  // measured best at config 5 (96 MB of t): 1 -> 718, 2 -> 349, 3 -> 392, 4 -> 384 us/degree
    if (const char *e = getenv("NPC_SCHUR_SPLIT")) K = std::max(1, std::min(16, atoi(e)));
    const long long P = std::max(1LL, ((long long)op->nbp + K - 1) / K);
    for (int k = 0; k < K; ++k) op->parts.push_back(std::make_unique<SchurOperator::Part>());
    // per-row entry counts of every part, then each part's CSR filled in parallel row chunks
    std::vector<std::vector<int>> prp(K, std::vector<int>(n + 1, 0));
    for (int i = 0; i < n; ++i)
        for (int q = trp[i]; q < trp[i + 1]; ++q) prp[tc[q] / P][i + 1]++;
    for (int k = 0; k < K; ++k)
        for (int i = 0; i < n; ++i) prp[k][i + 1] += prp[k][i];
    for (int k = 0; k < K; ++k) {
        SchurOperator::Part &pt = *op->parts[k];
        std::vector<int> &rp = prp[k];
        std::vector<int> pc((size_t)rp[n] + 8, 0);  // + pad: aligned bulk copies may read past the end
        std::vector<double> pv((size_t)rp[n] + 8, 0.0);
        host_parallel_for(n, [&](long long b, long long e, int) {
            for (long long i = b; i < e; ++i) {
                int o = rp[i];
                for (int q = trp[i]; q < trp[i + 1]; ++q)
                    if (tc[q] / P == k) {
                        pc[o] = tc[q];
                        pv[o++] = tv[q];
                    }
            }
        });
        for (int tt = 0; tt * ST_TILE < n; ++tt) {
            const int r0 = tt * ST_TILE, r1 = std::min(n, r0 + ST_TILE);
            const int pb = rp[r0], pe = rp[r1];
            pt.vspan = std::max(pt.vspan, ((pe + 1) & ~1) - (pb & ~1));
            pt.cspan = std::max(pt.cspan, ((pe + 3) & ~3) - (pb & ~3));
        }
        pt.vspan = (pt.vspan + 1) & ~1;
        pt.smem = (size_t)pt.vspan * 8 + (size_t)pt.cspan * 4 + 16;
        pt.staged = pt.smem <= (size_t)ST_MAX_SMEM;
        NPC_TRY(pt.rowptr.alloc(sizeof(int) * (n + 1)));
        NPC_TRY(pt.cols.alloc(sizeof(int) * pc.size()));
        NPC_TRY(pt.vals.alloc(sizeof(double) * pv.size()));
        NPC_CUDA_TRY(cudaMemcpy(pt.rowptr.p, rp.data(), sizeof(int) * (n + 1), cudaMemcpyHostToDevice));
        NPC_CUDA_TRY(cudaMemcpy(pt.cols.p, pc.data(), sizeof(int) * pc.size(), cudaMemcpyHostToDevice));
        NPC_CUDA_TRY(cudaMemcpy(pt.vals.p, pv.data(), sizeof(double) * pv.size(), cudaMemcpyHostToDevice));
    }
    NPC_TRY(op->yacc.alloc(sizeof(double) * std::max(n, 1)));
    // ---- upload
    NPC_TRY(op->cshift.alloc(sizeof(double) * std::max(n, 1)));
    NPC_TRY(op->t.alloc(sizeof(double) * std::max(op->nbp, 1)));
    NPC_TRY(op->chunk_off.alloc(sizeof(int) * (op->nchunks + 1)));
    NPC_TRY(op->chunk_len.alloc(sizeof(int) * std::max(op->nchunks, 1)));
    NPC_TRY(op->bcols.alloc(sizeof(int) * std::max<long long>(op->nslots, 1)));
    NPC_TRY(op->bvals.alloc(sizeof(double) * std::max<long long>(op->nslots, 1)));

    if (n) NPC_CUDA_TRY(cudaMemcpy(op->cshift.p, d->c, sizeof(double) * n, cudaMemcpyHostToDevice));
    NPC_CUDA_TRY(cudaMemset(op->t.p, 0, op->t.bytes));
    NPC_CUDA_TRY(cudaMemcpy(op->chunk_off.p, coff.data(), sizeof(int) * coff.size(), cudaMemcpyHostToDevice));
    if (op->nchunks) {
        NPC_CUDA_TRY(cudaMemcpy(op->chunk_len.p, clen.data(), sizeof(int) * clen.size(), cudaMemcpyHostToDevice));
        NPC_CUDA_TRY(cudaMemcpy(op->bcols.p, scols.data(), sizeof(int) * scols.size(), cudaMemcpyHostToDevice));
        NPC_CUDA_TRY(cudaMemcpy(op->bvals.p, svals.data(), sizeof(double) * svals.size(), cudaMemcpyHostToDevice));
    }

    out = std::move(op);
    return NPC_SUCCESS;
}

// ---------------------------------------------------------------- callback operator
class CallbackOperator : public Operator {
  public:
    npc_apply_fn fn = nullptr;
    void *user = nullptr;
    DevBuf y;
    bool capture_safe() const override { return false; }
    int num_partials() const override { return vec_grid(n_local); }
    double bytes_per_step(bool has_s2, bool has_r) const override {
        double b = 3.0 * 8.0 * n_local;  // epilogue only: y, x, out (the user's A is opaque)
        if (has_s2) b += 8.0 * n_local;
        if (has_r) b += 8.0 * n_local;
        return b;
    }
    npc_status step(const StepArgs &s) override {
        if (n_local == 0) return NPC_SUCCESS;
        int rc = fn(user, s.x, y.as<double>(), (void *)ctx->stream);
        if (rc != 0) {
            set_error("callback operator returned %d", rc);
            return NPC_ERR_INVALID_ARGUMENT;
        }
        NPC_CUDA_TRY(cudaGetLastError());
        return launch_axpby_step(ctx, y.as<double>(), s, n_local);
    }
};

npc_status make_callback_operator(Context *ctx, const npc_operator_desc *d, std::unique_ptr<Operator> &out) {
    if (!d->apply) {
        set_error("CALLBACK: apply is NULL");
        return NPC_ERR_INVALID_ARGUMENT;
    }
    // nranks > 1: the user's apply owns its halo traffic; the library allreduces the dots.
    auto op = std::make_unique<CallbackOperator>();
    op->ctx = ctx;
    op->kind = NPC_OP_CALLBACK;
    op->n_local = d->n_local;
    op->n_global = d->n_global ? d->n_global : d->n_local;
    op->row_begin = d->row_begin;
    op->fn = d->apply;
    op->user = d->user;
    NPC_TRY(op->y.alloc(sizeof(double) * std::max(d->n_local, 1)));
    out = std::move(op);
    return NPC_SUCCESS;
}

}  // namespace npc
