// op_schur.cu -- matrix-free Schur-complement operator S = C + B^T D^{-1} B (BASELINE
// config 5), never assembled, with the Chebyshev recurrence fused into the second pass.
//
// This is the "global sparse product - local inverse - transposed product" shape of the
// paper's S_u application (Alg. 3), with D standing in for
// the block-diagonal A^{-1} and C = tridiag(-1, 2 + c, -1) for G^u.
//   create: Bt = D^{-1/2} B (so S = C + Bt^T Bt, D is never read per application); the rows
//           of Bt are reordered by length (2, 3, 4 entries) -- the order of B's rows is free
//           since t = Bt v is internal -- and stored SELL-32 column-major: no padding except
//           the tail chunk of each length class, every load coalesced.
//   pass 1 (k_schur_bpass):   t_q = sum_p Bt_qp v_p ;  y[col_p] += Bt_qp t_q  (fp64 atomics
//                              into y, which stays L2-resident)
//   pass 2 (k_schur_tstep):   (S v)_i = (2 + c_i) v_i - v_{i-1} - v_{i+1} + y_i ; y_i = 0 ;
//                              out = a (S v) + b v + c s2 + d r   (+ dot partial)
#include <algorithm>
#include <numeric>

#include "device_util.cuh"
#include "npc_internal.cuh"

namespace npc {

static constexpr int SB_WARPS = 8;
static constexpr int ST_T = 256;

__global__ void __launch_bounds__(32 * SB_WARPS) k_schur_bpass(const int *__restrict__ chunk_off,
                                                               const int *__restrict__ chunk_len, int nchunks,
                                                               const int *__restrict__ cols,
                                                               const double *__restrict__ vals, int nrows,
                                                               const double *__restrict__ v, double *y,
                                                               const int *done) {
    if (done && *done) return;
    const int lane = threadIdx.x & 31;
    const int ch = blockIdx.x * SB_WARPS + (threadIdx.x >> 5);
    if (ch >= nchunks) return;
    const int row = ch * 32 + lane;
    const int len = chunk_len[ch];
    const long long base = (long long)chunk_off[ch] + lane;
    int c[4];
    double b[4];
    double t = 0.0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        if (j < len) {
            c[j] = __ldcs(cols + base + 32LL * j);
            b[j] = __ldcs(vals + base + 32LL * j);
            t += b[j] * __ldg(v + c[j]);
        }
    }
    if (row >= nrows) return;
#pragma unroll
    for (int j = 0; j < 4; ++j)
        if (j < len) atomicAdd(y + c[j], b[j] * t);
}

template <bool HAS_S2, bool HAS_R, bool DOT>
__global__ void __launch_bounds__(ST_T) k_schur_tstep(const double *__restrict__ cshift, double *y, int n, StepArgs s) {
    if (s.done && *s.done) return;
    __shared__ double red[ST_T / 32];
    double acc = 0.0;
    const double *__restrict__ X = s.x;
    for (int i = blockIdx.x * ST_T + threadIdx.x; i < n; i += gridDim.x * ST_T) {
        const double xi = X[i];
        double sv = (2.0 + cshift[i]) * xi;
        if (i > 0) sv -= X[i - 1];
        if (i < n - 1) sv -= X[i + 1];
        sv += y[i];
        y[i] = 0.0;
        double o = s.a * sv + s.b * xi;
        if (HAS_S2) o += s.c * s.s2[i];
        if (HAS_R) o += s.d * s.r[i];
        s.out[i] = o;
        if (DOT) acc += o * s.dotv[i];
    }
    if (DOT) {
        acc = block_sum<ST_T>(acc, red);
        if (threadIdx.x == 0) s.partials[blockIdx.x] = acc;
    }
}

class SchurOperator : public Operator {
  public:
    DevBuf cshift, chunk_off, chunk_len, cols, vals, y;
    int nb = 0, nchunks = 0;
    long long nnz = 0, nslots = 0;
    int grid2 = 1;

    int num_partials() const override { return grid2; }
    double bytes_per_step(bool has_s2, bool has_r) const override {
        // Bt slots once (D folded in), c once, x read once, y written (atomics) + read/reset,
        // out written; s_{j-2}, r when present.  SURVEY §8(d) row 5 (the ~704 MB variant).
        double b = (double)nslots * 12.0 + 8.0 * n_local /*c*/ + 2.0 * 8.0 * n_local /*x,out*/ +
                   2.0 * 8.0 * n_local /*y*/;
        if (has_s2) b += 8.0 * n_local;
        if (has_r) b += 8.0 * n_local;
        return b;
    }
    template <bool H2, bool HR, bool DT>
    npc_status launch2(const StepArgs &s) {
        k_schur_tstep<H2, HR, DT><<<grid2, ST_T, 0, ctx->stream>>>(cshift.as<double>(), y.as<double>(), n_local, s);
        NPC_LAUNCH_CHECK();
        return NPC_SUCCESS;
    }
    npc_status step(const StepArgs &s) override {
        if (n_local == 0) return NPC_SUCCESS;
        if (nchunks) {
            k_schur_bpass<<<ceil_div(nchunks, SB_WARPS), 32 * SB_WARPS, 0, ctx->stream>>>(
                chunk_off.as<int>(), chunk_len.as<int>(), nchunks, cols.as<int>(), vals.as<double>(), nb, s.x,
                y.as<double>(), s.done);
            NPC_LAUNCH_CHECK();
        }
        const bool h2 = s.s2 != nullptr, hr = s.r != nullptr, dt = s.dotv != nullptr;
        if (h2 && hr && dt) return launch2<true, true, true>(s);
        if (h2 && hr) return launch2<true, true, false>(s);
        if (h2 && dt) return launch2<true, false, true>(s);
        if (h2) return launch2<true, false, false>(s);
        if (hr && dt) return launch2<false, true, true>(s);
        if (hr) return launch2<false, true, false>(s);
        if (dt) return launch2<false, false, true>(s);
        return launch2<false, false, false>(s);
    }
};

npc_status make_schur_operator(Context *ctx, const npc_operator_desc *d, std::unique_ptr<Operator> &out) {
    if (ctx->nranks > 1) {
        set_error("SCHUR: nranks > 1 is not supported in this version");
        return NPC_ERR_UNSUPPORTED;
    }
    const int n = d->n_local, nb = d->b_n_local;
    if (n < 0 || nb < 0 || !d->c || (nb > 0 && (!d->b_rowptr || !d->b_colidx || !d->b_vals || !d->d))) {
        set_error("SCHUR: invalid arrays");
        return NPC_ERR_INVALID_ARGUMENT;
    }
    if ((d->n_global && d->n_global != n) || (d->b_rows_global && d->b_rows_global != nb)) {
        set_error("SCHUR: sizes disagree");
        return NPC_ERR_DIMENSION;
    }
    if (d->b_rowptr[0] != 0) {
        set_error("SCHUR: b_rowptr[0] != 0");
        return NPC_ERR_DIMENSION;
    }
    for (int i = 0; i < n; ++i)
        if (!std::isfinite(d->c[i])) {
            set_error("SCHUR: non-finite c");
            return NPC_ERR_DIMENSION;
        }
    std::vector<int> byl[5];
    for (int q = 0; q < nb; ++q) {
        int L = d->b_rowptr[q + 1] - d->b_rowptr[q];
        if (L < 0 || L > 4) {
            set_error("SCHUR: B rows must have 0..4 entries (row %d has %d)", q, L);
            return L < 0 ? NPC_ERR_DIMENSION : NPC_ERR_UNSUPPORTED;
        }
        if (!(d->d[q] > 0.0) || !std::isfinite(d->d[q])) {
            set_error("SCHUR: D must be positive and finite (row %d)", q);
            return NPC_ERR_DIMENSION;
        }
        for (int p = d->b_rowptr[q]; p < d->b_rowptr[q + 1]; ++p)
            if (d->b_colidx[p] < 0 || d->b_colidx[p] >= n || !std::isfinite(d->b_vals[p])) {
                set_error("SCHUR: bad B entry in row %d", q);
                return NPC_ERR_DIMENSION;
            }
        byl[L].push_back(q);
    }
    auto op = std::make_unique<SchurOperator>();
    op->ctx = ctx;
    op->kind = NPC_OP_SCHUR;
    op->n_local = n;
    op->n_global = n;
    op->nb = nb;
    op->nnz = nb ? d->b_rowptr[nb] : 0;
    // order B rows by length (4, 3, 2, 1; empty rows dropped), chunks of 32 rows
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
    op->nslots = coff.back();
    std::vector<int> scols((size_t)op->nslots, 0);
    std::vector<double> svals((size_t)op->nslots, 0.0);
    for (int ch = 0; ch < op->nchunks; ++ch)
        for (int l = 0; l < 32; ++l) {
            int q = order[(size_t)ch * 32 + l];
            for (int j = 0; j < clen[ch]; ++j) {
                size_t slot = (size_t)coff[ch] + (size_t)j * 32 + l;
                if (q >= 0) {
                    int p = d->b_rowptr[q] + j;
                    scols[slot] = d->b_colidx[p];
                    svals[slot] = d->b_vals[p] / std::sqrt(d->d[q]);
                }
            }
        }
    op->grid2 = vec_grid(n);
    NPC_TRY(op->cshift.alloc(sizeof(double) * std::max(n, 1)));
    NPC_TRY(op->y.alloc(sizeof(double) * std::max(n, 1)));
    NPC_TRY(op->chunk_off.alloc(sizeof(int) * (op->nchunks + 1)));
    NPC_TRY(op->chunk_len.alloc(sizeof(int) * std::max(op->nchunks, 1)));
    NPC_TRY(op->cols.alloc(sizeof(int) * std::max<long long>(op->nslots, 1)));
    NPC_TRY(op->vals.alloc(sizeof(double) * std::max<long long>(op->nslots, 1)));
    if (n) NPC_CUDA_TRY(cudaMemcpy(op->cshift.p, d->c, sizeof(double) * n, cudaMemcpyHostToDevice));
    NPC_CUDA_TRY(cudaMemset(op->y.p, 0, op->y.bytes));
    NPC_CUDA_TRY(cudaMemcpy(op->chunk_off.p, coff.data(), sizeof(int) * coff.size(), cudaMemcpyHostToDevice));
    if (op->nchunks) {
        NPC_CUDA_TRY(cudaMemcpy(op->chunk_len.p, clen.data(), sizeof(int) * clen.size(), cudaMemcpyHostToDevice));
        NPC_CUDA_TRY(cudaMemcpy(op->cols.p, scols.data(), sizeof(int) * scols.size(), cudaMemcpyHostToDevice));
        NPC_CUDA_TRY(cudaMemcpy(op->vals.p, svals.data(), sizeof(double) * svals.size(), cudaMemcpyHostToDevice));
    }
    // rows beyond nb inside padded chunks have value 0 (their atomics add 0.0): the kernel
    // also skips them via the row index of the padded order
    op->nb = (int)order.size();
    out = std::move(op);
    return NPC_SUCCESS;
}

// ---------------------------------------------------------------- callback operator
class CallbackOperator : public Operator {
  public:
    npc_apply_fn fn = nullptr;
    void *user = nullptr;
    DevBuf y;
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
