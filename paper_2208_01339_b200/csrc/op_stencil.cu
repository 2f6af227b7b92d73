// op_stencil.cu -- matrix-free constant-coefficient 2D 5-point / 3D 7-point Dirichlet
// operator (BASELINE config 2) with the Chebyshev recurrence fused in.
//
// "only the application of the matrix to a vector is available as a routine (matrix-free
// regime)".  Kernel: 32x8 threads own an (x, y) tile and march along z,
// keeping x[z-1], x[z], x[z+1] in registers (2.5D blocking) so each plane of the input is
// read from L2/HBM once; the in-plane neighbours come from L1.  Epilogue as in op_csr.cu.
// Multi-rank: z-slabs; ghost planes z_begin-1 and z_end arrive through the generic halo
// (planes are contiguous row ranges), overlapped with the interior planes.
#include <algorithm>

#include "device_util.cuh"
#include "npc_internal.cuh"

namespace npc {

static constexpr int ST_BX = 32, ST_BY = 8, ST_ZC = 8;

struct StencilDev {
    int nx, ny, nzl;
    double diag, off;
    const double *glo;  // ghost plane below z = 0 (nullable)
    const double *ghi;  // ghost plane above z = nzl-1 (nullable)
};

template <int DIM, bool HAS_S2, bool HAS_R, bool DOT>
__global__ void __launch_bounds__(ST_BX *ST_BY) k_stencil_step(StencilDev S, StepArgs s, int z_lo, int z_hi, int zc) {
    if (s.done && *s.done) return;
    __shared__ double red[ST_BX * ST_BY / 32];
    const int x = blockIdx.x * ST_BX + threadIdx.x;
    const int y = blockIdx.y * ST_BY + threadIdx.y;
    const int z0 = z_lo + blockIdx.z * zc;
    const int z1 = min(z0 + zc, z_hi);
    const long long plane = (long long)S.nx * S.ny;
    const double *__restrict__ X = s.x;
    double acc = 0.0;
    if (x < S.nx && y < S.ny && z0 < z1) {
        const int pidx = x + S.nx * y;
        long long i = pidx + plane * z0;
        double below = 0.0, cur = X[i];
        if (DIM == 3) {
            if (z0 > 0)
                below = X[i - plane];
            else if (S.glo)
                below = S.glo[pidx];
        }
        for (int z = z0; z < z1; ++z, i += plane) {
            double above = 0.0;
            if (DIM == 3) {
                if (z + 1 < S.nzl)
                    above = X[i + plane];
                else if (S.ghi)
                    above = S.ghi[pidx];
            }
            double nb = below;
            if (y > 0) nb += X[i - S.nx];
            if (x > 0) nb += X[i - 1];
            if (x < S.nx - 1) nb += X[i + 1];
            if (y < S.ny - 1) nb += X[i + S.nx];
            nb += above;
            const double ax = S.diag * cur + S.off * nb;
            double o = s.a * ax + s.b * cur;
            if (HAS_S2) o += s.c * s.s2[i];
            if (HAS_R) o += s.d * s.r[i];
            s.out[i] = o;
            if (DOT) acc += o * s.dotv[i];
            below = cur;
            cur = above;
        }
    }
    if (DOT) {
        acc = block_sum<ST_BX * ST_BY>(acc, red);
        if (threadIdx.x == 0 && threadIdx.y == 0) s.partials[linear_bid()] = acc;
    }
}

// ---------------------------------------------------------------- temporal blocking
// Two consecutive degrees in one pass (goes beyond the paper), used
// for stencils whose vectors do not fit L2 (see supports_step2):
//     s_j     = a1 A s_{j-1} + b1 s_{j-1} + c1 s_{j-2} + d1 r
//     s_{j+1} = a2 A s_j     + b2 s_j     + c2 s_{j-1} + d2 r
// A CTA owns a TBX x TBY tile of a z-chunk and marches z.  s_{j-1} is staged in shared
// memory with a halo of 2 (ring of 3 planes), s_j is computed on the tile + a halo of 1
// (ring of 3 planes, zero outside the domain: Dirichlet), and s_{j+1} on the tile.  Per
// interior point and two degrees the pass reads s_{j-1}, s_{j-2}, r and writes s_j, s_{j+1}:
// 5 vector streams instead of 8 (the halo re-reads hit L2).  Outputs go to two buffers that
// are not inputs (neighbouring tiles still read s_{j-1} and s_{j-2} near the tile border).
static constexpr int TBX = 32, TBY = 8, TBT = TBX * TBY;
static constexpr int TPX = TBX + 4, TPY = TBY + 4;  // s_{j-1} plane with halo 2
static constexpr int TQX = TBX + 2, TQY = TBY + 2;  // s_j plane with halo 1
static constexpr int NPE = (TPX * TPY + TBT - 1) / TBT, NQE = (TQX * TQY + TBT - 1) / TBT;

struct Step2Args {
    const double *x1;   // s_{j-1}
    const double *x2;   // s_{j-2} (nullable: c1 = 0)
    const double *r;
    double *o1, *o2;    // s_j, s_{j+1}
    const double *dotv; // partial <s_{j+1}, dotv> (nullable)
    double *partials;
    const int *done;
    double a1, b1, c1, d1, a2, b2, c2, d2;
};

// Software-pipelined: while plane zz is computed, the loads of s_{j-1} at plane zz+2 and of
// s_{j-2}, r at plane zz+1 are in flight in registers.  Rings of 4 (s_{j-1}, s_j) and 3 (r)
// planes let two barriers per plane suffice.
template <bool DOT>
__global__ void __launch_bounds__(TBT) k_stencil_step2(int nx, int ny, int nz, int zc, double diag, double off,
                                                      Step2Args S) {
    if (S.done && *S.done) return;
    __shared__ double P[4][TPY * TPX];  // s_{j-1}
    __shared__ double Q[4][TQY * TQX];  // s_j
    __shared__ double Rr[3][TQY * TQX]; // r at the s_j points
    __shared__ double red[TBT / 32];
    const int tid = threadIdx.y * TBX + threadIdx.x;
    const int gx0 = blockIdx.x * TBX, gy0 = blockIdx.y * TBY;
    const int z0 = blockIdx.z * zc, z1 = min(z0 + zc, nz);
    const long long plane = (long long)nx * ny;
    // this thread's P and Q elements: global (x, y) offsets, or -1 outside the domain
    long long pidx[NPE], qidx[NQE];
#pragma unroll
    for (int u = 0; u < NPE; ++u) {
        const int e = tid + u * TBT;
        const int gx = gx0 + e % TPX - 2, gy = gy0 + e / TPX - 2;
        pidx[u] = (e < TPX * TPY && gx >= 0 && gx < nx && gy >= 0 && gy < ny) ? gx + (long long)nx * gy : -1;
    }
#pragma unroll
    for (int u = 0; u < NQE; ++u) {
        const int e = tid + u * TBT;
        const int gx = gx0 + e % TQX - 1, gy = gy0 + e / TQX - 1;
        qidx[u] = (e < TQX * TQY && gx >= 0 && gx < nx && gy >= 0 && gy < ny) ? gx + (long long)nx * gy : -1;
    }
    auto ldP = [&](int u, int zz) -> double {
        return (pidx[u] >= 0 && zz >= 0 && zz < nz) ? S.x1[pidx[u] + plane * zz] : 0.0;
    };
    auto ldQ = [&](const double *v, int u, int zz) -> double {
        return (v && qidx[u] >= 0 && zz >= 0 && zz < nz) ? v[qidx[u] + plane * zz] : 0.0;
    };
    auto stP = [&](int zz, const double *vals) {
#pragma unroll
        for (int u = 0; u < NPE; ++u) {
            const int e = tid + u * TBT;
            if (e < TPX * TPY) P[(zz + 4) & 3][e] = vals[u];
        }
    };
    // prologue: s_{j-1} planes z0-2, z0-1 stored; plane z0 and s_{j-2}, r of plane z0-1 loaded
    double pn[NPE], s2c[NQE], rc[NQE], s2n[NQE], rn[NQE];
    {
        double t[NPE];
#pragma unroll
        for (int u = 0; u < NPE; ++u) t[u] = ldP(u, z0 - 2);
        stP(z0 - 2, t);
#pragma unroll
        for (int u = 0; u < NPE; ++u) t[u] = ldP(u, z0 - 1);
        stP(z0 - 1, t);
    }
#pragma unroll
    for (int u = 0; u < NPE; ++u) pn[u] = ldP(u, z0);
#pragma unroll
    for (int u = 0; u < NQE; ++u) {
        s2c[u] = ldQ(S.x2, u, z0 - 1);
        rc[u] = ldQ(S.r, u, z0 - 1);
    }
    double acc = 0.0;
    for (int zz = z0 - 1; zz <= z1; ++zz) {
        stP(zz + 1, pn);  // s_{j-1} plane zz+1 (prefetched in the previous iteration)
        __syncthreads();
        // next loads in flight during this plane's compute
#pragma unroll
        for (int u = 0; u < NPE; ++u) pn[u] = ldP(u, zz + 2);
#pragma unroll
        for (int u = 0; u < NQE; ++u) {
            s2n[u] = ldQ(S.x2, u, zz + 1);
            rn[u] = ldQ(S.r, u, zz + 1);
        }
        // s_j at plane zz on the tile + halo 1
        const double *Pm = P[(zz + 3) & 3], *P0 = P[(zz + 4) & 3], *Pp = P[(zz + 5) & 3];
        double *Qz = Q[(zz + 4) & 3], *Rz = Rr[(zz + 3) % 3];
#pragma unroll
        for (int u = 0; u < NQE; ++u) {
            const int e = tid + u * TBT;
            if (e < TQX * TQY) {
                double v = 0.0;
                if (qidx[u] >= 0 && zz >= 0 && zz < nz) {
                    const int pe = (e / TQX + 1) * TPX + e % TQX + 1;  // position in P
                    const double cur = P0[pe];
                    double nb = Pm[pe];
                    nb += P0[pe - TPX];
                    nb += P0[pe - 1];
                    nb += P0[pe + 1];
                    nb += P0[pe + TPX];
                    nb += Pp[pe];
                    const double ax = diag * cur + off * nb;
                    v = S.a1 * ax + S.b1 * cur;
                    if (S.x2) v += S.c1 * s2c[u];
                    v += S.d1 * rc[u];
                }
                Qz[e] = v;
                Rz[e] = rc[u];
            }
        }
        __syncthreads();
        // s_{j+1} at plane zz-1 on the tile, from s_j planes zz-2, zz-1, zz
        const int zo = zz - 1;
        if (zo >= z0 && zo < z1) {
            const int gx = gx0 + threadIdx.x, gy = gy0 + threadIdx.y;
            if (gx < nx && gy < ny) {
                const double *Qm = Q[(zo + 3) & 3], *Q0 = Q[(zo + 4) & 3], *Qp = Q[(zo + 5) & 3];
                const int qe = (threadIdx.y + 1) * TQX + threadIdx.x + 1;
                const double cur = Q0[qe];
                double nb = Qm[qe];
                nb += Q0[qe - TQX];
                nb += Q0[qe - 1];
                nb += Q0[qe + 1];
                nb += Q0[qe + TQX];
                nb += Qp[qe];
                const double ax = diag * cur + off * nb;
                const double sjm1 = P[(zo + 4) & 3][(threadIdx.y + 2) * TPX + threadIdx.x + 2];
                const double o = S.a2 * ax + S.b2 * cur + S.c2 * sjm1 + S.d2 * Rr[(zo + 3) % 3][qe];
                const long long i = gx + (long long)nx * gy + plane * zo;
                S.o1[i] = cur;
                S.o2[i] = o;
                if (DOT) acc += o * S.dotv[i];
            }
        }
#pragma unroll
        for (int u = 0; u < NQE; ++u) {
            s2c[u] = s2n[u];
            rc[u] = rn[u];
        }
    }
    if (DOT) {
        acc = block_sum<TBT>(acc, red);
        if (tid == 0) S.partials[linear_bid()] = acc;
    }
}

class StencilOperator : public Operator {
  public:
    int dim = 3, nx = 0, ny = 0, nzg = 1, zb = 0, nzl = 1;
    double diag = 0, off = 0;
    bool multi = false, has_lo = false, has_hi = false;
    int zc_main = ST_ZC;  // z-planes marched per CTA (NPC_ST_ZC for A/B)
    HaloPlan plan;
    HaloRuntime halo;

    dim3 grid_for(int nplanes, int zc) const {
        return dim3(ceil_div(nx, ST_BX), ceil_div(ny, ST_BY), std::max(1, ceil_div(nplanes, zc)));
    }
    int blocks_for(int nplanes, int zc) const {
        dim3 g = grid_for(nplanes, zc);
        return (int)(g.x * g.y * g.z);
    }
    // multi-rank launch segments: the planes that need no ghost (launched while the halo is in
    // flight) and then the boundary planes next to a neighbour rank (after the halo wait); a
    // side without a neighbour (the global z boundary) is part of the first segment
    struct Seg {
        int z0, z1, zc;
        bool after_wait;
    };
    int segments(Seg *o) const {
        if (nzl <= 0) return 0;
        int n = 0;
        const int lo_i = has_lo ? 1 : 0, hi_i = std::max(lo_i, has_hi ? nzl - 1 : nzl);
        if (hi_i > lo_i) o[n++] = {lo_i, hi_i, zc_main, false};
        if (lo_i == 1) o[n++] = {0, 1, 1, true};
        if (hi_i < nzl) o[n++] = {hi_i, nzl, 1, true};
        return n;
    }
    int num_partials() const override {
        if (!multi) return blocks_for(nzl, zc_main);
        Seg sg[3];
        const int ns = segments(sg);
        int tot = 0;
        for (int i = 0; i < ns; ++i) tot += blocks_for(sg[i].z1 - sg[i].z0, sg[i].zc);
        return std::max(tot, 1);
    }
    double bytes_per_step(bool has_s2, bool has_r) const override {
        double b = 2.0 * 8.0 * n_local;  // read x once, write out
        if (has_s2) b += 8.0 * n_local;
        if (has_r) b += 8.0 * n_local;
        return b;
    }

    template <int D, bool H2, bool HR, bool DT>
    npc_status launch_t(const StepArgs &s, int z_lo, int z_hi, int zc, double *partials) {
        if (z_hi <= z_lo) return NPC_SUCCESS;
        StencilDev S{nx, ny, nzl, diag, off, nullptr, nullptr};
        if (multi) {
            const double *g = halo.ghost_buf.as<double>();
            S.glo = has_lo ? g : nullptr;
            S.ghi = has_hi ? g + (has_lo ? (long long)nx * ny : 0) : nullptr;
        }
        StepArgs a = s;
        a.partials = partials;
        k_stencil_step<D, H2, HR, DT><<<grid_for(z_hi - z_lo, zc), dim3(ST_BX, ST_BY), 0, ctx->stream>>>(S, a, z_lo, z_hi, zc);
        NPC_LAUNCH_CHECK();
        return NPC_SUCCESS;
    }
    template <int D>
    npc_status launch_d(const StepArgs &s, int z_lo, int z_hi, int zc, double *p) {
        const bool h2 = s.s2 != nullptr, hr = s.r != nullptr, dt = s.dotv != nullptr;
        if (h2 && hr && dt) return launch_t<D, true, true, true>(s, z_lo, z_hi, zc, p);
        if (h2 && hr) return launch_t<D, true, true, false>(s, z_lo, z_hi, zc, p);
        if (h2 && dt) return launch_t<D, true, false, true>(s, z_lo, z_hi, zc, p);
        if (h2) return launch_t<D, true, false, false>(s, z_lo, z_hi, zc, p);
        if (hr && dt) return launch_t<D, false, true, true>(s, z_lo, z_hi, zc, p);
        if (hr) return launch_t<D, false, true, false>(s, z_lo, z_hi, zc, p);
        if (dt) return launch_t<D, false, false, true>(s, z_lo, z_hi, zc, p);
        return launch_t<D, false, false, false>(s, z_lo, z_hi, zc, p);
    }
    npc_status launch(const StepArgs &s, int z_lo, int z_hi, int zc, double *p) {
        return dim == 3 ? launch_d<3>(s, z_lo, z_hi, zc, p) : launch_d<2>(s, z_lo, z_hi, zc, p);
    }

    // z-chunk of the fused pass: about 4 CTAs per SM (the register-limited residency) in one
    // wave; each chunk recomputes s_j on its two boundary planes, so chunks are not made shorter
    int zc2() const {
        const long long tiles = (long long)ceil_div(nx, TBX) * ceil_div(ny, TBY);
        const long long want = 4LL * ctx->num_sms;
        return std::max(4, ceil_div((long long)nzl * tiles, std::max(want, 1LL)));
    }
    dim3 grid2() const { return dim3(ceil_div(nx, TBX), ceil_div(ny, TBY), std::max(1, ceil_div(nzl, zc2()))); }
    // Measured (profiles/r01_temporal_blocking.md): the fused pass is ~10 % faster per degree
    // when the four vector streams exceed L2 (HBM-bound: 200^3, 256^3) and 1.6x slower when
    // they are L2-resident (128^3, config 2), so it is used only above ~3/4 of the L2 size.
    // NPC_STEP2=1 forces it on, NPC_NO_STEP2=1 off.
    bool supports_step2() const override {
        // multi-rank: only in a 1-rank distributed context -- a neighbour's plane would be
        // needed two degrees deep
        if (dim != 3 || (multi && ctx->nranks > 1) || n_local == 0 || getenv("NPC_NO_STEP2")) return false;
        if (getenv("NPC_STEP2")) return true;
        int l2 = 0;
        if (cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, ctx->device) != cudaSuccess || l2 <= 0)
            l2 = 126 << 20;
        return 4.0 * 8.0 * n_local > 0.75 * l2;
    }
    int num_partials2() const override {
        dim3 g = grid2();
        return (int)(g.x * g.y * g.z);
    }
    double bytes_per_step2() const override { return 5.0 * 8.0 * n_local; }
    npc_status step2(const StepArgs &s1, const StepArgs &s2) override {
        Step2Args S{s1.x, s1.s2, s1.r, s1.out, s2.out, s2.dotv, s2.partials, s1.done,
                    s1.a, s1.b, s1.c, s1.d, s2.a, s2.b, s2.c, s2.d};
        if (!S.r) {
            set_error("stencil step2: r is required");
            return NPC_ERR_INVALID_ARGUMENT;
        }
        const int zc = zc2();
        if (s2.dotv)
            k_stencil_step2<true><<<grid2(), dim3(TBX, TBY), 0, ctx->stream>>>(nx, ny, nzl, zc, diag, off, S);
        else
            k_stencil_step2<false><<<grid2(), dim3(TBX, TBY), 0, ctx->stream>>>(nx, ny, nzl, zc, diag, off, S);
        NPC_LAUNCH_CHECK();
        return NPC_SUCCESS;
    }

    npc_status step(const StepArgs &s) override {
        if (n_local == 0 && !multi) return NPC_SUCCESS;
        if (!multi) return launch(s, 0, nzl, zc_main, s.partials);
        Seg sg[3];
        const int ns = segments(sg);
        double *p = s.partials;
        if (ns == 0) return p ? launch_fill(ctx, p, 0.0, 1) : NPC_SUCCESS;
        const bool need_halo = ctx->nranks > 1;  // collective for the local transport
        if (need_halo) NPC_TRY(halo_start(ctx, plan, halo, s.x));
        bool waited = !need_halo;
        for (int i = 0; i < ns; ++i) {
            if (sg[i].after_wait && !waited) {
                NPC_TRY(halo_wait(ctx, halo));
                waited = true;
            }
            NPC_TRY(launch(s, sg[i].z0, sg[i].z1, sg[i].zc, p));
            if (p) p += blocks_for(sg[i].z1 - sg[i].z0, sg[i].zc);
        }
        return NPC_SUCCESS;
    }
};

npc_status make_stencil_operator(Context *ctx, const npc_operator_desc *d, std::unique_ptr<Operator> &out) {
    if (d->stencil_dim != 2 && d->stencil_dim != 3) {
        set_error("stencil: dim must be 2 or 3");
        return NPC_ERR_INVALID_ARGUMENT;
    }
    if (d->nx < 1 || d->ny < 1 || (d->stencil_dim == 3 && (d->nz_global < 1 || d->nz_local < 0 || d->z_begin < 0 ||
                                                            d->z_begin + d->nz_local > d->nz_global))) {
        set_error("stencil: invalid grid");
        return NPC_ERR_DIMENSION;
    }
    if (!std::isfinite(d->diag) || !std::isfinite(d->offdiag)) {
        set_error("stencil: non-finite coefficients");
        return NPC_ERR_INVALID_ARGUMENT;
    }
    auto op = std::make_unique<StencilOperator>();
    op->ctx = ctx;
    op->kind = NPC_OP_STENCIL;
    op->dim = d->stencil_dim;
    op->nx = d->nx;
    op->ny = d->ny;
    op->nzg = d->stencil_dim == 3 ? d->nz_global : 1;
    op->zb = d->stencil_dim == 3 ? d->z_begin : 0;
    op->nzl = d->stencil_dim == 3 ? d->nz_local : 1;
    op->diag = d->diag;
    op->off = d->offdiag;
    if (const char *e = getenv("NPC_ST_ZC")) op->zc_main = std::max(1, atoi(e));
    const long long plane = (long long)op->nx * op->ny;
    if (plane * op->nzl >= (1LL << 31)) {
        set_error("stencil: more than 2^31 local rows");
        return NPC_ERR_UNSUPPORTED;
    }
    op->n_local = (int)(plane * op->nzl);
    op->n_global = plane * op->nzg;
    op->row_begin = plane * op->zb;
    if (d->n_local != op->n_local || (d->n_global && d->n_global != op->n_global)) {
        set_error("stencil: n_local/n_global disagree with the grid");
        return NPC_ERR_DIMENSION;
    }
    if (ctx->distributed()) {
        if (op->dim != 3) {
            set_error("stencil: multi-rank needs dim 3 (z-slabs)");
            return NPC_ERR_UNSUPPORTED;
        }
        op->multi = true;
        // neighbours in z: the ranks owning plane zb-1 and plane zb+nzl (ranks ordered by z)
        op->has_lo = op->zb > 0;
        op->has_hi = op->zb + op->nzl < op->nzg;
        HaloPlan &P = op->plan;
        const int R = ctx->nranks, me = ctx->rank;
        P.recv_count.assign(R, 0);
        P.recv_off.assign(R, 0);
        P.send_count.assign(R, 0);
        P.send_off.assign(R, 0);
        if ((op->has_lo && me == 0) || (op->has_hi && me == R - 1)) {
            set_error("stencil: z-slabs must be assigned to ranks in z order");
            return NPC_ERR_DIMENSION;
        }
        int off = 0;
        if (op->has_lo) {
            P.recv_count[me - 1] = (int)plane;
            P.recv_off[me - 1] = 0;
            P.send_count[me - 1] = (int)plane;
            for (long long k = 0; k < plane; ++k) P.send_idx.push_back((int)k);
            off = (int)plane;
        }
        if (op->has_hi) {
            P.recv_count[me + 1] = (int)plane;
            P.recv_off[me + 1] = off;
            P.send_off[me + 1] = (int)P.send_idx.size();
            P.send_count[me + 1] = (int)plane;
            for (long long k = 0; k < plane; ++k) P.send_idx.push_back((int)(plane * (op->nzl - 1) + k));
        }
        P.n_ghost = off + (op->has_hi ? (int)plane : 0);
        NPC_TRY(halo_setup(ctx, P, op->halo));
    }
    out = std::move(op);
    return NPC_SUCCESS;
}

}  // namespace npc
