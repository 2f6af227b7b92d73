// op_dfn.cu -- the paper's DFN Schur complement as a matrix-free operator (SURVEY §8(f) NEXT
// row 2; §4.2-4.3, Eq. schur, Alg. 3, Alg. 4):
//
//     S_u = G^u - a B^T A^-1 C - a C^T A^-1 B + C^T A^-1 G^h A^-1 C      (n^u x n^u)
//
// A, G^h block-diagonal over the fractures (n^h head unknowns), C fracture-local, B = C + E
// global, G^u global.  With dfn_scaled the operator is the Jacobi-scaled
// S^ = D_S^{-1/2} S_u D_S^{-1/2}, D_S = diag(S_u) by Alg. 4, which is what
// the polynomial preconditioner is applied to.
//
// Create (host, setup -- "the exact Cholesky factorization of A is computed"):
//   * banded Cholesky of every diagonal block of A (band = the block's bandwidth in the given
//     ordering; a grid block in natural order has band nx), stored row-wise L[i][i-bw..i];
//   * D_S by Alg. 4 one column of C at a time (z = A_f^-1 c, D_S = G^u_ii + z^T G^h z -
//     2 a z^T b; the printed algorithm's "-2B" assumes a = 1, reading A8), host threads;
//   * the scaling folded into the stored matrices: Cs = C D^-1/2, Bs = B D^-1/2 (input side),
//     BsT = D^-1/2 B^T, CsT = D^-1/2 C^T (output side, stored transposed so the last pass
//     gathers instead of scattering), GuS = D^-1/2 G^u D^-1/2.
// Application (2-3 kernels instead of Alg. 3's 11 steps; everything in steps 1-6 and 8-10 is
// local to a fracture block):
//   k_dfn_dense: blocks of <= DFN_DENSE_MAX rows (the paper's Frac16/32 have ~34): one CTA per
//     block applies the block's explicit inverse A_f^-1 = L_f^-T L_f^-1 (formed on the host from
//     the Cholesky factor; symmetric, so a thread reads its COLUMN -- coalesced).  A serial
//     triangular solve on a 36-row block is a chain of 36 dependent steps per sweep; the
//     explicit inverse turns the 6 solves of Alg. 3 into 3 independent-row dense products (one
//     HBM read of A_f^-1 per application, the second from L2);
//   k_dfn_block: larger blocks: one group of G lanes per block, forward/backward banded solves
//     in shared memory (lanes split the band of a row);
//   both: v = Cs x, z = Bs x on the block's rows; t = A^-1 v, w = A^-1 z; v2 = G^h t;
//     w2 = A^-1 v2; write t and u2 = w2 - a w.
//   k_dfn_out: one thread per u row: y = GuS x - a BsT t + CsT u2  (Alg. 3 steps 7 and 11),
//     fused with the Chebyshev epilogue out = a_j y + b_j x + c_j s2 + d_j r (+ PCG partial).
// Multi-rank: the paper's DSMat partition -- whole fracture blocks per rank,
// u rows grouped by owning fracture (C is fracture-local, so Alg. 4 stays rank-local); per
// application a u-space halo of x (B's E part, G^u) and an h-space halo of t (rows of B^T held
// by other ranks' fractures, gathered once at setup; u2 needs none: C is fracture-local).
// Both halos overlap block work: the fracture blocks are ordered [t sent, no x ghost | t sent,
// x ghosts | t not sent], the first group runs while the x halo is in flight, the last while
// the t halo is, and the ghosts land straight in the tails of xg and t.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <thread>
#include <vector>

#include "device_util.cuh"
#include "npc_internal.cuh"

namespace npc {

static constexpr int DFN_OUT_T = 256;
static constexpr int DFN_MAX_NF = 8192;    // rows of one fracture block (3 x 8 B x rows of smem)
static constexpr int DFN_DENSE_MAX = 128;  // blocks up to this size use the explicit inverse
#ifndef NPC_DFN_UNROLL
#define NPC_DFN_UNROLL 8  // j-loop unroll of the dense products (A/B-tuned)
#endif
#ifndef NPC_DFN_WARPS
#define NPC_DFN_WARPS 8  // blocks (warps) per CTA of the dense kernel (A/B-tuned)
#endif
// NPC_DFN_MINB (A/B builds only): min resident CTAs per SM of the dense kernel.  Left unset
// on purpose: ptxas then settles at 64 registers; an explicit 1 lets it take 108 and cost
// 20 % (8.9 -> 10.7 ms per p_30 on config 6).
#ifdef NPC_DFN_MINB
#define NPC_DFN_LB(t) __launch_bounds__(t, NPC_DFN_MINB)
#else
#define NPC_DFN_LB(t) __launch_bounds__(t)
#endif
static constexpr int DFN_WARPS = NPC_DFN_WARPS;
static constexpr int DFN_UNROLL = NPC_DFN_UNROLL;

struct DfnDev {
    const int *hblk, *bw;
    const long long *loff;
    const double *L;
    const int *crp, *cci;
    const double *cv;
    const int *brp, *bci;
    const double *bv;
    const int *ghrp, *ghci;
    const double *ghv;
    int nblk;
    double alpha;
};

template <int G>
__device__ __forceinline__ double group_sum(double v, unsigned mask) {
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) v += __shfl_xor_sync(mask, v, o, G);
    return v;
}

// In-place forward (L y = rhs) and backward (L^T x = y) banded solves of NR right-hand sides
// held in shared memory, by the G lanes of a group (lanes split the band of each row).
template <int G, int NR>
__device__ __forceinline__ void band_solve(const double *__restrict__ L, int m, int bw, double *r0, double *r1,
                                           int lane, unsigned mask) {
    const int ld = bw + 1;
    for (int i = 0; i < m; ++i) {
        double a0 = 0.0, a1 = 0.0;
        const int kmax = min(bw, i);
        for (int k = 1 + lane; k <= kmax; k += G) {
            const double l = L[(size_t)i * ld + bw - k];
            a0 += l * r0[i - k];
            if (NR == 2) a1 += l * r1[i - k];
        }
        a0 = group_sum<G>(a0, mask);
        if (NR == 2) a1 = group_sum<G>(a1, mask);
        if (lane == 0) {
            const double d = L[(size_t)i * ld + bw];
            r0[i] = (r0[i] - a0) / d;
            if (NR == 2) r1[i] = (r1[i] - a1) / d;
        }
        __syncwarp(mask);
    }
    for (int i = m - 1; i >= 0; --i) {
        double a0 = 0.0, a1 = 0.0;
        const int kmax = min(bw, m - 1 - i);
        for (int k = 1 + lane; k <= kmax; k += G) {
            const double l = L[(size_t)(i + k) * ld + bw - k];
            a0 += l * r0[i + k];
            if (NR == 2) a1 += l * r1[i + k];
        }
        a0 = group_sum<G>(a0, mask);
        if (NR == 2) a1 = group_sum<G>(a1, mask);
        if (lane == 0) {
            const double d = L[(size_t)i * ld + bw];
            r0[i] = (r0[i] - a0) / d;
            if (NR == 2) r1[i] = (r1[i] - a1) / d;
        }
        __syncwarp(mask);
    }
}

template <int G>
__global__ void __launch_bounds__(256) k_dfn_block(DfnDev D, const int *__restrict__ list, int nlist,
                                                   const double *__restrict__ x, double *__restrict__ t_out,
                                                   double *__restrict__ u2_out, int smem_nf, const int *done) {
    if (done && *done) return;
    extern __shared__ __align__(16) double sm[];
    const int lane = threadIdx.x % G, gl = threadIdx.x / G;
    const int li = blockIdx.x * (blockDim.x / G) + gl;
    if (li >= nlist) return;  // the whole group leaves together
    const int f = list[li];
    const unsigned mask = (G == 32) ? 0xffffffffu : (((1u << G) - 1u) << ((threadIdx.x & 31) / G * G));
    double *v = sm + (size_t)gl * 3 * smem_nf, *z = v + smem_nf, *q = z + smem_nf;
    const int h0 = D.hblk[f], m = D.hblk[f + 1] - h0, bw = D.bw[f];
    const double *__restrict__ L = D.L + D.loff[f];
    // Alg. 3 steps 1-2 on the block's rows: v = Cs x, z = Bs x
    for (int i = lane; i < m; i += G) {
        const int row = h0 + i;
        double sv = 0.0, sz = 0.0;
        for (int p = D.crp[row]; p < D.crp[row + 1]; ++p) sv += D.cv[p] * __ldg(x + D.cci[p]);
        for (int p = D.brp[row]; p < D.brp[row + 1]; ++p) sz += D.bv[p] * __ldg(x + D.bci[p]);
        v[i] = sv;
        z[i] = sz;
    }
    __syncwarp(mask);
    band_solve<G, 2>(L, m, bw, v, z, lane, mask);  // steps 3-6: t = A^-1 v, w = A^-1 z
    for (int i = lane; i < m; i += G) {             // step 8: q = G^h t (block-local)
        const int row = h0 + i;
        double s = 0.0;
        for (int p = D.ghrp[row]; p < D.ghrp[row + 1]; ++p) s += D.ghv[p] * v[D.ghci[p] - h0];
        q[i] = s;
        t_out[row] = v[i];
    }
    __syncwarp(mask);
    band_solve<G, 1>(L, m, bw, q, nullptr, lane, mask);  // steps 9-10: w2 = A^-1 q
    for (int i = lane; i < m; i += G) u2_out[h0 + i] = q[i] - D.alpha * z[i];
}

// One WARP per small block (8 blocks per CTA): A_f^-1 applied as dense products (A_f^-1
// symmetric, row-major m x m at doff[f]; lane i reads column i: consecutive lanes ->
// consecutive addresses), RPL rows per lane (m <= 32 RPL).  The kernel is bound by the
// latency of its dependent phases (gather -> product -> G^h -> product), so blocks are
// independent warps synchronised with __syncwarp only (a CTA-per-block variant spent 15 % of
// its issue slots at __syncthreads; a bulk-TMA-staged variant cut residency to 12 warps/SM
// and ran 2.3x slower).
template <int RPL>
__global__ void NPC_DFN_LB(32 * DFN_WARPS) k_dfn_dense(DfnDev D, const int4 *__restrict__ binfo, int nlist,
                                                   const double *__restrict__ Ainv, const double *__restrict__ x,
                                                   double *__restrict__ t_out, double *__restrict__ u2_out,
                                                   const int *done) {
    if (done && *done) return;
    constexpr int MW = 32 * RPL;
    __shared__ double sh[DFN_WARPS][4][MW];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int li = blockIdx.x * DFN_WARPS + wib;
    if (li >= nlist) return;
    double *v = sh[wib][0], *z = sh[wib][1], *tt = sh[wib][2], *q = sh[wib][3];
    // per-block record {h0, m, doff lo, doff hi} + the block's CSR entry ranges of Cs, Bs, G^h:
    // one dependent load, then every byte the block will touch is prefetched into L2 at once,
    // so the dependent phases below wait on L2 instead of HBM
    const int4 bi = binfo[2 * li], br = binfo[2 * li + 1];
    const int h0 = bi.x, m = bi.y;
    const double *__restrict__ Ai = Ainv + (((long long)(unsigned)bi.w << 32) | (unsigned)bi.z);
    {
        const int gb = D.ghrp[h0], ge = D.ghrp[h0 + m];
        auto pf = [&](const void *base, size_t bytes) {
            const char *c = static_cast<const char *>(base);
            for (size_t o = (size_t)lane * 128; o < bytes; o += 32 * 128)
                asm volatile("prefetch.global.L2 [%0];" ::"l"(c + o));
        };
#ifndef NPC_DFN_NOPF_AI
        pf(Ai, (size_t)m * m * 8);
#endif
        pf(D.cv + br.x, (size_t)(br.y - br.x) * 8);
        pf(D.cci + br.x, (size_t)(br.y - br.x) * 4);
        pf(D.bv + br.z, (size_t)(br.w - br.z) * 8);
        pf(D.bci + br.z, (size_t)(br.w - br.z) * 4);
        pf(D.ghv + gb, (size_t)(ge - gb) * 8);
        pf(D.ghci + gb, (size_t)(ge - gb) * 4);
    }
#pragma unroll
    for (int r = 0; r < RPL; ++r) {  // Alg. 3 steps 1-2 on the block's rows
        const int i = lane + 32 * r;
        if (i < m) {
            const int row = h0 + i;
            double sv = 0.0, sz = 0.0;
            const int c0 = D.crp[row], c1 = D.crp[row + 1], b0 = D.brp[row], b1 = D.brp[row + 1];
#pragma unroll 4
            for (int p = c0; p < c1; ++p) sv += D.cv[p] * __ldg(x + D.cci[p]);
#pragma unroll 4
            for (int p = b0; p < b1; ++p) sz += D.bv[p] * __ldg(x + D.bci[p]);
            v[i] = sv;
            z[i] = sz;
        }
    }
    __syncwarp();
    // steps 3-6: t = A^-1 v, w = A^-1 z -- the RPL rows of a lane share one j loop, so their
    // loads are in flight together (rows beyond m load nothing: index clamped, result unused)
    double wi[RPL], ai[RPL];
#pragma unroll
    for (int r = 0; r < RPL; ++r) ai[r] = wi[r] = 0.0;
#pragma unroll DFN_UNROLL
    for (int j = 0; j < m; ++j) {
        const double vj = v[j], zj = z[j];
#pragma unroll
        for (int r = 0; r < RPL; ++r) {
            const int i = lane + 32 * r;
#ifdef NPC_DFN_EVL  // A/B: the first pass marks A_f^-1 evict-last so that the second pass hits L2
            double aij = 0.0;
            if (i < m) {
                const double *pa = Ai + (size_t)j * m + i;
                uint64_t pol;
                asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
                asm volatile("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(aij) : "l"(pa), "l"(pol));
            }
#else
            const double aij = (i < m) ? __ldg(Ai + (size_t)j * m + i) : 0.0;
#endif
            ai[r] += aij * vj;
            wi[r] += aij * zj;
        }
    }
#pragma unroll
    for (int r = 0; r < RPL; ++r) {
        const int i = lane + 32 * r;
        if (i < m) {
            tt[i] = ai[r];
            t_out[h0 + i] = ai[r];
        }
    }
    __syncwarp();
#pragma unroll
    for (int r = 0; r < RPL; ++r) {  // step 8: q = G^h t
        const int i = lane + 32 * r;
        if (i < m) {
            const int row = h0 + i;
            double sq = 0.0;
            const int g0 = D.ghrp[row], g1 = D.ghrp[row + 1];
#pragma unroll 4
            for (int p = g0; p < g1; ++p) sq += D.ghv[p] * tt[D.ghci[p] - h0];
            q[i] = sq;
        }
    }
    __syncwarp();
    // steps 9-10: w2 = A^-1 q; u2 = w2 - a w
#pragma unroll
    for (int r = 0; r < RPL; ++r) ai[r] = 0.0;
#pragma unroll DFN_UNROLL
    for (int j = 0; j < m; ++j) {
        const double qj = q[j];
#pragma unroll
        for (int r = 0; r < RPL; ++r) {
            const int i = lane + 32 * r;
            if (i < m) ai[r] += __ldg(Ai + (size_t)j * m + i) * qj;
        }
    }
#pragma unroll
    for (int r = 0; r < RPL; ++r) {
        const int i = lane + 32 * r;
        if (i < m) u2_out[h0 + i] = ai[r] - D.alpha * wi[r];
    }
}

struct DfnOutDev {
    const int *gurp, *guci;
    const double *guv;
    const int *btrp, *btci;
    const double *btv;
    const int *ctrp, *ctci;
    const double *ctv;
    const double *t, *u2;
    const double *xg;  // x for the G^u gathers (owned rows + ghosts when multi-rank)
    double alpha;
    int n;
};

// y = GuS x - a BsT t + CsT u2 (Alg. 3 steps 7, 11) fused with the recurrence epilogue
template <bool HAS_S2, bool HAS_R, bool DOT>
__global__ void __launch_bounds__(DFN_OUT_T) k_dfn_out(DfnOutDev O, StepArgs s) {
    if (s.done && *s.done) return;
    __shared__ double red[DFN_OUT_T / 32];
    const int i = blockIdx.x * DFN_OUT_T + threadIdx.x;
    double acc = 0.0;
    if (i < O.n) {
        const double *__restrict__ X = s.x;
        double g = 0.0, bt = 0.0, ct = 0.0;
        for (int p = O.gurp[i]; p < O.gurp[i + 1]; ++p) g += O.guv[p] * __ldg(O.xg + O.guci[p]);
        for (int p = O.btrp[i]; p < O.btrp[i + 1]; ++p) bt += O.btv[p] * __ldg(O.t + O.btci[p]);
        for (int p = O.ctrp[i]; p < O.ctrp[i + 1]; ++p) ct += O.ctv[p] * __ldg(O.u2 + O.ctci[p]);
        const double y = g - O.alpha * bt + ct;
        double o = s.a * y + s.b * X[i];
        if (HAS_S2) o += s.c * s.s2[i];
        if (HAS_R) o += s.d * s.r[i];
        s.out[i] = o;
        if (DOT) acc = o * s.dotv[i];
    }
    if (DOT) {
        acc = block_sum<DFN_OUT_T>(acc, red);
        if (threadIdx.x == 0) s.partials[blockIdx.x] = acc;
    }
}

// ---------------------------------------------------------------- host helpers
struct HostCsr {
    std::vector<int> rp, ci;
    std::vector<double> v;
};

static HostCsr transpose(int nrows, int ncols, const int *rp, const int *ci, const double *v) {
    HostCsr T;
    T.rp.assign(ncols + 1, 0);
    const int nnz = rp[nrows];
    for (int p = 0; p < nnz; ++p) T.rp[ci[p] + 1]++;
    for (int j = 0; j < ncols; ++j) T.rp[j + 1] += T.rp[j];
    T.ci.resize(std::max(nnz, 1));
    T.v.resize(std::max(nnz, 1));
    std::vector<int> fill(T.rp.begin(), T.rp.end() - 1);
    for (int i = 0; i < nrows; ++i)  // rows ascending -> columns of T ascending
        for (int p = rp[i]; p < rp[i + 1]; ++p) {
            T.ci[fill[ci[p]]] = i;
            T.v[fill[ci[p]]++] = v[p];
        }
    return T;
}

static npc_status check_csr(const char *name, int nrows, int ncols, const int *rp, const int *ci, const double *v) {
    if (!rp || (rp[nrows] > 0 && (!ci || !v)) || rp[0] != 0) {
        set_error("DFN: %s: missing arrays or rowptr[0] != 0", name);
        return NPC_ERR_INVALID_ARGUMENT;
    }
    for (int i = 0; i < nrows; ++i) {
        if (rp[i + 1] < rp[i]) {
            set_error("DFN: %s: rowptr decreases at row %d", name, i);
            return NPC_ERR_DIMENSION;
        }
        for (int p = rp[i]; p < rp[i + 1]; ++p)
            if (ci[p] < 0 || ci[p] >= ncols || !std::isfinite(v[p])) {
                set_error("DFN: %s: bad entry in row %d", name, i);
                return NPC_ERR_DIMENSION;
            }
    }
    return NPC_SUCCESS;
}

class DfnOperator : public Operator {
  public:
    DevBuf hblk, bw, loff, L;
    DevBuf crp, cci, cv, brp, bci, bv, ghrp, ghci, ghv;
    DevBuf gurp, guci, guv, btrp, btci, btv, ctrp, ctci, ctv;
    DevBuf t, u2;
    DevBuf ainv, dense_info, band_list, perm;
    // multi-rank (the paper's DSMat partition): whole fracture blocks per
    // rank, u rows by owning fracture; per application a u-space halo of x (columns of B's E
    // part and of G^u) and an h-space halo of t (rows of B^T from other ranks' fractures)
    bool multi = false;
    int ngu = 0, ngh = 0;
    HaloPlan uplan, hplan;
    HaloRuntime urt, trt;
    // block groups in the dense / band lists: [0, cut[0]) t rows sent, no x ghost; [cut[0],
    // cut[1]) t rows sent, x ghosts read; [cut[1], n) no t row sent (single rank: all group 0)
    int dense_cut[2] = {0, 0}, band_cut[2] = {0, 0};
    DevBuf xg;  // x of the owned u rows followed by the u ghosts
    bool permuted() const override { return !multi; }
    npc_status to_internal(const double *in, double *out) override {
        return launch_gather(ctx, in, perm.as<int>(), out, n_local);
    }
    npc_status to_external(const double *in, double *out) override {
        return launch_scatter(ctx, in, perm.as<int>(), out, n_local);
    }
    int n_dense = 0, n_band = 0, dense_nt = 64, band_max_nf = 0;
    long long dense_entries = 0;
    int nblk = 0, nh = 0, max_nf = 0, max_bw = 0, lanes = 32, groups_per_cta = 8;
    double alpha = 0.0;
    long long nnz_c = 0, nnz_b = 0, nnz_gh = 0, nnz_gu = 0, band = 0;

    int num_partials() const override { return std::max(1, ceil_div(n_local, DFN_OUT_T)); }
    double bytes_per_step(bool has_s2, bool has_r) const override {
        // matrices once: Cs, Bs, their transposes, G^h, G^u (12 B/nnz + row pointers), the
        // band factor (8 B per stored entry); vectors: x (twice: block gathers + out pass),
        // t and u2 written and read, out (+ s2, r)
        // (+ the explicit inverses of the small blocks, 8 B per entry, once)
        double b = 12.0 * (2.0 * nnz_c + 2.0 * nnz_b + nnz_gh + nnz_gu) + 4.0 * (5.0 * nh + 3.0 * n_local) +
                   8.0 * band + 8.0 * dense_entries + 8.0 * (2.0 * n_local + 4.0 * nh + n_local);
        if (has_s2) b += 8.0 * n_local;
        if (has_r) b += 8.0 * n_local;
        return b;
    }
    template <int G>
    npc_status launch_block(const double *x, const int *done, int b0, int b1) {
        DfnDev D{hblk.as<int>(), bw.as<int>(), loff.as<long long>(), L.as<double>(), crp.as<int>(), cci.as<int>(),
                 cv.as<double>(), brp.as<int>(), bci.as<int>(), bv.as<double>(), ghrp.as<int>(), ghci.as<int>(),
                 ghv.as<double>(), nblk, alpha};
        const int threads = groups_per_cta * G;
        const size_t sm = sizeof(double) * 3 * (size_t)band_max_nf * groups_per_cta;
        auto kern = k_dfn_block<G>;
        if (sm > 48 * 1024) NPC_TRY(allow_max_dynamic_smem(kern));
        if (b1 <= b0) return NPC_SUCCESS;
        kern<<<ceil_div(b1 - b0, groups_per_cta), threads, sm, ctx->stream>>>(D, band_list.as<int>() + b0, b1 - b0, x,
                                                                           t.as<double>(), u2.as<double>(),
                                                                           band_max_nf, done);
        NPC_LAUNCH_CHECK();
        return NPC_SUCCESS;
    }
    template <int NT>
    npc_status launch_dense(const double *x, const int *done, int b0, int b1) {
        DfnDev D{hblk.as<int>(), bw.as<int>(), loff.as<long long>(), L.as<double>(), crp.as<int>(), cci.as<int>(),
                 cv.as<double>(), brp.as<int>(), bci.as<int>(), bv.as<double>(), ghrp.as<int>(), ghci.as<int>(),
                 ghv.as<double>(), nblk, alpha};
        if (b1 <= b0) return NPC_SUCCESS;
        k_dfn_dense<NT><<<ceil_div(b1 - b0, DFN_WARPS), 32 * DFN_WARPS, 0, ctx->stream>>>(D,
                                                                                        dense_info.as<int4>() + 2 * b0,
                                                                                        b1 - b0,
                                                                       ainv.as<double>(), x, t.as<double>(),
                                                                       u2.as<double>(), done);
        NPC_LAUNCH_CHECK();
        return NPC_SUCCESS;
    }
    template <bool H2, bool HR, bool DT>
    npc_status launch_out(const StepArgs &s) {
        DfnOutDev O{gurp.as<int>(), guci.as<int>(), guv.as<double>(), btrp.as<int>(), btci.as<int>(),
                    btv.as<double>(), ctrp.as<int>(), ctci.as<int>(), ctv.as<double>(), t.as<double>(),
                    u2.as<double>(), multi && ctx->nranks > 1 ? xg.as<double>() : s.x, alpha, n_local};
        k_dfn_out<H2, HR, DT><<<num_partials(), DFN_OUT_T, 0, ctx->stream>>>(O, s);
        NPC_LAUNCH_CHECK();
        return NPC_SUCCESS;
    }
    // the dense blocks at list positions [g0, g1) and the band blocks at [b0, b1)
    npc_status launch_blocks(const double *xin, const int *done, int g0, int g1, int b0, int b1) {
        if (dense_nt == 32) NPC_TRY(launch_dense<1>(xin, done, g0, g1));
        else if (dense_nt == 64) NPC_TRY(launch_dense<2>(xin, done, g0, g1));
        else NPC_TRY(launch_dense<4>(xin, done, g0, g1));
        if (lanes == 4) NPC_TRY(launch_block<4>(xin, done, b0, b1));
        else if (lanes == 8) NPC_TRY(launch_block<8>(xin, done, b0, b1));
        else if (lanes == 16) NPC_TRY(launch_block<16>(xin, done, b0, b1));
        else NPC_TRY(launch_block<32>(xin, done, b0, b1));
        return NPC_SUCCESS;
    }
    npc_status step(const StepArgs &s) override {
        if (n_local == 0 && !multi) return NPC_SUCCESS;
        const bool halo = multi && ctx->nranks > 1;  // a 1-rank distributed context has no ghosts
        if (!halo) {
            NPC_TRY(launch_blocks(s.x, s.done, 0, n_dense, 0, n_band));
        } else {
            // x | x ghosts in xg: the ghosts arrive while the blocks that read no x ghost (and
            // send t rows) run; then the t halo overlaps the blocks whose t stays on this rank.
            // Receive buffers are safe to overwrite: their readers precede the pack on ctx->stream.
            double *xg_ = xg.as<double>(), *t_ = t.as<double>();
            if (n_local)
                NPC_CUDA_TRY(cudaMemcpyAsync(xg_, s.x, sizeof(double) * n_local, cudaMemcpyDeviceToDevice,
                                             ctx->stream));
            NPC_TRY(halo_start(ctx, uplan, urt, s.x, xg_ + n_local));
            NPC_TRY(launch_blocks(xg_, s.done, 0, dense_cut[0], 0, band_cut[0]));
            NPC_TRY(halo_wait(ctx, urt));
            NPC_TRY(launch_blocks(xg_, s.done, dense_cut[0], dense_cut[1], band_cut[0], band_cut[1]));
            NPC_TRY(halo_start(ctx, hplan, trt, t_, t_ + nh));
            NPC_TRY(launch_blocks(xg_, s.done, dense_cut[1], n_dense, band_cut[1], n_band));
            NPC_TRY(halo_wait(ctx, trt));
            // a rank without rows writes zero dot partials (num_partials() >= 1 of them are read)
            if (n_local == 0) return s.dotv ? launch_fill(ctx, s.partials, 0.0, num_partials()) : NPC_SUCCESS;
        }
        const bool h2 = s.s2 != nullptr, hr = s.r != nullptr, dt = s.dotv != nullptr;
        if (h2 && hr && dt) return launch_out<true, true, true>(s);
        if (h2 && hr) return launch_out<true, true, false>(s);
        if (h2 && dt) return launch_out<true, false, true>(s);
        if (h2) return launch_out<true, false, false>(s);
        if (hr && dt) return launch_out<false, true, true>(s);
        if (hr) return launch_out<false, true, false>(s);
        if (dt) return launch_out<false, false, true>(s);
        return launch_out<false, false, false>(s);
    }
};

template <class T>
static npc_status upload(DevBuf &b, const T *src, size_t n) {
    NPC_TRY(b.alloc(sizeof(T) * std::max<size_t>(n, 1)));
    if (n) NPC_CUDA_TRY(cudaMemcpy(b.p, src, sizeof(T) * n, cudaMemcpyHostToDevice));
    return NPC_SUCCESS;
}

npc_status make_dfn_operator(Context *ctx, const npc_operator_desc *d0, std::unique_ptr<Operator> &out) {
    const bool multi = ctx->distributed();
    const int P = ctx->nranks, me = ctx->rank;
    // ---- partition (multi-rank): u rows [U0, U0 + n_local), h rows [H0, H0 + n^h_local) in rank
    // order; the desc's A / G^h columns are GLOBAL h ids, C / B / G^u columns GLOBAL u ids.
    std::vector<long long> u_starts{0}, h_starts{0};
    if (multi) {
        std::vector<long long> all_nu, all_nh;
        NPC_TRY(ctx->tr->allgather_i64(ctx, d0->n_local, all_nu));
        NPC_TRY(ctx->tr->allgather_i64(ctx, d0->dfn_nh, all_nh));
        for (int q = 0; q < P; ++q) {
            u_starts.push_back(u_starts.back() + all_nu[q]);
            h_starts.push_back(h_starts.back() + all_nh[q]);
        }
        if (d0->row_begin != u_starts[me] || (d0->n_global && d0->n_global != u_starts[P])) {
            set_error("DFN: row_begin / n_global disagree with the rank-ordered u partition");
            return NPC_ERR_DIMENSION;
        }
    } else {
        u_starts.push_back(d0->n_local);
        h_starts.push_back(d0->dfn_nh);
    }
    const long long U0 = u_starts[me], H0 = h_starts[me], NU = u_starts[P], NH = h_starts[P];
    npc_operator_desc dl = *d0;  // localized copy: the rest works in local ids
    const npc_operator_desc *d = &dl;
    const int nh0 = (int)std::max(0LL, std::min(d0->dfn_nh, (long long)INT32_MAX));
    std::vector<int> a_ci, gh_ci, c_ci, b_ci, gu_ci;
    HaloPlan uplan;
    std::vector<long long> b_glob;  // B column ids (global) for the multi-rank B^T exchange
    if (multi) {
        if (d0->dfn_nh < 0 || !d0->a_rowptr || !d0->gh_rowptr || !d0->c_rowptr || !d0->bm_rowptr ||
            !d0->gu_rowptr) {
            set_error("DFN: missing arrays");
            return NPC_ERR_INVALID_ARGUMENT;
        }
        NPC_TRY(check_csr("A", nh0, (int)std::min(NH, (long long)INT32_MAX), d0->a_rowptr, d0->a_colidx, d0->a_vals));
        NPC_TRY(check_csr("G^h", nh0, (int)std::min(NH, (long long)INT32_MAX), d0->gh_rowptr, d0->gh_colidx,
                          d0->gh_vals));
        NPC_TRY(check_csr("C", nh0, (int)NU, d0->c_rowptr, d0->c_colidx, d0->c_vals));
        NPC_TRY(check_csr("B", nh0, (int)NU, d0->bm_rowptr, d0->bm_colidx, d0->bm_vals));
        NPC_TRY(check_csr("G^u", d0->n_local, (int)NU, d0->gu_rowptr, d0->gu_colidx, d0->gu_vals));
        auto shift = [&](const int *rp, const int *ci, int nrows, long long base, std::vector<int> &o) {
            o.assign(ci, ci + rp[nrows]);
            for (int &c : o) c = (int)(c - base);  // block checks below reject foreign columns
        };
        shift(d0->a_rowptr, d0->a_colidx, nh0, H0, a_ci);
        shift(d0->gh_rowptr, d0->gh_colidx, nh0, H0, gh_ci);
        c_ci.assign(d0->c_colidx, d0->c_colidx + d0->c_rowptr[nh0]);
        for (int &c : c_ci) {
            if (c < U0 || c >= U0 + d0->n_local) {
                set_error("DFN: rank %d: column %d of C is not an owned u row (the u partition must follow "
                          "fracture ownership: C is fracture-local)", me, c);
                return NPC_ERR_UNSUPPORTED;
            }
            c = (int)(c - U0);
        }
        std::vector<long long> ids;
        for (int p = 0; p < d0->bm_rowptr[nh0]; ++p) ids.push_back(d0->bm_colidx[p]);
        for (int p = 0; p < d0->gu_rowptr[d0->n_local]; ++p) ids.push_back(d0->gu_colidx[p]);
        b_glob.assign(d0->bm_colidx, d0->bm_colidx + d0->bm_rowptr[nh0]);
        NPC_TRY(halo_plan_from_ids(ids, P, u_starts.data(), me, uplan));
        NPC_TRY(halo_plan_exchange(ctx, U0, uplan));
        auto uloc = [&](long long c) -> int {
            if (c >= U0 && c < U0 + d0->n_local) return (int)(c - U0);
            return d0->n_local +
                   (int)(std::lower_bound(uplan.ghost_ids.begin(), uplan.ghost_ids.end(), c) - uplan.ghost_ids.begin());
        };
        b_ci.resize(d0->bm_rowptr[nh0]);
        for (int p = 0; p < d0->bm_rowptr[nh0]; ++p) b_ci[p] = uloc(d0->bm_colidx[p]);
        gu_ci.resize(d0->gu_rowptr[d0->n_local]);
        for (int p = 0; p < d0->gu_rowptr[d0->n_local]; ++p) gu_ci[p] = uloc(d0->gu_colidx[p]);
        dl.a_colidx = a_ci.data();
        dl.gh_colidx = gh_ci.data();
        dl.c_colidx = c_ci.data();
        dl.bm_colidx = b_ci.data();
        dl.gu_colidx = gu_ci.data();
    }
    const int ngu = multi ? uplan.n_ghost : 0;
    const int nu = d->n_local, nblk = d->dfn_nblk;
    const long long nhl = d->dfn_nh;
    if (nhl < 0 || nhl >= (1LL << 31) || nblk < 0 || (nblk > 0 && !d->dfn_hblk) || !(std::isfinite(d->dfn_alpha))) {
        set_error("DFN: invalid sizes / alpha");
        return NPC_ERR_INVALID_ARGUMENT;
    }
    const int nh = (int)nhl;
    const int *hb = d->dfn_hblk;
    if (nblk > 0 && (hb[0] != 0 || hb[nblk] != nh)) {
        set_error("DFN: block offsets must run from 0 to n^h");
        return NPC_ERR_DIMENSION;
    }
    if (nblk == 0 && nh != 0) {
        set_error("DFN: n^h > 0 needs at least one block");
        return NPC_ERR_DIMENSION;
    }
    NPC_TRY(check_csr("A", nh, nh, d->a_rowptr, d->a_colidx, d->a_vals));
    NPC_TRY(check_csr("G^h", nh, nh, d->gh_rowptr, d->gh_colidx, d->gh_vals));
    NPC_TRY(check_csr("C", nh, nu, d->c_rowptr, d->c_colidx, d->c_vals));
    NPC_TRY(check_csr("B", nh, nu + ngu, d->bm_rowptr, d->bm_colidx, d->bm_vals));
    NPC_TRY(check_csr("G^u", nu, nu + ngu, d->gu_rowptr, d->gu_colidx, d->gu_vals));
    auto op = std::make_unique<DfnOperator>();
    op->ctx = ctx;
    op->kind = NPC_OP_DFN;
    op->n_local = nu;
    op->n_global = multi ? NU : nu;
    op->row_begin = U0;
    op->multi = multi;
    op->ngu = ngu;
    op->nblk = nblk;
    op->nh = nh;
    op->alpha = d->dfn_alpha;
    // ---- per-block bandwidth (A and G^h must be block-diagonal), banded Cholesky of A
    std::vector<int> bwv(std::max(nblk, 1), 0);
    std::vector<long long> loffv(std::max(nblk, 1), 0);
    long long band = 0;
    for (int f = 0; f < nblk; ++f) {
        const int h0 = hb[f], h1 = hb[f + 1];
        if (h1 < h0) {
            set_error("DFN: block offsets decrease at block %d", f);
            return NPC_ERR_DIMENSION;
        }
        op->max_nf = std::max(op->max_nf, h1 - h0);
        int w = 0;
        for (int i = h0; i < h1; ++i) {
            for (int p = d->a_rowptr[i]; p < d->a_rowptr[i + 1]; ++p) {
                const int j = d->a_colidx[p];
                if (j < h0 || j >= h1) {
                    set_error("DFN: A is not block-diagonal (row %d, column %d)", i, j);
                    return NPC_ERR_DIMENSION;
                }
                w = std::max(w, std::abs(i - j));
            }
            for (int p = d->gh_rowptr[i]; p < d->gh_rowptr[i + 1]; ++p)
                if (d->gh_colidx[p] < h0 || d->gh_colidx[p] >= h1) {
                    set_error("DFN: G^h is not block-diagonal (row %d)", i);
                    return NPC_ERR_DIMENSION;
                }
        }
        bwv[f] = w;
        op->max_bw = std::max(op->max_bw, w);
        loffv[f] = band;
        band += (long long)(h1 - h0) * (w + 1);
    }
    if (op->max_nf > DFN_MAX_NF) {
        set_error("DFN: a fracture block has %d > %d rows", op->max_nf, DFN_MAX_NF);
        return NPC_ERR_UNSUPPORTED;
    }
    std::vector<double> Lh((size_t)std::max(band, 1LL), 0.0);
    for (int f = 0; f < nblk; ++f) {
        const int h0 = hb[f], m = hb[f + 1] - h0, w = bwv[f], ld = w + 1;
        double *Lf = Lh.data() + loffv[f];
        for (int i = 0; i < m; ++i)
            for (int p = d->a_rowptr[h0 + i]; p < d->a_rowptr[h0 + i + 1]; ++p) {
                const int j = d->a_colidx[p] - h0;
                if (j <= i) Lf[(size_t)i * ld + w - (i - j)] += d->a_vals[p];  // lower triangle of A_f
            }
        for (int i = 0; i < m; ++i)
            for (int j = std::max(0, i - w); j <= i; ++j) {
                double sacc = Lf[(size_t)i * ld + w - (i - j)];
                for (int k = std::max(std::max(0, i - w), j - w); k < j; ++k)
                    sacc -= Lf[(size_t)i * ld + w - (i - k)] * Lf[(size_t)j * ld + w - (j - k)];
                if (i == j) {
                    if (!(sacc > 0.0)) {
                        set_error("DFN: block %d of A is not SPD (pivot %d)", f, i);
                        return NPC_ERR_DIMENSION;
                    }
                    Lf[(size_t)i * ld + w] = std::sqrt(sacc);
                } else {
                    Lf[(size_t)i * ld + w - (i - j)] = sacc / Lf[(size_t)j * ld + w];
                }
            }
    }
    // ---- D_S = diag(S_u) by Alg. 4 (with alpha), one column of C at a time, host threads
    std::vector<double> dscale(std::max(nu, 1), 1.0);
    const int *brp = d->bm_rowptr, *bci = d->bm_colidx;
    const double *bvals = d->bm_vals;
    if (d->dfn_scaled) {
        HostCsr CT = transpose(nh, nu, d->c_rowptr, d->c_colidx, d->c_vals);
        HostCsr BT = transpose(nh, nu + ngu, brp, bci, bvals);  // ghost columns are never visited
        std::vector<int> blk_of(std::max(nh, 1));
        for (int f = 0; f < nblk; ++f)
            for (int i = hb[f]; i < hb[f + 1]; ++i) blk_of[i] = f;
        std::vector<double> ds(nu);
        const int nth = std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
        std::vector<std::thread> th;
        std::vector<int> bad(nth, -1);
        for (int tid = 0; tid < nth; ++tid)
            th.emplace_back([&, tid]() {
                std::vector<double> z(op->max_nf + 1), gz(op->max_nf + 1);
                for (int c = tid; c < nu; c += nth) {
                    double gii = 0.0;
                    for (int p = d->gu_rowptr[c]; p < d->gu_rowptr[c + 1]; ++p)
                        if (d->gu_colidx[p] == c) gii += d->gu_vals[p];
                    double acc = gii;
                    int p = CT.rp[c];
                    while (p < CT.rp[c + 1]) {  // blocks touched by column c of C (rows ascending)
                        const int f = blk_of[CT.ci[p]];
                        const int h0 = hb[f], m = hb[f + 1] - h0, w = bwv[f], ld = w + 1;
                        const double *Lf = Lh.data() + loffv[f];
                        std::fill(z.begin(), z.begin() + m, 0.0);
                        for (; p < CT.rp[c + 1] && CT.ci[p] < hb[f + 1]; ++p) z[CT.ci[p] - h0] = CT.v[p];
                        for (int i = 0; i < m; ++i) {  // z = A_f^-1 c (banded forward/backward)
                            double sacc = z[i];
                            for (int k = std::max(0, i - w); k < i; ++k) sacc -= Lf[(size_t)i * ld + w - (i - k)] * z[k];
                            z[i] = sacc / Lf[(size_t)i * ld + w];
                        }
                        for (int i = m - 1; i >= 0; --i) {
                            double sacc = z[i];
                            for (int k = i + 1; k <= std::min(m - 1, i + w); ++k)
                                sacc -= Lf[(size_t)k * ld + w - (k - i)] * z[k];
                            z[i] = sacc / Lf[(size_t)i * ld + w];
                        }
                        for (int i = 0; i < m; ++i) {  // z^T G^h z on the block
                            double sacc = 0.0;
                            for (int q = d->gh_rowptr[h0 + i]; q < d->gh_rowptr[h0 + i + 1]; ++q)
                                sacc += d->gh_vals[q] * z[d->gh_colidx[q] - h0];
                            gz[i] = sacc;
                            acc += z[i] * gz[i];
                        }
                        for (int q = BT.rp[c]; q < BT.rp[c + 1]; ++q)  // - 2 a z^T b_c on the block
                            if (BT.ci[q] >= h0 && BT.ci[q] < hb[f + 1]) acc -= 2.0 * d->dfn_alpha * z[BT.ci[q] - h0] * BT.v[q];
                    }
                    ds[c] = acc;
                    if (!(acc > 0.0) && bad[tid] < 0) bad[tid] = c;
                }
            });
        for (auto &t_ : th) t_.join();
        for (int b_ : bad)
            if (b_ >= 0) {
                set_error("DFN: diag(S_u) entry %d is not positive (S_u not SPD for this alpha)", b_);
                return NPC_ERR_DIMENSION;
            }
        for (int c = 0; c < nu; ++c) dscale[c] = 1.0 / std::sqrt(ds[c]);
    }
    // ---- multi-rank: D_S^{-1/2} of the ghost u columns (B's E part, G^u) from their owners
    dscale.resize(std::max(nu + ngu, 1), 1.0);
    if (multi) {
        op->uplan = uplan;
        NPC_TRY(halo_setup(ctx, op->uplan, op->urt));
        if (d->dfn_scaled) {
            DevBuf dd;
            NPC_TRY(dd.alloc(sizeof(double) * std::max(nu, 1)));
            if (nu) NPC_CUDA_TRY(cudaMemcpy(dd.p, dscale.data(), sizeof(double) * nu, cudaMemcpyHostToDevice));
            NPC_TRY(halo_start(ctx, op->uplan, op->urt, dd.as<double>()));
            NPC_TRY(halo_wait(ctx, op->urt));
            NPC_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
            if (ngu)
                NPC_CUDA_TRY(cudaMemcpy(dscale.data() + nu, op->urt.ghost_buf.p, sizeof(double) * ngu,
                                        cudaMemcpyDeviceToHost));
        }
    }
    // ---- internal order of the u unknowns: grouped by the fracture block that owns them (the
    // block of the first row of their column of C), stable.  A symmetric permutation (PCG and
    // p_k are unchanged; vectors are permuted once on entry/exit): the C part of a block's rows
    // then gathers a contiguous range of x, and consecutive u rows of the output pass gather t
    // and u2 from the same fracture -- the random L2 gathers bound both kernels.
    std::vector<int> perm(std::max(nu, 1)), inv(std::max(nu + ngu, 1));
    for (int i = 0; i < nu + ngu; ++i) inv[i] = i;  // ghosts keep their slots
    if (!multi) {  // multi-rank: the caller's order (halos index owned rows directly)
        std::vector<int> own(std::max(nu, 1), nblk);
        std::vector<int> blk_of(std::max(nh, 1), 0);
        for (int f = 0; f < nblk; ++f)
            for (int i = hb[f]; i < hb[f + 1]; ++i) blk_of[i] = f;
        for (int i = nh - 1; i >= 0; --i)  // rows descending: the smallest row wins
            for (int p = d->c_rowptr[i]; p < d->c_rowptr[i + 1]; ++p) own[d->c_colidx[p]] = blk_of[i];
        for (int i = 0; i < nu; ++i) perm[i] = i;
        std::stable_sort(perm.begin(), perm.begin() + nu, [&](int a, int b) { return own[a] < own[b]; });
        for (int i = 0; i < nu; ++i) inv[perm[i]] = i;
    } else {
        for (int i = 0; i < nu; ++i) perm[i] = i;
    }
    // ---- scaled matrices, u columns / rows renumbered to the internal order
    std::vector<double> cs(d->c_vals, d->c_vals + d->c_rowptr[nh]), bs(bvals, bvals + brp[nh]);
    std::vector<int> cci_i(d->c_colidx, d->c_colidx + d->c_rowptr[nh]), bci_i(bci, bci + brp[nh]);
    for (int p = 0; p < d->c_rowptr[nh]; ++p) {
        cs[p] *= dscale[cci_i[p]];
        cci_i[p] = inv[cci_i[p]];
    }
    for (int p = 0; p < brp[nh]; ++p) {
        bs[p] *= dscale[bci_i[p]];
        bci_i[p] = inv[bci_i[p]];
    }
    std::vector<int> gurp_i(nu + 1, 0), guci_i(std::max(d->gu_rowptr[nu], 1));
    std::vector<double> gus(std::max(d->gu_rowptr[nu], 1));
    for (int i = 0; i < nu; ++i) {
        const int o = perm[i];
        gurp_i[i + 1] = gurp_i[i] + d->gu_rowptr[o + 1] - d->gu_rowptr[o];
        int q = gurp_i[i];
        for (int p = d->gu_rowptr[o]; p < d->gu_rowptr[o + 1]; ++p, ++q) {
            guci_i[q] = inv[d->gu_colidx[p]];
            gus[q] = d->gu_vals[p] * dscale[o] * dscale[d->gu_colidx[p]];
        }
    }
    HostCsr CsT = transpose(nh, nu, d->c_rowptr, cci_i.data(), cs.data());
    HostCsr BsT;
    if (!multi) {
        BsT = transpose(nh, nu, brp, bci_i.data(), bs.data());
    } else {
        // rows of B^T for the owned u columns: the owned B rows' entries plus the entries other
        // ranks' fractures hold for these columns (B's E part), exchanged once at setup as
        // (u global, h global, value bits) triples; then an h-space halo plan for t and u2
        std::vector<std::vector<long long>> out_t(P);
        std::vector<std::vector<std::pair<long long, double>>> rows(nu);
        for (int h = 0; h < nh; ++h)
            for (int q = brp[h]; q < brp[h + 1]; ++q) {
                const long long cg = b_glob[q];
                if (cg >= U0 && cg < U0 + nu) {
                    rows[cg - U0].push_back({H0 + h, bs[q]});
                } else {
                    const int owner = (int)(std::upper_bound(u_starts.begin(), u_starts.end(), cg) - u_starts.begin()) - 1;
                    long long bits;
                    memcpy(&bits, &bs[q], 8);
                    out_t[owner].insert(out_t[owner].end(), {cg, H0 + h, bits});
                }
            }
        std::vector<int> scount(P), soff(P, 0), all;
        for (int q = 0; q < P; ++q) scount[q] = (int)out_t[q].size();
        for (int q = 1; q < P; ++q) soff[q] = soff[q - 1] + scount[q - 1];
        NPC_TRY(ctx->tr->allgather_i32v(ctx, scount, all));
        std::vector<int> rcount(P), roff(P, 0);
        for (int q = 0; q < P; ++q) rcount[q] = all[(size_t)q * P + me];
        for (int q = 1; q < P; ++q) roff[q] = roff[q - 1] + rcount[q - 1];
        std::vector<long long> sbuf, rbuf((size_t)roff[P - 1] + rcount[P - 1]);
        for (int q = 0; q < P; ++q) sbuf.insert(sbuf.end(), out_t[q].begin(), out_t[q].end());
        rcount[me] = 0;  // nothing to myself
        NPC_TRY(ctx->tr->alltoallv_i64(ctx, sbuf, scount, soff, rbuf, rcount, roff));
        for (size_t e = 0; e + 2 < rbuf.size(); e += 3) {
            double v;
            memcpy(&v, &rbuf[e + 2], 8);
            const long long cg = rbuf[e];
            if (cg < U0 || cg >= U0 + nu) {
                set_error("DFN: received a B^T entry for u row %lld not owned here", cg);
                return NPC_ERR_DIMENSION;
            }
            rows[cg - U0].push_back({rbuf[e + 1], v});
        }
        std::vector<long long> hids;
        for (auto &r : rows) {
            std::sort(r.begin(), r.end());  // ascending global h: the same order on any partition
            for (auto &e : r) hids.push_back(e.first);
        }
        NPC_TRY(halo_plan_from_ids(hids, P, h_starts.data(), me, op->hplan));
        NPC_TRY(halo_plan_exchange(ctx, H0, op->hplan));
        op->ngh = op->hplan.n_ghost;
        const auto &gh = op->hplan.ghost_ids;
        BsT.rp.assign(nu + 1, 0);
        for (int c = 0; c < nu; ++c) {
            BsT.rp[c + 1] = BsT.rp[c] + (int)rows[c].size();
            for (auto &e : rows[c]) {
                const long long hg = e.first;
                BsT.ci.push_back(hg >= H0 && hg < H0 + nh
                                     ? (int)(hg - H0)
                                     : nh + (int)(std::lower_bound(gh.begin(), gh.end(), hg) - gh.begin()));
                BsT.v.push_back(e.second);
            }
        }
        if (BsT.ci.empty()) {
            BsT.ci.push_back(0);
            BsT.v.push_back(0.0);
        }
        NPC_TRY(halo_setup(ctx, op->hplan, op->trt));
        NPC_TRY(op->xg.alloc(sizeof(double) * std::max(nu + ngu, 1)));
    }
    op->nnz_c = d->c_rowptr[nh];
    op->nnz_b = multi ? BsT.rp[nu] : brp[nh];
    op->nnz_gh = d->gh_rowptr[nh];
    op->nnz_gu = d->gu_rowptr[nu];
    // ---- small blocks: explicit inverse A_f^-1 = L^-T L^-1 (column j = banded solve of e_j),
    // symmetrised; large blocks keep the band factor
    std::vector<int> dlist, blist;
    std::vector<long long> doffv(std::max(nblk, 1), 0);
    long long dtot = 0;
    int dense_max_m = 0, band_max_bw = 0;
    for (int f = 0; f < nblk; ++f) {
        const int m = hb[f + 1] - hb[f];
        if (m <= DFN_DENSE_MAX) {
            dlist.push_back(f);
            doffv[f] = dtot;
            dtot += ((long long)m * m + 1) & ~1LL;  // 16 B aligned blocks
            dense_max_m = std::max(dense_max_m, m);
        } else {
            blist.push_back(f);
            op->band_max_nf = std::max(op->band_max_nf, m);
            band_max_bw = std::max(band_max_bw, bwv[f]);
        }
    }
    if (multi) {  // group order (see dense_cut): a stable partition of each list
        std::vector<char> snd_h(std::max(nh, 1), 0);
        for (int h : op->hplan.send_idx) snd_h[h] = 1;
        auto group = [&](int f) {
            bool snd = false, ng = false;
            for (int h = hb[f]; h < hb[f + 1]; ++h) {
                snd = snd || snd_h[h];
                for (int p = brp[h]; p < brp[h + 1] && !ng; ++p) ng = bci_i[p] >= nu;
            }
            return snd ? (ng ? 1 : 0) : 2;
        };
        auto partition = [&](std::vector<int> &lst, int *cut) {
            std::vector<int> g(lst.size()), o;
            for (size_t q = 0; q < lst.size(); ++q) g[q] = group(lst[q]);
            for (int k = 0; k < 3; ++k) {
                for (size_t q = 0; q < lst.size(); ++q)
                    if (g[q] == k) o.push_back(lst[q]);
                if (k < 2) cut[k] = (int)o.size();
            }
            lst.swap(o);
        };
        partition(dlist, op->dense_cut);
        partition(blist, op->band_cut);
    } else {
        op->dense_cut[0] = op->dense_cut[1] = (int)dlist.size();
        op->band_cut[0] = op->band_cut[1] = (int)blist.size();
    }
    std::vector<double> ainvh((size_t)std::max(dtot, 1LL), 0.0);
    {
        const int nth = std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
        std::vector<std::thread> th;
        for (int tid = 0; tid < nth; ++tid)
            th.emplace_back([&, tid]() {
                std::vector<double> col(DFN_DENSE_MAX);
                for (size_t q = tid; q < dlist.size(); q += nth) {
                    const int f = dlist[q], m = hb[f + 1] - hb[f], w = bwv[f], ld = w + 1;
                    const double *Lf = Lh.data() + loffv[f];
                    double *X = ainvh.data() + doffv[f];
                    for (int j = 0; j < m; ++j) {
                        std::fill(col.begin(), col.begin() + m, 0.0);
                        col[j] = 1.0;
                        for (int i = 0; i < m; ++i) {
                            double sacc = col[i];
                            for (int k = std::max(0, i - w); k < i; ++k) sacc -= Lf[(size_t)i * ld + w - (i - k)] * col[k];
                            col[i] = sacc / Lf[(size_t)i * ld + w];
                        }
                        for (int i = m - 1; i >= 0; --i) {
                            double sacc = col[i];
                            for (int k = i + 1; k <= std::min(m - 1, i + w); ++k)
                                sacc -= Lf[(size_t)k * ld + w - (k - i)] * col[k];
                            col[i] = sacc / Lf[(size_t)i * ld + w];
                        }
                        for (int i = 0; i < m; ++i) X[(size_t)i * m + j] = col[i];
                    }
                    for (int i = 0; i < m; ++i)
                        for (int j = 0; j < i; ++j) {
                            const double a = 0.5 * (X[(size_t)i * m + j] + X[(size_t)j * m + i]);
                            X[(size_t)i * m + j] = X[(size_t)j * m + i] = a;
                        }
                }
            });
        for (auto &t_ : th) t_.join();
    }
    op->n_dense = (int)dlist.size();
    op->n_band = (int)blist.size();
    op->dense_entries = dtot;
    op->dense_nt = dense_max_m <= 32 ? 32 : dense_max_m <= 64 ? 64 : 128;
    op->band = 0;
    for (int f : blist) op->band += (long long)(hb[f + 1] - hb[f]) * (bwv[f] + 1);
    // ---- lanes per band-block group: the smallest power of two >= the largest band (>= 4)
    op->lanes = band_max_bw <= 4 ? 4 : band_max_bw <= 8 ? 8 : band_max_bw <= 16 ? 16 : 32;
    const size_t per_group = sizeof(double) * 3 * (size_t)std::max(op->band_max_nf, 1);
    op->groups_per_cta = (int)std::max<size_t>(1, std::min<size_t>(256 / op->lanes, (200 * 1024) / per_group));
    // ---- upload
    std::vector<int> hbv(hb, hb + nblk + 1);
    if (nblk == 0) hbv.assign(1, 0);
    NPC_TRY(upload(op->hblk, hbv.data(), hbv.size()));
    NPC_TRY(upload(op->bw, bwv.data(), bwv.size()));
    NPC_TRY(upload(op->loff, loffv.data(), loffv.size()));
    NPC_TRY(upload(op->L, Lh.data(), Lh.size()));
    NPC_TRY(upload(op->crp, d->c_rowptr, (size_t)nh + 1));
    NPC_TRY(upload(op->cci, cci_i.data(), (size_t)d->c_rowptr[nh]));
    NPC_TRY(upload(op->cv, cs.data(), cs.size()));
    NPC_TRY(upload(op->brp, brp, (size_t)nh + 1));
    NPC_TRY(upload(op->bci, bci_i.data(), (size_t)brp[nh]));
    NPC_TRY(upload(op->bv, bs.data(), bs.size()));
    NPC_TRY(upload(op->ghrp, d->gh_rowptr, (size_t)nh + 1));
    NPC_TRY(upload(op->ghci, d->gh_colidx, (size_t)d->gh_rowptr[nh]));
    NPC_TRY(upload(op->ghv, d->gh_vals, (size_t)d->gh_rowptr[nh]));
    NPC_TRY(upload(op->gurp, gurp_i.data(), (size_t)nu + 1));
    NPC_TRY(upload(op->guci, guci_i.data(), (size_t)d->gu_rowptr[nu]));
    NPC_TRY(upload(op->perm, perm.data(), (size_t)nu));
    NPC_TRY(upload(op->guv, gus.data(), gus.size()));
    NPC_TRY(upload(op->btrp, BsT.rp.data(), BsT.rp.size()));
    NPC_TRY(upload(op->btci, BsT.ci.data(), (size_t)BsT.rp[nu]));
    NPC_TRY(upload(op->btv, BsT.v.data(), (size_t)BsT.rp[nu]));
    NPC_TRY(upload(op->ctrp, CsT.rp.data(), CsT.rp.size()));
    NPC_TRY(upload(op->ctci, CsT.ci.data(), (size_t)d->c_rowptr[nh]));
    NPC_TRY(upload(op->ctv, CsT.v.data(), (size_t)d->c_rowptr[nh]));
    NPC_TRY(upload(op->ainv, ainvh.data(), ainvh.size()));
    std::vector<int> dinfo(8 * std::max<size_t>(dlist.size(), 1), 0);  // two int4 per dense block
    for (size_t q = 0; q < dlist.size(); ++q) {
        const int f = dlist[q], h0 = hb[f], h1 = hb[f + 1];
        int *e = dinfo.data() + 8 * q;
        e[0] = h0;
        e[1] = h1 - h0;
        e[2] = (int)(unsigned)(doffv[f] & 0xffffffffLL);
        e[3] = (int)(unsigned)(doffv[f] >> 32);
        e[4] = d->c_rowptr[h0];
        e[5] = d->c_rowptr[h1];
        e[6] = brp[h0];
        e[7] = brp[h1];
    }
    NPC_TRY(upload(op->dense_info, dinfo.data(), dinfo.size()));
    NPC_TRY(upload(op->band_list, blist.data(), blist.size()));
    NPC_TRY(op->t.alloc(sizeof(double) * std::max(nh + op->ngh, 1)));   // owned h rows + h ghosts
    NPC_TRY(op->u2.alloc(sizeof(double) * std::max(nh, 1)));  // read by C^T only: fracture-local
    out = std::move(op);
    return NPC_SUCCESS;
}

}  // namespace npc
