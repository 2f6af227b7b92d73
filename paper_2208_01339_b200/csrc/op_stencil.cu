// op_stencil.cu -- matrix-free constant-coefficient 2D 5-point / 3D 7-point Dirichlet
// operator (BASELINE config 2) with the Chebyshev recurrence fused in.
//
// "only the application of the matrix to a vector is available as a routine (matrix-free
// regime)".  Kernel: 32x8 threads own an (x, y) tile and march along z,
// keeping x[z-1], x[z], x[z+1] in registers (2.5D blocking) so each plane of the input is
// read from L2/HBM once; the in-plane neighbours come from L1.  Epilogue as in op_csr.cu.
// Default for even nx: the 128-bit form k_stencil_step_v2 (two x-points per thread, every
// stream as double2); grids whose vectors exceed L2 take the TMA-staged kernel k_stencil_tma.
// Multi-rank: z-slabs; ghost planes z_begin-1 and z_end arrive through the generic halo
// (planes are contiguous row ranges), overlapped with the interior planes.
#include <algorithm>
#include <map>

#include <cooperative_groups.h>
#include <cuda.h>
#include <cudaTypedefs.h>

#include "device_util.cuh"
#include "npc_internal.cuh"

namespace npc {

namespace cg = cooperative_groups;

static constexpr int ST_BX = 32, ST_BY = 8, ST_ZC = 8;

// The fused epilogue's arithmetic, spelled out as explicit FMAs so that every stencil kernel
// (register, TMA, one- and two-degree) rounds identically whatever the compiler would contract:
//   A x = diag x_i + off (sum of neighbours);  out = a (A x) + b x  [+ c s_{j-2}] [+ d r]
__device__ __forceinline__ double st_ax(double diag, double x, double off, double nb) {
    return __fma_rn(diag, x, off * nb);
}
__device__ __forceinline__ double st_lin(double a, double ax, double b, double x) {
    return __fma_rn(a, ax, b * x);
}



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
            const double ax = st_ax(S.diag, cur, S.off, nb);
            double o = st_lin(s.a, ax, s.b, cur);
            if (HAS_S2) o = __fma_rn(s.c, s.s2[i], o);
            if (HAS_R) o = __fma_rn(s.d, s.r[i], o);
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

// ---------------------------------------------------------------- two x-points per thread
// k_stencil_step with 128-bit accesses: a thread owns the points (x0, x0 + 1), x0 even, of its
// row and marches z as above, so every stream (s_{j-1} planes, the y neighbours, s_{j-2}, r,
// the store) moves as double2 and the kernel issues 7 loads + 1 store per TWO points instead of
// per point (config 2 is latency / LSU-issue bound, not bandwidth bound: profiles/
// r02_ncu_summary.md).  A CTA is 16 x 8 threads on the SAME 32 x 8 point tile and grid as
// k_stencil_step (same partial slots).  The neighbour sum keeps k_stencil_step's order
// (z-1, y-1, x-1, x+1, y+1, z+1) and explicit FMAs, so out is bitwise the same.  Needs an even
// nx and 16-byte aligned vectors (checked at dispatch).
static constexpr int SV_BX = ST_BX / 2;
template <int DIM, bool HAS_S2, bool HAS_R, bool DOT>
__global__ void __launch_bounds__(SV_BX *ST_BY) k_stencil_step_v2(StencilDev S, StepArgs s, int z_lo, int z_hi, int zc) {
    // (Programmatic dependent launch -- griddepcontrol.launch_dependents / .wait here and the
    // stream-serialization launch attribute -- was measured and removed: config 2 p_30 0.278 vs
    // 0.270 ms, PCG 9.3 vs 8.3 ms, and the two instructions alone cost an ordinary launch 9 %:
    // profiles/r02_stencil_vec2_ab.md.)
    if (s.done && *s.done) return;
    __shared__ double red[SV_BX * ST_BY / 32];
    const int x0 = blockIdx.x * ST_BX + 2 * threadIdx.x;
    const int y = blockIdx.y * ST_BY + threadIdx.y;
    const int z0 = z_lo + blockIdx.z * zc;
    const int z1 = min(z0 + zc, z_hi);
    const long long plane = (long long)S.nx * S.ny;
    const double *__restrict__ X = s.x;
    double acc = 0.0;
    if (x0 < S.nx && y < S.ny && z0 < z1) {
        const int pidx = x0 + S.nx * y;
        long long i = pidx + plane * z0;
        const bool has_l = x0 > 0, has_r = x0 + 2 < S.nx, has_d = y > 0, has_u = y < S.ny - 1;
        double2 below = make_double2(0.0, 0.0), cur = *reinterpret_cast<const double2 *>(X + i);
        if (DIM == 3) {
            if (z0 > 0)
                below = *reinterpret_cast<const double2 *>(X + i - plane);
            else if (S.glo)
                below = *reinterpret_cast<const double2 *>(S.glo + pidx);
        }
        for (int z = z0; z < z1; ++z, i += plane) {
            double2 above = make_double2(0.0, 0.0);
            if (DIM == 3) {
                if (z + 1 < S.nzl)
                    above = *reinterpret_cast<const double2 *>(X + i + plane);
                else if (S.ghi)
                    above = *reinterpret_cast<const double2 *>(S.ghi + pidx);
            }
            double na = below.x, nb = below.y;
            if (has_d) {
                const double2 t = *reinterpret_cast<const double2 *>(X + i - S.nx);
                na += t.x;
                nb += t.y;
            }
            if (has_l) na += X[i - 1];
            nb += cur.x;
            na += cur.y;
            if (has_r) nb += X[i + 2];
            if (has_u) {
                const double2 t = *reinterpret_cast<const double2 *>(X + i + S.nx);
                na += t.x;
                nb += t.y;
            }
            na += above.x;
            nb += above.y;
            double2 o;
            o.x = st_lin(s.a, st_ax(S.diag, cur.x, S.off, na), s.b, cur.x);
            o.y = st_lin(s.a, st_ax(S.diag, cur.y, S.off, nb), s.b, cur.y);
            if (HAS_S2) {
                const double2 t = *reinterpret_cast<const double2 *>(s.s2 + i);
                o.x = __fma_rn(s.c, t.x, o.x);
                o.y = __fma_rn(s.c, t.y, o.y);
            }
            if (HAS_R) {
                const double2 t = *reinterpret_cast<const double2 *>(s.r + i);
                o.x = __fma_rn(s.d, t.x, o.x);
                o.y = __fma_rn(s.d, t.y, o.y);
            }
            *reinterpret_cast<double2 *>(s.out + i) = o;
            if (DOT) {
                const double2 t = *reinterpret_cast<const double2 *>(s.dotv + i);
                acc += o.x * t.x;
                acc += o.y * t.y;
            }
            below = cur;
            cur = above;
        }
    }
    if (DOT) {
        acc = block_sum<SV_BX * ST_BY>(acc, red);
        if (threadIdx.x == 0 && threadIdx.y == 0) s.partials[linear_bid()] = acc;
    }
}

// ---------------------------------------------------------------- all k degrees in one launch
// For grids whose vectors sit in L2 (config 2: 4 x 16.8 MB), a degree takes ~10 us and kernel
// boundaries (launch gap, ramp-up, tail) are a large part of it.  This cooperative kernel runs
// every degree of p_k(A) r with a grid-wide barrier between degrees instead of a kernel
// boundary: each CTA takes (x, y, z-chunk) items of k_stencil_step's decomposition and marches
// them with the same arithmetic (same neighbour order, same explicit FMAs), so s_k is bitwise
// equal to k launches of k_stencil_step.  s_j is written over s_{j-2} (the same element, read
// first by the same thread); the barrier after degree j makes s_j visible before any CTA
// gathers it and frees s_{j-1} for s_{j+1}.  Coefficients as the per-degree path
// (solvers.cu: j = 1 folds s_0 = r / theta_bar, j = 2 its c_2 s_0 term).  The <r_or_dotv, z>
// partial of the last degree goes to partials[blockIdx.x] (nparts = grid).
#ifndef NPC_GRID_MINB
#define NPC_GRID_MINB 4  // A/B (config 2): 4 CTAs per SM (62 registers, no spill); 6 or 8 spill and run 1.8x slower
#endif
// V2: two x-points per thread with 128-bit accesses, as k_stencil_step_v2 (a CTA is 16 x 8
// threads on the same 32 x 8 tile, twice as many CTAs per SM at the same register cap); needs an
// even nx and 16-byte aligned vectors.  Same element arithmetic, so s_k is bitwise the same.
#ifndef NPC_GRID_MINB_V2
#define NPC_GRID_MINB_V2 4  // A/B (config 2 p_30): 4 CTAs of 128 threads per SM 0.257 ms, 6 0.265, 8 (64 registers) 0.294
#endif
template <int DIM, bool V2>
__global__ void __launch_bounds__((V2 ? SV_BX : ST_BX) * ST_BY, V2 ? NPC_GRID_MINB_V2 : NPC_GRID_MINB)
    k_stencil_poly_grid(StencilDev S, const double *__restrict__ r, double *z, double *tmp,
                        const double *__restrict__ coef, int k, double tb, int zc, const double *__restrict__ dotv,
                        double *partials, const int *done) {
    if (done && *done) return;  // uniform over the grid (no kernel writes the flag meanwhile)
    cg::grid_group grid = cg::this_grid();
    __shared__ double red[ST_BX * ST_BY / 32];
    const int gx = (S.nx + ST_BX - 1) / ST_BX, gy = (S.ny + ST_BY - 1) / ST_BY;
    const int gz = DIM == 3 ? (S.nzl + zc - 1) / zc : 1;
    const int items = gx * gy * gz;
    const long long plane = (long long)S.nx * S.ny;
    double acc = 0.0;
    for (int j = 1; j <= k; ++j) {
        const double *cf = coef + 4 * (j - 1);
        double a, b, c = 0.0, d = 0.0;
        double *out = ((k - j) & 1) ? tmp : z;  // s_k lands in z
        const double *X = j == 1 ? r : (((k - j + 1) & 1) ? tmp : z);
        if (j == 1) {
            a = cf[0] / tb;
            b = cf[1] / tb + cf[3];
        } else if (j == 2) {
            a = cf[0];
            b = cf[1];
            d = cf[2] / tb + cf[3];
        } else {
            a = cf[0];
            b = cf[1];
            c = cf[2];
            d = cf[3];
        }
        for (int it = blockIdx.x; it < items; it += gridDim.x) {
            const int bx = it % gx, by = (it / gx) % gy, bz = it / (gx * gy);
            const int x = bx * ST_BX + (V2 ? 2 : 1) * threadIdx.x, y = by * ST_BY + threadIdx.y;
            const int z0 = DIM == 3 ? bz * zc : 0, z1 = DIM == 3 ? min(z0 + zc, S.nzl) : 1;
            if (x >= S.nx || y >= S.ny) continue;
            if (V2) {
                const int pidx = x + S.nx * y;
                long long i = pidx + plane * z0;
                const bool has_l = x > 0, has_r = x + 2 < S.nx, has_d = y > 0, has_u = y < S.ny - 1;
                double2 below = make_double2(0.0, 0.0), cur = *reinterpret_cast<const double2 *>(X + i);
                if (DIM == 3 && z0 > 0) below = *reinterpret_cast<const double2 *>(X + i - plane);
                for (int zz = z0; zz < z1; ++zz, i += plane) {
                    double2 above = make_double2(0.0, 0.0);
                    if (DIM == 3 && zz + 1 < S.nzl) above = *reinterpret_cast<const double2 *>(X + i + plane);
                    double na = below.x, nb = below.y;
                    if (has_d) {
                        const double2 t = *reinterpret_cast<const double2 *>(X + i - S.nx);
                        na += t.x;
                        nb += t.y;
                    }
                    if (has_l) na += X[i - 1];
                    nb += cur.x;
                    na += cur.y;
                    if (has_r) nb += X[i + 2];
                    if (has_u) {
                        const double2 t = *reinterpret_cast<const double2 *>(X + i + S.nx);
                        na += t.x;
                        nb += t.y;
                    }
                    na += above.x;
                    nb += above.y;
                    double2 o;
                    o.x = st_lin(a, st_ax(S.diag, cur.x, S.off, na), b, cur.x);
                    o.y = st_lin(a, st_ax(S.diag, cur.y, S.off, nb), b, cur.y);
                    if (j >= 3) {
                        const double2 t = *reinterpret_cast<const double2 *>(out + i);
                        o.x = __fma_rn(c, t.x, o.x);
                        o.y = __fma_rn(c, t.y, o.y);
                    }
                    if (j >= 2) {
                        const double2 t = *reinterpret_cast<const double2 *>(r + i);
                        o.x = __fma_rn(d, t.x, o.x);
                        o.y = __fma_rn(d, t.y, o.y);
                    }
                    *reinterpret_cast<double2 *>(out + i) = o;
                    if (j == k && dotv) {
                        const double2 t = *reinterpret_cast<const double2 *>(dotv + i);
                        acc += o.x * t.x;
                        acc += o.y * t.y;
                    }
                    below = cur;
                    cur = above;
                }
                continue;
            }
            const int pidx = x + S.nx * y;
            long long i = pidx + plane * z0;
            double below = 0.0, cur = X[i];
            if (DIM == 3 && z0 > 0) below = X[i - plane];
            for (int zz = z0; zz < z1; ++zz, i += plane) {
                double above = 0.0;
                if (DIM == 3 && zz + 1 < S.nzl) above = X[i + plane];
                double nb = below;
                if (y > 0) nb += X[i - S.nx];
                if (x > 0) nb += X[i - 1];
                if (x < S.nx - 1) nb += X[i + 1];
                if (y < S.ny - 1) nb += X[i + S.nx];
                nb += above;
                const double ax = st_ax(S.diag, cur, S.off, nb);
                double o = st_lin(a, ax, b, cur);
                if (j >= 3) o = __fma_rn(c, out[i], o);
                if (j >= 2) o = __fma_rn(d, r[i], o);
                out[i] = o;
                if (j == k && dotv) acc += o * dotv[i];
                below = cur;
                cur = above;
            }
        }
        if (j < k) grid.sync();
    }
    if (dotv) {
        acc = block_sum<(V2 ? SV_BX : ST_BX) * ST_BY>(acc, red);
        if (threadIdx.x == 0 && threadIdx.y == 0) partials[blockIdx.x] = acc;
    }
}

// ---------------------------------------------------------------- TMA-staged one-degree kernel
// The north-star stencil design: the input vector is staged in shared memory by TMA tensor
// copies.  A CTA owns a TX x TY (x, y) tile and marches z through a chunk of planes; plane z
// of s_{j-1} arrives as ONE cp.async.bulk.tensor box of (TX + 4) x (TY + 2) x 1 elements
// starting at (x0 - 2, y0 - 1, z): the in-plane halo comes with it and the hardware zero-
// fills everything outside the grid, which IS the homogeneous Dirichlet boundary (reading A13),
// so the kernel has no boundary branches.  The planes z-1, z, z+1 the 7-point product needs sit
// in a ring of ST_NS stages; s_{j-2} and r of plane z ride in the same stage (two TX x TY boxes)
// and plane z+3 is issued as soon as plane z is done, so two planes of every stream are in
// flight while one is computed.  Each stage has its own mbarrier (expect_tx = box bytes).
// Persistent grid (2 CTAs per SM); work items are (tile, z-chunk) pairs, neighbouring tiles
// of one chunk on consecutive CTAs so that halos are re-read from L2.  The neighbour sum is
// formed in the order of k_stencil_step (z-1, y-1, x-1, x+1, y+1, z+1) and a zero-filled
// neighbour adds +0.0, so both kernels give bitwise the same result.
#ifndef NPC_TS_Y
#define NPC_TS_Y 16
#endif
#ifndef NPC_TS_NS
#define NPC_TS_NS 4
#endif
static constexpr int TS_X = 32, TS_Y = NPC_TS_Y, TS_THREADS = 256, TS_NS = NPC_TS_NS;  // A/B: NPC_TS_Y, NPC_TS_NS
static constexpr int TS_CTAS_PER_SM = (227 * 1024) / ((TS_NS * ((((TS_X + 4) * (TS_Y + 2) * 8 + 127) / 128) * 128 +
                                                                2 * TS_X * TS_Y * 8)) + 128 + 1024);
// the box's inner (x) start must be 16-byte aligned (an odd fp64 start faults), so the x halo is
// 2 wide on each side: box (TS_X + 4) x (TS_Y + 2) from (x0 - 2, y0 - 1)
static constexpr int TS_PX = TS_X + 4, TS_PY = TS_Y + 2;
static constexpr int TS_XBOX = TS_PX * TS_PY;                     // doubles of a staged x plane
static constexpr int TS_XSLOT = ((TS_XBOX * 8 + 127) / 128) * 16;  // its slot, 128-byte multiple
static constexpr int TS_VBOX = TS_X * TS_Y;                       // s_{j-2} / r plane box
static constexpr int TS_STAGE = TS_XSLOT + 2 * TS_VBOX;           // doubles per stage
static constexpr size_t TS_SMEM = (size_t)TS_NS * TS_STAGE * 8 + 128;  // + alignment slack

struct StencilTma {
    int nx, ny, nz, zc, tiles_x, tiles_y, items, npart_total;
    double diag, off;
};

template <int DIM, bool HAS_S2, bool HAS_R, bool DOT>
__global__ void __launch_bounds__(TS_THREADS) k_stencil_tma(const __grid_constant__ CUtensorMap mx,
                                                            const __grid_constant__ CUtensorMap ms2,
                                                            const __grid_constant__ CUtensorMap mr, StencilTma T,
                                                            StepArgs s) {
    extern __shared__ __align__(128) unsigned char sm_raw[];
    // tensor copies need a 128-byte aligned destination: align the dynamic base explicitly
    double *sm = reinterpret_cast<double *>(sm_raw + ((128u - (smem_u32(sm_raw) & 127u)) & 127u));
    __shared__ uint64_t bar[TS_NS];
    __shared__ double red[TS_THREADS / 32];
    if (s.done && *s.done) return;  // uniform: before any copy is issued
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    if (threadIdx.x == 0) {
        for (int b = 0; b < TS_NS; ++b) mbar_init(&bar[b], 1);
        fence_mbar_init();
        tma_prefetch_desc(&mx);
        if (HAS_S2) tma_prefetch_desc(&ms2);
        if (HAS_R) tma_prefetch_desc(&mr);
    }
    __syncthreads();
    uint32_t phase = 0;  // bit b: parity of stage b's next completion
    const long long plane = (long long)T.nx * T.ny;
    const int ntiles = T.tiles_x * T.tiles_y;
    double acc = 0.0;
    for (int item = blockIdx.x; item < T.items; item += gridDim.x) {
        const int tile = item % ntiles, chunk = item / ntiles;
        const int x0 = (tile % T.tiles_x) * TS_X, y0 = (tile / T.tiles_x) * TS_Y;
        const int z0 = DIM == 3 ? chunk * T.zc : 0, z1 = DIM == 3 ? min(z0 + T.zc, T.nz) : 1;
        // plane q (z0 - 1 <= q <= z1) lives in stage (q - z0 + 1) % TS_NS
        auto issue = [&](int q) {
            const int b = (q - z0 + 1) % TS_NS;
            double *st = sm + (size_t)b * TS_STAGE;
            const bool own = q >= z0 && q < z1;  // s_{j-2} and r only for computed planes
            const uint32_t bytes = TS_XBOX * 8u + (own ? ((HAS_S2 ? 1u : 0u) + (HAS_R ? 1u : 0u)) * TS_VBOX * 8u : 0u);
            mbar_arrive_expect_tx(&bar[b], bytes);
            if (DIM == 3) {
                tma_load_3d(st, &mx, x0 - 2, y0 - 1, q, &bar[b]);
                if (own && HAS_S2) tma_load_3d(st + TS_XSLOT, &ms2, x0, y0, q, &bar[b]);
                if (own && HAS_R) tma_load_3d(st + TS_XSLOT + TS_VBOX, &mr, x0, y0, q, &bar[b]);
            } else {
                tma_load_2d(st, &mx, x0 - 2, y0 - 1, &bar[b]);
                if (HAS_S2) tma_load_2d(st + TS_XSLOT, &ms2, x0, y0, &bar[b]);
                if (HAS_R) tma_load_2d(st + TS_XSLOT + TS_VBOX, &mr, x0, y0, &bar[b]);
            }
        };
        const int qlo = DIM == 3 ? z0 - 1 : 0, qhi = DIM == 3 ? z1 : 0;  // planes to stage
        if (threadIdx.x == 0)
            for (int q = qlo; q <= min(qhi, qlo + TS_NS - 1); ++q) issue(q);
        int waited = qlo - 1;  // planes <= waited have landed
        for (int z = z0; z < z1; ++z) {
            for (int q = waited + 1; q <= min(DIM == 3 ? z + 1 : z, qhi); ++q) {
                const int b = (q - z0 + 1) % TS_NS;
                mbar_wait(&bar[b], (phase >> b) & 1u);
                phase ^= 1u << b;
            }
            waited = min(DIM == 3 ? z + 1 : z, qhi);
            const double *cur = sm + (size_t)((z - z0 + 1) % TS_NS) * TS_STAGE;
            const double *blw = sm + (size_t)((z - z0) % TS_NS) * TS_STAGE;
            const double *abv = sm + (size_t)((z - z0 + 2) % TS_NS) * TS_STAGE;
#pragma unroll
            for (int k = 0; k < TS_Y / (TS_THREADS / 32); ++k) {
                const int ly = ty + (TS_THREADS / 32) * k;
                const int x = x0 + tx, y = y0 + ly;
                const int c = (ly + 1) * TS_PX + tx + 2;
                const double xc = cur[c];
                double nb = DIM == 3 ? blw[c] : 0.0;
                nb += cur[c - TS_PX];
                nb += cur[c - 1];
                nb += cur[c + 1];
                nb += cur[c + TS_PX];
                if (DIM == 3) nb += abv[c];
                const double ax = st_ax(T.diag, xc, T.off, nb);
                double o = st_lin(s.a, ax, s.b, xc);
                if (HAS_S2) o = __fma_rn(s.c, cur[TS_XSLOT + ly * TS_X + tx], o);
                if (HAS_R) o = __fma_rn(s.d, cur[TS_XSLOT + TS_VBOX + ly * TS_X + tx], o);
                if (x < T.nx && y < T.ny) {
                    const long long i = x + (long long)T.nx * y + plane * z;
                    s.out[i] = o;
                    if (DOT) acc += o * s.dotv[i];
                }
            }
            __syncthreads();  // every thread is done with plane z - 1's stage
            // plane z + TS_NS - 1 takes plane z - 1's stage (the prologue staged up to z0 + TS_NS - 2)
            if (DIM == 3 && threadIdx.x == 0 && z + TS_NS - 1 <= qhi) issue(z + TS_NS - 1);
        }
    }
    if (DOT) {
        acc = block_sum<TS_THREADS>(acc, red);
        if (threadIdx.x == 0) s.partials[blockIdx.x] = acc;
        if (blockIdx.x == 0)  // the other path's extra partial slots
            for (int k = gridDim.x + threadIdx.x; k < T.npart_total; k += TS_THREADS) s.partials[k] = 0.0;
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
                    const double ax = st_ax(diag, cur, off, nb);
                    v = st_lin(S.a1, ax, S.b1, cur);
                    if (S.x2) v = __fma_rn(S.c1, s2c[u], v);
                    v = __fma_rn(S.d1, rc[u], v);
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
                const double ax = st_ax(diag, cur, off, nb);
                const double sjm1 = P[(zo + 4) & 3][(threadIdx.y + 2) * TPX + threadIdx.x + 2];
                double o = st_lin(S.a2, ax, S.b2, cur);
                o = __fma_rn(S.c2, sjm1, o);
                o = __fma_rn(S.d2, Rr[(zo + 3) % 3][qe], o);
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

// ---------------------------------------------------------------- TMA-staged two-degree kernel
// Temporal blocking (as k_stencil_step2) on the TMA pipeline of k_stencil_tma: a 32 x 16 tile
// marches z; stage q holds three tensor boxes of plane q -- s_{j-1} with a halo of 2
// ((32 + 4) x (16 + 4) from (x0 - 2, y0 - 2)), s_{j-2} and r with a halo of 1 rounded to the
// aligned box (32 + 4) x (16 + 2) from (x0 - 2, y0 - 1) -- in a ring of T2_NS stages; s_j is
// computed on the tile + halo 1 into a shared ring of 3 planes (zero outside the grid), and
// s_{j+1} of plane z - 1 from s_j planes z - 2 .. z.  Both outputs are written (s_j is the next
// pair's s_{j-2}).  Per point and two degrees HBM sees s_{j-1}, s_{j-2}, r read and s_j, s_{j+1}
// written: 5 streams instead of 8; the halo re-reads come from L2.  Same arithmetic and order
// as the one-degree kernels: bitwise equal to two k_stencil_tma / k_stencil_step launches.
static constexpr int T2_X = 32, T2_Y = 16, T2_THREADS = 256, T2_NS = 5;
static constexpr int T2_PX = T2_X + 4, T2_PY = T2_Y + 4;  // s_{j-1} box
static constexpr int T2_VX = T2_X + 4, T2_VY = T2_Y + 2;  // s_{j-2} / r box
static constexpr int T2_QX = T2_X + 2, T2_QY = T2_Y + 2;  // s_j region (halo 1)
static constexpr int T2_PSLOT = ((T2_PX * T2_PY * 8 + 127) / 128) * 16;  // doubles, 128-byte multiple
static constexpr int T2_VSLOT = ((T2_VX * T2_VY * 8 + 127) / 128) * 16;
static constexpr int T2_STAGE = T2_PSLOT + 2 * T2_VSLOT;
static constexpr int T2_QN = T2_QX * T2_QY;
static constexpr size_t T2_SMEM = ((size_t)T2_NS * T2_STAGE + 3 * T2_QN) * 8 + 128;

struct StencilTma2 {
    int nx, ny, nz, zc, tiles_x, tiles_y, items, npart_total;
    double diag, off;
    double a1, b1, c1, d1, a2, b2, c2, d2;
    double *o1, *o2;
    const double *dotv;
    double *partials;
    const int *done;
    bool has_s2;
};

template <bool DOT>
__global__ void __launch_bounds__(T2_THREADS) k_stencil_tma2(const __grid_constant__ CUtensorMap mp,
                                                             const __grid_constant__ CUtensorMap m2,
                                                             const __grid_constant__ CUtensorMap mr, StencilTma2 T) {
    extern __shared__ __align__(128) unsigned char t2_raw[];
    double *sm = reinterpret_cast<double *>(t2_raw + ((128u - (smem_u32(t2_raw) & 127u)) & 127u));
    double *Q = sm + (size_t)T2_NS * T2_STAGE;  // s_j ring, 3 planes
    __shared__ uint64_t bar[T2_NS];
    __shared__ double red[T2_THREADS / 32];
    if (T.done && *T.done) return;
    if (threadIdx.x == 0) {
        for (int b = 0; b < T2_NS; ++b) mbar_init(&bar[b], 1);
        fence_mbar_init();
    }
    __syncthreads();
    uint32_t phase = 0;
    const long long plane = (long long)T.nx * T.ny;
    const int ntiles = T.tiles_x * T.tiles_y;
    double acc = 0.0;
    for (int item = blockIdx.x; item < T.items; item += gridDim.x) {
        const int tile = item % ntiles, chunk = item / ntiles;
        const int x0 = (tile % T.tiles_x) * T2_X, y0 = (tile / T.tiles_x) * T2_Y;
        const int z0 = chunk * T.zc, z1 = min(z0 + T.zc, T.nz);
        const int qlo = z0 - 2, qhi = z1 + 1;  // planes staged: s_j is needed on z0-1 .. z1
        auto slot = [&](int q) { return (q - qlo) % T2_NS; };
        auto issue = [&](int q) {
            const int b = slot(q);
            double *st = sm + (size_t)b * T2_STAGE;
            const bool need_v = q >= z0 - 1 && q <= z1;  // s_{j-2}, r: where s_j is computed
            const uint32_t bytes = T2_PX * T2_PY * 8u + (need_v ? ((T.has_s2 ? 1u : 0u) + 1u) * T2_VX * T2_VY * 8u : 0u);
            mbar_arrive_expect_tx(&bar[b], bytes);
            tma_load_3d(st, &mp, x0 - 2, y0 - 2, q, &bar[b]);
            if (need_v) {
                if (T.has_s2) tma_load_3d(st + T2_PSLOT, &m2, x0 - 2, y0 - 1, q, &bar[b]);
                tma_load_3d(st + T2_PSLOT + T2_VSLOT, &mr, x0 - 2, y0 - 1, q, &bar[b]);
            }
        };
        if (threadIdx.x == 0)
            for (int q = qlo; q <= min(qhi, qlo + T2_NS - 1); ++q) issue(q);
        int waited = qlo - 1;
        for (int zz = z0 - 1; zz <= z1; ++zz) {
            // s_j at plane zz needs s_{j-1} planes zz-1 .. zz+1 (and s_{j-2}, r of plane zz)
            for (int q = waited + 1; q <= zz + 1; ++q) {
                const int b = slot(q);
                mbar_wait(&bar[b], (phase >> b) & 1u);
                phase ^= 1u << b;
            }
            waited = zz + 1;
            const double *Pm = sm + (size_t)slot(zz - 1) * T2_STAGE, *P0 = sm + (size_t)slot(zz) * T2_STAGE,
                         *Pp = sm + (size_t)slot(zz + 1) * T2_STAGE;
            double *Qz = Q + (size_t)((zz + 3) % 3) * T2_QN;
            for (int e = threadIdx.x; e < T2_QN; e += T2_THREADS) {
                const int qx = e % T2_QX, qy = e / T2_QX;
                const int gx = x0 + qx - 1, gy = y0 + qy - 1;
                double v = 0.0;
                if (gx >= 0 && gx < T.nx && gy >= 0 && gy < T.ny && zz >= 0 && zz < T.nz) {
                    const int pe = (qy + 1) * T2_PX + qx + 1;  // s_{j-1} box position
                    const int ve = qy * T2_VX + qx + 1;        // s_{j-2} / r box position
                    const double cur = P0[pe];
                    double nb = Pm[pe];
                    nb += P0[pe - T2_PX];
                    nb += P0[pe - 1];
                    nb += P0[pe + 1];
                    nb += P0[pe + T2_PX];
                    nb += Pp[pe];
                    const double ax = st_ax(T.diag, cur, T.off, nb);
                    v = st_lin(T.a1, ax, T.b1, cur);
                    if (T.has_s2) v = __fma_rn(T.c1, P0[T2_PSLOT + ve], v);
                    v = __fma_rn(T.d1, P0[T2_PSLOT + T2_VSLOT + ve], v);
                }
                Qz[e] = v;
            }
            __syncthreads();  // s_j plane zz complete
            // s_{j+1} at plane zo = zz - 1 on the tile
            const int zo = zz - 1;
            if (zo >= z0 && zo < z1) {
                const double *Qm = Q + (size_t)((zo + 2) % 3) * T2_QN, *Q0 = Q + (size_t)((zo + 3) % 3) * T2_QN,
                             *Qp = Q + (size_t)((zo + 4) % 3) * T2_QN;
                const double *Po = sm + (size_t)slot(zo) * T2_STAGE;
                for (int e = threadIdx.x; e < T2_X * T2_Y; e += T2_THREADS) {
                    const int lx = e % T2_X, ly = e / T2_X;
                    const int gx = x0 + lx, gy = y0 + ly;
                    if (gx < T.nx && gy < T.ny) {
                        const int qe = (ly + 1) * T2_QX + lx + 1;
                        const double cur = Q0[qe];
                        double nb = Qm[qe];
                        nb += Q0[qe - T2_QX];
                        nb += Q0[qe - 1];
                        nb += Q0[qe + 1];
                        nb += Q0[qe + T2_QX];
                        nb += Qp[qe];
                        const double ax = st_ax(T.diag, cur, T.off, nb);
                        const double sjm1 = Po[(ly + 2) * T2_PX + lx + 2];
                        const double rr = Po[T2_PSLOT + T2_VSLOT + (ly + 1) * T2_VX + lx + 2];
                        double o = st_lin(T.a2, ax, T.b2, cur);
                        o = __fma_rn(T.c2, sjm1, o);
                        o = __fma_rn(T.d2, rr, o);
                        const long long i = gx + (long long)T.nx * gy + plane * zo;
                        T.o1[i] = cur;
                        T.o2[i] = o;
                        if (DOT) acc += o * T.dotv[i];
                    }
                }
            }
            __syncthreads();  // stage of plane zz - 1 and s_j plane zz - 2 are free
            // plane zz - 1's stage is free once s_{j+1} of plane zz - 1 is done: refill it with
            // plane zz - 1 + T2_NS
            if (threadIdx.x == 0 && zz - 1 + T2_NS <= qhi && zz - 1 >= qlo) issue(zz - 1 + T2_NS);
        }
    }
    if (DOT) {
        acc = block_sum<T2_THREADS>(acc, red);
        if (threadIdx.x == 0) T.partials[blockIdx.x] = acc;
        if (blockIdx.x == 0)
            for (int k = gridDim.x + threadIdx.x; k < T.npart_total; k += T2_THREADS) T.partials[k] = 0.0;
    }
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda at link time)
static PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = []() -> PFN_cuTensorMapEncodeTiled_v12000 {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            return nullptr;
        return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }();
    return fn;
}

class StencilOperator : public Operator {
  public:
    int dim = 3, nx = 0, ny = 0, nzg = 1, zb = 0, nzl = 1;
    double diag = 0, off = 0;
    bool multi = false, has_lo = false, has_hi = false;
    int zc_main = ST_ZC;  // z-planes marched per CTA (NPC_ST_ZC for A/B)
    HaloPlan plan;
    HaloRuntime halo;
    // TMA-staged kernel (k_stencil_tma): single rank, even nx (16-byte row strides), 16-byte
    // aligned vectors; tensor maps cached per (pointer, box kind)
    bool tma = false;
    bool vec2 = false;  // k_stencil_step_v2 (two x-points per thread, 128-bit accesses)
    int tma_blocks = 0, tma_zc = 0, tma_items = 0;
    bool tma2 = false;  // k_stencil_tma2 for the paired degrees (step2)
    // k_stencil_poly_grid: single rank, vectors L2-resident; co-resident grid size (0 = off)
    int grid_blocks = 0, grid_zc = 1, grid_cap_scalar = 0;
    DevBuf poly_tmp;  // its scratch vector (s_{k-1}, s_{k-3}, ...), allocated at create
    int tma2_blocks = 0, tma2_zc = 0, tma2_items = 0;
    std::map<std::pair<const void *, int>, CUtensorMap> tmaps;

    // box kinds: 0 = TS_X x TS_Y (k_stencil_tma s_{j-2}, r), 1 = its s_{j-1} box with halo,
    // 2 = T2_PX x T2_PY (k_stencil_tma2 s_{j-1}), 3 = T2_VX x T2_VY (its s_{j-2}, r)
    const CUtensorMap *tensor_map(const double *p, int box_kind) {
        static const cuuint32_t BX[4] = {TS_X, TS_PX, T2_PX, T2_VX}, BY[4] = {TS_Y, TS_PY, T2_PY, T2_VY};
        auto key = std::make_pair((const void *)p, box_kind);
        auto it = tmaps.find(key);
        if (it != tmaps.end()) return &it->second;
        auto enc = tensor_map_encoder();
        if (!enc) return nullptr;
        CUtensorMap m;
        const cuuint64_t dims[3] = {(cuuint64_t)nx, (cuuint64_t)ny, (cuuint64_t)std::max(nzl, 1)};
        const cuuint64_t strides[2] = {(cuuint64_t)nx * 8, (cuuint64_t)nx * ny * 8};
        const cuuint32_t box[3] = {BX[box_kind], BY[box_kind], 1};
        const cuuint32_t es[3] = {1, 1, 1};
        const CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, dim == 3 ? 3 : 2, const_cast<double *>(p), dims,
                               strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                               CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) return nullptr;
        if (tmaps.size() > 64) tmaps.clear();  // bounded: a few work vectors per polynomial
        return &(tmaps[key] = m);
    }
    static bool al16(const void *p) { return p == nullptr || ((uintptr_t)p & 15) == 0; }

    template <int D, bool H2, bool HR, bool DT>
    npc_status launch_tma_t(const StepArgs &s, const CUtensorMap *mx, const CUtensorMap *m2, const CUtensorMap *mr) {
        StencilTma T{nx, ny, nzl, tma_zc, ceil_div(nx, TS_X), ceil_div(ny, TS_Y), tma_items, num_partials(), diag, off};
        auto kern = k_stencil_tma<D, H2, HR, DT>;
        NPC_TRY(allow_max_dynamic_smem(kern));
        kern<<<tma_blocks, TS_THREADS, TS_SMEM, ctx->stream>>>(*mx, m2 ? *m2 : *mx, mr ? *mr : *mx, T, s);
        NPC_LAUNCH_CHECK();
        return NPC_SUCCESS;
    }
    template <int D>
    npc_status launch_tma_d(const StepArgs &s, const CUtensorMap *mx, const CUtensorMap *m2, const CUtensorMap *mr) {
        const bool h2 = s.s2 != nullptr, hr = s.r != nullptr, dt = s.dotv != nullptr;
        if (h2 && hr && dt) return launch_tma_t<D, true, true, true>(s, mx, m2, mr);
        if (h2 && hr) return launch_tma_t<D, true, true, false>(s, mx, m2, mr);
        if (h2 && dt) return launch_tma_t<D, true, false, true>(s, mx, m2, mr);
        if (h2) return launch_tma_t<D, true, false, false>(s, mx, m2, mr);
        if (hr && dt) return launch_tma_t<D, false, true, true>(s, mx, m2, mr);
        if (hr) return launch_tma_t<D, false, true, false>(s, mx, m2, mr);
        if (dt) return launch_tma_t<D, false, false, true>(s, mx, m2, mr);
        return launch_tma_t<D, false, false, false>(s, mx, m2, mr);
    }
    // true if launched; false -> the caller takes k_stencil_step
    npc_status try_launch_tma(const StepArgs &s, bool *done) {
        *done = false;
        if (!tma || !al16(s.x) || !al16(s.s2) || !al16(s.r)) return NPC_SUCCESS;
        const CUtensorMap *mx = tensor_map(s.x, 1);
        const CUtensorMap *m2 = s.s2 ? tensor_map(s.s2, 0) : nullptr;
        const CUtensorMap *mr = s.r ? tensor_map(s.r, 0) : nullptr;
        if (!mx || (s.s2 && !m2) || (s.r && !mr)) return NPC_SUCCESS;
        *done = true;
        return dim == 3 ? launch_tma_d<3>(s, mx, m2, mr) : launch_tma_d<2>(s, mx, m2, mr);
    }

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
        if (!multi) return std::max(std::max(blocks_for(nzl, zc_main), tma ? tma_blocks : 0), grid_blocks);
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
        if (vec2 && al16(s.x) && al16(s.s2) && al16(s.r) && al16(s.out) && al16(s.dotv) && al16(S.glo) && al16(S.ghi)) {
            k_stencil_step_v2<D, H2, HR, DT><<<grid_for(z_hi - z_lo, zc), dim3(SV_BX, ST_BY), 0, ctx->stream>>>(S, a, z_lo, z_hi, zc);
        } else
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
        if (tma) return tma2;  // k_stencil_tma2 only when opted in (NPC_ST_TMA2=1)
        int l2 = 0;
        if (cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, ctx->device) != cudaSuccess || l2 <= 0)
            l2 = 126 << 20;
        return 4.0 * 8.0 * n_local > 0.75 * l2;
    }
    int num_partials2() const override {
        dim3 g = grid2();
        return std::max((int)(g.x * g.y * g.z), tma2 ? tma2_blocks : 0);
    }
    double bytes_per_step2() const override { return 5.0 * 8.0 * n_local; }
    npc_status step2(const StepArgs &s1, const StepArgs &s2) override {
        Step2Args S{s1.x, s1.s2, s1.r, s1.out, s2.out, s2.dotv, s2.partials, s1.done,
                    s1.a, s1.b, s1.c, s1.d, s2.a, s2.b, s2.c, s2.d};
        if (!S.r) {
            set_error("stencil step2: r is required");
            return NPC_ERR_INVALID_ARGUMENT;
        }
        if (tma2 && al16(s1.x) && al16(s1.s2) && al16(s1.r)) {
            const CUtensorMap *mp = tensor_map(s1.x, 2);
            const CUtensorMap *m2 = s1.s2 ? tensor_map(s1.s2, 3) : nullptr;
            const CUtensorMap *mr = tensor_map(s1.r, 3);
            if (mp && mr && (!s1.s2 || m2)) {
                StencilTma2 T{nx, ny, nzl, tma2_zc, ceil_div(nx, T2_X), ceil_div(ny, T2_Y), tma2_items,
                              num_partials2(), diag, off, s1.a, s1.b, s1.c, s1.d, s2.a, s2.b, s2.c, s2.d,
                              s1.out, s2.out, s2.dotv, s2.partials, s1.done, s1.s2 != nullptr};
                if (s2.dotv) {
                    NPC_TRY(allow_max_dynamic_smem(k_stencil_tma2<true>));
                    k_stencil_tma2<true><<<tma2_blocks, T2_THREADS, T2_SMEM, ctx->stream>>>(*mp, m2 ? *m2 : *mr, *mr, T);
                } else {
                    NPC_TRY(allow_max_dynamic_smem(k_stencil_tma2<false>));
                    k_stencil_tma2<false><<<tma2_blocks, T2_THREADS, T2_SMEM, ctx->stream>>>(*mp, m2 ? *m2 : *mr, *mr, T);
                }
                NPC_LAUNCH_CHECK();
                return NPC_SUCCESS;
            }
        }
        if (S.dotv && num_partials2() > (int)(grid2().x * grid2().y * grid2().z)) {
            const int nb = (int)(grid2().x * grid2().y * grid2().z);
            NPC_TRY(launch_fill(ctx, S.partials + nb, 0.0, num_partials2() - nb));
        }
        const int zc = zc2();
        if (s2.dotv)
            k_stencil_step2<true><<<grid2(), dim3(TBX, TBY), 0, ctx->stream>>>(nx, ny, nzl, zc, diag, off, S);
        else
            k_stencil_step2<false><<<grid2(), dim3(TBX, TBY), 0, ctx->stream>>>(nx, ny, nzl, zc, diag, off, S);
        NPC_LAUNCH_CHECK();
        return NPC_SUCCESS;
    }

    // Eager calls only: while the PCG captures its CUDA graph the per-degree kernels are taken.
    // Measured on config 2 (profiles/r02_stencil_grid_ab.md): eagerly, k launches pay ~1 us of
    // launch gap each and the one cooperative launch is 9 % faster per p_30; inside a graph the
    // kernel nodes follow each other as closely as the grid barriers do, and the per-degree
    // kernel's 8 CTAs/SM beat the grid kernel's 4 (PCG solve 8.87 vs 9.12 ms).
    bool supports_fused_poly() const override {
        if (grid_blocks <= 0 || getenv("NPC_NO_GRID_POLY")) return false;
        if (getenv("NPC_GRID_IN_GRAPH")) return true;  // A/B
        // with the 128-bit kernels k per-degree launches beat the cooperative launch even eagerly
        // (config 2 p_30: 0.248 vs 0.257 ms, profiles/r02_stencil_vec2_ab.md); NPC_GRID_POLY=1 forces it
        if (vec2 && !getenv("NPC_GRID_POLY")) return false;
        cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
        return cudaStreamIsCapturing(ctx->stream, &cs) == cudaSuccess && cs == cudaStreamCaptureStatusNone;
    }
    npc_status apply_poly_fused(const double *r, double *z, const double *coef_dev, int k, double tb,
                                const double *dotv, double *partials, int *nparts, const int *done) override {
        double *tmp = poly_tmp.as<double>();  // z holds s_k, s_{k-2}, ...
        StencilDev S{nx, ny, nzl, diag, off, nullptr, nullptr};
        const int zc = grid_zc;
        cudaLaunchConfig_t cfg = {};
        // the 128-bit form needs aligned vectors; otherwise the scalar form on at most its own
        // co-resident grid (items are strided over whatever grid is launched)
        const bool v2 = vec2 && al16(r) && al16(z) && al16(dotv);
        const int gb = v2 ? grid_blocks : std::min(grid_blocks, grid_cap_scalar);
        cfg.gridDim = dim3(gb, 1, 1);
        cfg.blockDim = dim3(v2 ? SV_BX : ST_BX, ST_BY, 1);
        cfg.dynamicSmemBytes = 0;
        cfg.stream = ctx->stream;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeCooperative;
        at[0].val.cooperative = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        if (dim == 3 && v2)
            NPC_CUDA_TRY(cudaLaunchKernelEx(&cfg, k_stencil_poly_grid<3, true>, S, r, z, tmp, coef_dev, k, tb, zc, dotv,
                                            partials, done));
        else if (dim == 3)
            NPC_CUDA_TRY(cudaLaunchKernelEx(&cfg, k_stencil_poly_grid<3, false>, S, r, z, tmp, coef_dev, k, tb, zc,
                                            dotv, partials, done));
        else if (v2)
            NPC_CUDA_TRY(cudaLaunchKernelEx(&cfg, k_stencil_poly_grid<2, true>, S, r, z, tmp, coef_dev, k, tb, zc, dotv,
                                            partials, done));
        else
            NPC_CUDA_TRY(cudaLaunchKernelEx(&cfg, k_stencil_poly_grid<2, false>, S, r, z, tmp, coef_dev, k, tb, zc,
                                            dotv, partials, done));
        NPC_LAUNCH_CHECK();
        if (dotv && nparts) *nparts = gb;
        return NPC_SUCCESS;
    }

    npc_status step(const StepArgs &s) override {
        if (n_local == 0 && !multi) return NPC_SUCCESS;
        if (!multi) {
            bool done = false;
            NPC_TRY(try_launch_tma(s, &done));
            if (done) return NPC_SUCCESS;
            // k_stencil_step writes fewer partial slots than the TMA grid: zero the rest
            const int nb = blocks_for(nzl, zc_main);
            if (s.dotv && num_partials() > nb) NPC_TRY(launch_fill(ctx, s.partials + nb, 0.0, num_partials() - nb));
            return launch(s, 0, nzl, zc_main, s.partials);
        }
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
    op->vec2 = op->nx % 2 == 0 && !getenv("NPC_ST_NOV2");  // A/B: NPC_ST_NOV2=1 keeps the scalar kernels
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
    // the TMA kernel when the four vector streams exceed ~3/4 of L2 (HBM-bound: 256^3 0.94 of the
    // measured copy rate vs 0.84 for k_stencil_step); L2-resident grids keep the register kernel,
    // which reads planes through L1 without a copy round trip (128^3: 10.1 vs 12.3 us per degree).
    // NPC_ST_TMA=1 forces it on, NPC_ST_NOTMA=1 off.
    int l2 = 0;
    if (cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, ctx->device) != cudaSuccess || l2 <= 0) l2 = 126 << 20;
    const bool big = 4.0 * 8.0 * (double)op->n_local > 0.75 * l2;
    if (!ctx->distributed() && op->n_local > 0 && op->nx % 2 == 0 && !getenv("NPC_ST_NOTMA") &&
        (big || getenv("NPC_ST_TMA")) && tensor_map_encoder()) {
        op->tma = true;
        const int tiles = ceil_div(op->nx, TS_X) * ceil_div(op->ny, TS_Y);
        const int blocks_max = std::min(8, TS_CTAS_PER_SM) * ctx->num_sms;  // CTAs of TS_SMEM per SM
        // z-chunks: ~4 items per CTA for balance, >= 4 planes (each chunk re-stages 2 planes)
        int zc = op->dim == 3 ? std::max(4, (int)((long long)op->nzl * tiles / (4LL * blocks_max))) : 1;
        if (const char *e = getenv("NPC_ST_TZC")) zc = std::max(2, atoi(e));
        op->tma_zc = std::min(zc, std::max(op->nzl, 1));
        op->tma_items = tiles * (op->dim == 3 ? ceil_div(op->nzl, op->tma_zc) : 1);
        op->tma_blocks = std::min(op->tma_items, blocks_max);
        // paired degrees (opt-in, NPC_ST_TMA2=1): measured slower than the one-degree TMA kernel
        // (256^3 p_30 2.65 vs 2.55 ms, 200^3 1.51 vs 1.39 ms: two barriers and two compute phases per
        // plane at 16 warps per SM do not keep enough copies in flight), so k_stencil_tma serves
        // every degree by default
        if (op->dim == 3 && getenv("NPC_ST_TMA2")) {  // 2 CTAs of T2_SMEM per SM
            op->tma2 = true;
            const int tiles2 = ceil_div(op->nx, T2_X) * ceil_div(op->ny, T2_Y);
            const int bmax2 = std::max(1, (int)((227 * 1024) / (T2_SMEM + 1024))) * ctx->num_sms;
            int zc2v = std::max(8, (int)((long long)op->nzl * tiles2 / (4LL * bmax2)));
            if (const char *e = getenv("NPC_ST_T2ZC")) zc2v = std::max(2, atoi(e));
            op->tma2_zc = std::min(zc2v, std::max(op->nzl, 1));
            op->tma2_items = tiles2 * ceil_div(op->nzl, op->tma2_zc);
            op->tma2_blocks = std::min(op->tma2_items, bmax2);
        }
    }
    // all degrees in one cooperative launch when the vectors are L2-resident (single rank):
    // grid = min(items, co-resident CTAs)
    if (!ctx->distributed() && !big && !op->tma && op->n_local > 0 && !getenv("NPC_NO_GRID_POLY")) {
        int per_sm = 0, per_sm_s = 0, coop = 0;
        auto occ = [&](bool v2, int *out) {
            return v2 ? cudaOccupancyMaxActiveBlocksPerMultiprocessor(
                            out, op->dim == 3 ? k_stencil_poly_grid<3, true> : k_stencil_poly_grid<2, true>,
                            SV_BX * ST_BY, 0)
                      : cudaOccupancyMaxActiveBlocksPerMultiprocessor(
                            out, op->dim == 3 ? k_stencil_poly_grid<3, false> : k_stencil_poly_grid<2, false>,
                            ST_BX * ST_BY, 0);
        };
        if (cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, ctx->device) == cudaSuccess && coop &&
            occ(op->vec2, &per_sm) == cudaSuccess && occ(false, &per_sm_s) == cudaSuccess && per_sm > 0 &&
            per_sm_s > 0) {
            op->grid_cap_scalar = per_sm_s * ctx->num_sms;
            // z-chunks sized so that every (x, y, z-chunk) item has its own co-resident CTA (one
            // round per degree, no tail): chunks = co-resident CTAs / (x, y) tiles
            const long long tiles = (long long)ceil_div(op->nx, ST_BX) * ceil_div(op->ny, ST_BY);
            const long long cap = (long long)per_sm * ctx->num_sms;
            const long long chunks = std::max(1LL, std::min<long long>(op->nzl, cap / std::max(tiles, 1LL)));
            op->grid_zc = op->dim == 3 ? (int)ceil_div((long long)op->nzl, chunks) : 1;
            if (const char *e = getenv("NPC_GRID_ZC")) op->grid_zc = std::max(1, atoi(e));
            const long long items = tiles * (op->dim == 3 ? ceil_div(op->nzl, op->grid_zc) : 1);
            op->grid_blocks = (int)std::min<long long>(items, cap);
            NPC_TRY(op->poly_tmp.alloc(sizeof(double) * (size_t)op->n_local));
        }
        cudaGetLastError();
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
