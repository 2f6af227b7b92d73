// op_csr.cu -- general sparse operator in CSR (BASELINE configs 1 and 3) with the Chebyshev
// recurrence fused into the SpMV epilogue (Alg. 2 steps 5-6).
//
// Kernel design ("G2 CSR tile kernel"): one CTA per tile of 256 consecutive
// rows.  Thread 0 issues two 1D bulk-TMA copies (cp.async.bulk, mbarrier completion, L2
// evict-first) of the tile's contiguous value/column segments into shared memory while the
// other threads load rowptr, s_{j-2} and r; every thread then forms its row's dot product
// from shared memory, gathering x through L1/L2, and writes
//     out = a (A x) + b x + c s_{j-2} + d r      (+ per-CTA partial of <out, dotv>).
// Matrix bytes therefore move exactly once per degree with perfectly coalesced bulk
// transactions; the x gather of a 7-point row touches 3 planes that stay in L2.
// Multi-rank: columns outside the owned block are remapped to ghost slots; tiles that touch
// a ghost run after the halo exchange, the others overlap it.
//
// Coded column ids (default when every tile qualifies): the kernel is HBM-bound and the int32
// column ids are a third of the matrix bytes, so each tile keeps a dictionary of its distinct
// offsets (col - row), at most 256, and every entry streams a 1-byte code instead of a 4-byte
// id: 12 -> 9 B per nonzero (config 3: 2,008.5 -> 1,657 MB per degree).  Same values, same
// summation order: bitwise the same result as the plain form (NPC_CSR_PLAIN=1).
#include <unordered_map>
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <climits>
#include <cstring>
#include <thread>

#include "device_util.cuh"
#include "npc_internal.cuh"

namespace npc {

// Rows (= threads) per CTA, A/B-tuned on config 3 (p_50): plain 256 (15.21 ms; 512: 15.54),
// coded 512 (13.24 ms; 256: 13.60, 128: 13.69, 1024: 13.81) -- a coded tile carries 25 % fewer
// bytes, so it takes twice the rows to keep as much of the stream in flight per SM.
static constexpr int CSR_TILE = 256, CSR_TILE_CODED = 512;
static constexpr int CSR_MAX_SMEM = 200 * 1024;

static constexpr int CSR_DICT_MAX = 256;

struct CsrDev {
    const int *rowptr;
    const int *cols;  // local ids: [0, n) owned, [n, n + n_ghost) ghost slots
    const double *vals;
    int n;
    const double *ghost;
    const unsigned char *codes;  // coded form: entry p's column = row + dict[dict_off[tile] + codes[p]]
    const int *dict, *dict_off;
    const int *tptr;              // coded form: first entry of each tile (ntiles + 1)
    const unsigned short *roff;   // coded form: row start relative to its tile's first entry
};

template <bool STAGED, bool HAS_S2, bool HAS_R, bool DOT, bool GHOST, bool CODED,
          int TILE = CODED ? CSR_TILE_CODED : CSR_TILE>
__global__ void __launch_bounds__(TILE) k_csr_step(CsrDev A, StepArgs s, const int *__restrict__ tiles,
                                                   int vspan_max) {
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ uint64_t bar;
    __shared__ double red[TILE / 32];
    __shared__ int sdict[CODED ? CSR_DICT_MAX : 1];

    const int tile = tiles ? tiles[blockIdx.x] : blockIdx.x;
    const int row0 = tile * TILE;
    const int nrows = min(TILE, A.n - row0);
    const int pb = CODED ? A.tptr[tile] : A.rowptr[row0];
    const int v0 = pb & ~1;
    const int c0 = CODED ? (pb & ~15) : (pb & ~3);  // 16 B aligned bulk-copy start
    double *sv = reinterpret_cast<double *>(smem);
    int *sc = reinterpret_cast<int *>(smem + (size_t)vspan_max * 8);
    const unsigned char *scb = smem + (size_t)vspan_max * 8;

    if (STAGED) {
        if (threadIdx.x == 0) {
            mbar_init(&bar, 1);
            fence_mbar_init();
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            const int pe = CODED ? A.tptr[tile + 1] : A.rowptr[row0 + nrows];
            const int v1 = (pe + 1) & ~1, c1 = CODED ? ((pe + 15) & ~15) : ((pe + 3) & ~3);
            const uint32_t bv = (uint32_t)(v1 - v0) * 8u, bc = (uint32_t)(c1 - c0) * (CODED ? 1u : 4u);
            // an empty tile (pe == pb) may still have bv or bc != 0 from the alignment
            // rounding: expect exactly the bytes issued, none for an empty tile
            const bool any = pe > pb;
            mbar_arrive_expect_tx(&bar, any ? bv + bc : 0u);
            if (any) {
                const uint64_t pol = policy_evict_first();
                bulk_g2s_evict_first(sv, A.vals + v0, bv, &bar, pol);
                if (CODED)
                    bulk_g2s_evict_first(smem + (size_t)vspan_max * 8, A.codes + c0, bc, &bar, pol);
                else
                    bulk_g2s_evict_first(sc, A.cols + c0, bc, &bar, pol);
            }
        }
    }
    const int row = row0 + threadIdx.x;
    const bool active = threadIdx.x < nrows;
    int rb = 0, re = 0;
    double xs = 0.0, s2v = 0.0, rv = 0.0;
    if (CODED) {  // the tile's offset dictionary (<= 256 entries, coalesced)
        const int d0 = A.dict_off[tile], dn = A.dict_off[tile + 1] - d0;
        if ((int)threadIdx.x < dn) sdict[threadIdx.x] = A.dict[d0 + threadIdx.x];
    }
    if (active) {
        if (CODED) {  // 2 B per row instead of 4
            rb = pb + A.roff[row];
            re = (int)threadIdx.x + 1 < nrows ? pb + A.roff[row + 1] : A.tptr[tile + 1];
        } else {
            rb = A.rowptr[row];
            re = A.rowptr[row + 1];
        }
        xs = s.x[row];
        if (HAS_S2) s2v = s.s2[row];
        if (HAS_R) rv = s.r[row];
    }
    // The PCG's done flag is read only now, its latency hidden behind the tile's bulk copy and
    // the row loads (checked first, it delayed every CTA's start: 1.7 % of the degree time)
    const bool is_done = s.done && *s.done;
    if (STAGED) mbar_wait(&bar, 0);  // never leave with a bulk copy into shared memory in flight
    if (is_done) return;             // uniform over the CTA
    if (CODED) __syncthreads();      // dictionary visible
    double acc = 0.0;
    if (active) {
        double y = 0.0;
        const double *__restrict__ x = s.x;
        for (int p = rb; p < re; ++p) {
            int c;
            double v;
            if (CODED) {
                c = row + sdict[STAGED ? scb[p - c0] : __ldcs(A.codes + p)];
                v = STAGED ? sv[p - v0] : __ldcs(A.vals + p);
            } else if (STAGED) {
                c = sc[p - c0];
                v = sv[p - v0];
            } else {
                c = __ldcs(A.cols + p);
                v = __ldcs(A.vals + p);
            }
            double xv;
            if (GHOST && c >= A.n)
                xv = A.ghost[c - A.n];
            else
                xv = __ldg(x + c);
            y += v * xv;
        }
        const double o = degree_epilogue<HAS_S2, HAS_R>(s, y, xs, s2v, rv);
        s.out[row] = o;
        if (DOT) acc = o * s.dotv[row];
    }
    if (DOT) {
        acc = block_sum<TILE>(acc, red);
        if (threadIdx.x == 0) s.partials[blockIdx.x] = acc;
    }
}


// ------------------------------------------------------------------------------------------
// Pattern form (default when it fits): per-row pattern ids + symmetric value mirroring.
//
// Each row stores ONE byte, the id of its pattern in the tile's pattern table, instead of a
// byte per nonzero: a pattern is the row's entry list in stored (ascending column) order,
// one 32-bit word per entry.  An "own" entry (bit 0 = 0) carries its offset o = col - row
// and takes the row's next own value.  A "mirror" entry (bit 0 = 1) is a lower-triangle
// entry a_ij (j < i, same rank) whose transpose a_ji is stored in row j with the bitwise-
// identical value: it carries o = j - i and pos, the index of a_ji among row j's own values,
// and its value is read from there.  A symmetric matrix therefore streams only its upper
// triangle: config 3 moves ~4 values per row instead of ~7.  Entries without an equal
// transpose are own entries, so any CSR matrix qualifies as long as every tile has <= 256
// distinct patterns, a table of <= PAT_TBL_MAX words and little padding (below).
//
// Own values are stored per tile of PAT_TILE rows in ELL order (position-major: the k-th own
// value of every row of the tile, then the (k+1)-th, ...; W_t = the tile's longest own list,
// shorter rows padded with zeros).  Every read is then coalesced and sector-exact: a thread's
// own values are sv[k * nrows + tid] in shared memory, a mirror inside the tile is
// sv[pos * nrows + (j - row0)], and a mirror in an earlier tile (the -N^2 and half of the -N
// neighbours of a 3D grid) is one 8-byte L2 read whose 32 neighbouring lanes read the 256
// contiguous bytes of the same position column -- no 32-byte sector per 8-byte value.  Same
// values in the same order: bitwise the same result as the plain and coded forms.
#ifndef NPC_PAT_TILE
#define NPC_PAT_TILE 1024
#endif
static constexpr int PAT_TILE = NPC_PAT_TILE;  // rows per tile (A/B: NPC_PAT_TILE)
static constexpr int PAT_TBL_MAX = 2048;  // words of one tile's pattern table (8 KB of smem)
static constexpr int PAT_MIRROR_MAX_OFF = 1 << 22;

struct PatDev {
    const double *vals;           // own values: tile blocks of W_t x nrows (position-major)
    const int *tptr;              // first value of each tile's block (ntiles + 1)
    const unsigned char *pat;     // pattern id per row
    const int *tbl, *tbl_off;     // concatenated per-tile tables: [npat + 1 starts][entry words]
    int n;
    const double *ghost;
    const int *tbl2, *tbl2_off;   // staged kernel: per-tile x windows + decoded entries
};

template <bool HAS_S2, bool HAS_R, bool DOT, bool GHOST>
__global__ void __launch_bounds__(PAT_TILE) k_csr_pat_step(PatDev A, StepArgs s, const int *__restrict__ tiles,
                                                           int vspan_max, int tbl_max) {
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ uint64_t bar;
    __shared__ double red[PAT_TILE / 32];

    const int tile = tiles ? tiles[blockIdx.x] : blockIdx.x;
    const int row0 = tile * PAT_TILE;
    const int nrows = min(PAT_TILE, A.n - row0);
    const int pb = A.tptr[tile];  // even: every block holds an even number of values
    double *sv = reinterpret_cast<double *>(smem);
    int *stbl = reinterpret_cast<int *>(smem + (size_t)vspan_max * 8);

    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        fence_mbar_init();
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        const uint32_t bv = (uint32_t)(A.tptr[tile + 1] - pb) * 8u;
        mbar_arrive_expect_tx(&bar, bv);  // an empty block expects (and issues) nothing
        if (bv) bulk_g2s(sv, A.vals + pb, bv, &bar);  // default L2 policy: mirrors re-read it
    }
    {
        const int t0 = A.tbl_off[tile], tn = A.tbl_off[tile + 1] - t0;
        for (int k = threadIdx.x; k < tn; k += PAT_TILE) stbl[k] = A.tbl[t0 + k];
    }
    const int row = row0 + threadIdx.x;
    const bool active = threadIdx.x < nrows;
    int pid = 0;
    double xs = 0.0, s2v = 0.0, rv = 0.0;
    if (active) {
        pid = A.pat[row];
        xs = s.x[row];
        if (HAS_S2) s2v = s.s2[row];
        if (HAS_R) rv = s.r[row];
    }
    const bool is_done = s.done && *s.done;
    mbar_wait(&bar, 0);  // never leave with a bulk copy into shared memory in flight
    if (is_done) return;  // uniform over the CTA
    __syncthreads();      // table visible
    double acc = 0.0;
    if (active) {
        const double *__restrict__ x = s.x;
        const int e1 = stbl[pid + 1];
        const double *own = sv + threadIdx.x;
        double y = 0.0;
        for (int e = stbl[pid]; e < e1; ++e) {
            const int w = stbl[e];
            int c;
            double v;
            if (w & 1) {  // mirror: value of a_ji, position pos of row j = c
                const int pos = (w >> 1) & 255;
                c = row + (w >> 9);
                if (c >= row0) {
                    v = sv[pos * ((nrows + 1) & ~1) + (c - row0)];  // even column stride
                } else {  // an earlier (full) tile's block, through L2
                    const int tj = c / PAT_TILE;
                    v = __ldg(A.vals + __ldg(A.tptr + tj) + pos * PAT_TILE + (c - tj * PAT_TILE));
                }
            } else {
                c = row + (w >> 1);
                v = *own;
                own += (nrows + 1) & ~1;
            }
            double xv;
            if (GHOST && c >= A.n)
                xv = A.ghost[c - A.n];
            else
                xv = __ldg(x + c);
            y += v * xv;
        }
        const double o = degree_epilogue<HAS_S2, HAS_R>(s, y, xs, s2v, rv);
        s.out[row] = o;
        if (DOT) acc = o * s.dotv[row];
    }
    if (DOT) {
        acc = block_sum<PAT_TILE>(acc, red);
        if (threadIdx.x == 0) s.partials[blockIdx.x] = acc;
    }
}

// Staged pattern kernel (the default for tiles whose x windows fit in shared memory): the
// tile's input-vector windows -- x[row0 + o, row0 + o + nrows) for every distinct offset o of
// its patterns, merged when they overlap (a 3D grid: x[row0 - N^2 ..], x[row0 - N - 1 ..
// row0 + nrows + N], x[row0 + N^2 ..]) -- are bulk-copied (TMA) into shared memory next to the
// tile's own values, so every entry reads x and its value from shared memory: one table read,
// two shared loads and an FMA per entry, no per-entry L2 round trip, and each x element
// crosses L2 ~3.5 times per degree instead of once per (row, offset).  Mirrors of earlier tiles
// stay one coalesced L2 read.  Entries are pre-decoded per tile as {x base, value base, o,
// pos}: x = sx[xb + lr], value = sv[vb + lr] when lr + o >= 0 (own entries carry o = 0).
// Two rows per thread (lr = tid, tid + PAT_TILE / 2).
static constexpr int PAT_THREADS = PAT_TILE / 2;
static constexpr int PAT_STAGE_SMEM = 110 * 1024;  // own block + x windows + table, per tile

template <bool HAS_S2, bool HAS_R>
__device__ __forceinline__ double pat_row(const PatDev &A, const StepArgs &s, const double *sv, const double *sx,
                                          const int *st, const int4 *ent, int sidx, int row0, int lr, int pid,
                                          double xs, double s2v, double rv) {
    const int row = row0 + lr;
    const int e1 = st[sidx + pid + 1];
    double y = 0.0;
    for (int e = st[sidx + pid]; e < e1; ++e) {
        const int4 t = ent[e];
        const double xv = sx[t.x + lr];
        double v;
        if (lr + t.z >= 0) {
            v = sv[t.y + lr];
        } else {  // mirror in an earlier (full) tile's block, through L2
            const int c = row + t.z, tj = c / PAT_TILE;
            v = __ldg(A.vals + __ldg(A.tptr + tj) + t.w * PAT_TILE + (c - tj * PAT_TILE));
        }
        y += v * xv;
    }
    return degree_epilogue<HAS_S2, HAS_R>(s, y, xs, s2v, rv);
}

// Two rows with the same pattern (lr0 < lr1, the common case: rows tid and tid + PAT_TILE/2 of
// an interior tile): one table read per entry and two independent FMA chains (each row's sum in
// its own stored order, so bitwise the same as two pat_row calls).
__device__ __forceinline__ void pat_row_pair(const PatDev &A, const double *sv, const double *sx, const int *st,
                                             const int4 *ent, int sidx, int row0, int lr0, int lr1, int pid,
                                             double &y0, double &y1) {
    const int e1 = st[sidx + pid + 1];
    double a0 = 0.0, a1 = 0.0;
    for (int e = st[sidx + pid]; e < e1; ++e) {
        const int4 t = ent[e];
        const double x0 = sx[t.x + lr0], x1 = sx[t.x + lr1];
        double v0, v1;
        if (lr1 + t.z >= 0) {
            v1 = sv[t.y + lr1];
        } else {
#ifdef NPC_AB_NOL2M  // A/B only (results wrong): no earlier-tile mirror reads
            v1 = 0.0;
#else
            const int c = row0 + lr1 + t.z, tj = c / PAT_TILE;
            v1 = __ldg(A.vals + __ldg(A.tptr + tj) + t.w * PAT_TILE + (c - tj * PAT_TILE));
#endif
        }
        if (lr0 + t.z >= 0) {
            v0 = sv[t.y + lr0];
        } else {
#ifdef NPC_AB_NOL2M
            v0 = 0.0;
#else
            const int c = row0 + lr0 + t.z, tj = c / PAT_TILE;
            v0 = __ldg(A.vals + __ldg(A.tptr + tj) + t.w * PAT_TILE + (c - tj * PAT_TILE));
#endif
        }
        a0 += v0 * x0;
        a1 += v1 * x1;
    }
    y0 = a0;
    y1 = a1;
}

template <bool HAS_S2, bool HAS_R, bool DOT>
__global__ void __launch_bounds__(PAT_THREADS) k_csr_pat_stage(PatDev A, StepArgs s, const int *__restrict__ tiles,
                                                               int vspan_max, int xspan_max) {
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ uint64_t bar;
    __shared__ double red[PAT_THREADS / 32];

    const int tile = tiles ? tiles[blockIdx.x] : blockIdx.x;
    const int row0 = tile * PAT_TILE;
    const int nrows = min(PAT_TILE, A.n - row0);
    double *sv = reinterpret_cast<double *>(smem);
    double *sx = sv + vspan_max;
    int *st = reinterpret_cast<int *>(sx + xspan_max);
    const int *gt = A.tbl2 + A.tbl2_off[tile];
    const int nwin = gt[0];

    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        fence_mbar_init();
    }
    __syncthreads();
    if (threadIdx.x == 0) {  // own block + every x window on one barrier
        const int pb = A.tptr[tile];
        const uint32_t bv = (uint32_t)(A.tptr[tile + 1] - pb) * 8u;
        uint32_t bx = 0;
        for (int w = 0; w < nwin; ++w) bx += (uint32_t)gt[4 + 4 * w + 1] * 8u;
        mbar_arrive_expect_tx(&bar, bv + bx);
        if (bv) bulk_g2s(sv, A.vals + pb, bv, &bar);
        for (int w = 0; w < nwin; ++w) {
            const int ga = gt[4 + 4 * w], len = gt[4 + 4 * w + 1], sb = gt[4 + 4 * w + 2];
            if (len) bulk_g2s(sx + sb, s.x + ga, (uint32_t)len * 8u, &bar);
        }
    }
    {  // the table (header, windows, pattern starts, entries) and odd window tails
        const int tn = A.tbl2_off[tile + 1] - A.tbl2_off[tile];
        for (int k = threadIdx.x; k < tn; k += PAT_THREADS) st[k] = gt[k];
        if ((int)threadIdx.x < nwin && gt[4 + 4 * threadIdx.x + 3]) {
            const int ga = gt[4 + 4 * threadIdx.x], len = gt[4 + 4 * threadIdx.x + 1];
            sx[gt[4 + 4 * threadIdx.x + 2] + len] = s.x[ga + len];
        }
    }
    const int l0 = threadIdx.x, l1 = threadIdx.x + PAT_THREADS;
    const bool a0 = l0 < nrows, a1 = l1 < nrows;
    int p0 = 0, p1 = 0;
    double x0 = 0.0, x1 = 0.0, s20 = 0.0, s21 = 0.0, r0 = 0.0, r1 = 0.0;
    if (a0) {
        p0 = A.pat[row0 + l0];
        if (HAS_S2) s20 = s.s2[row0 + l0];
        if (HAS_R) r0 = s.r[row0 + l0];
    }
    if (a1) {
        p1 = A.pat[row0 + l1];
        if (HAS_S2) s21 = s.s2[row0 + l1];
        if (HAS_R) r1 = s.r[row0 + l1];
    }
    const bool is_done = s.done && *s.done;
    mbar_wait(&bar, 0);  // never leave with a bulk copy into shared memory in flight
    if (is_done) return;  // uniform over the CTA
    __syncthreads();      // table and window tails visible
    if (a0) x0 = sx[st[3] + l0];  // x[row] from the offset-0 window
    if (a1) x1 = sx[st[3] + l1];
    const int sidx = 4 + 4 * nwin;
    const int4 *ent = reinterpret_cast<const int4 *>(st + st[1]);
    double acc = 0.0;
#ifdef NPC_AB_NOSUM  // A/B only (results wrong): the copies and the epilogue, no row sums
    if (a0) s.out[row0 + l0] = s.b * x0 + s.c * s20 + s.d * r0 + sv[l0] + (double)p0;
    if (a1) s.out[row0 + l1] = s.b * x1 + s.c * s21 + s.d * r1 + sv[l1] + (double)p1;
    if (false)
#endif
#ifndef NPC_PAT_NOPAIR
    if (a1 && p0 == p1) {  // both rows, one pattern: interleaved sums
        double y0, y1;
        pat_row_pair(A, sv, sx, st, ent, sidx, row0, l0, l1, p0, y0, y1);
        const double o0 = degree_epilogue<HAS_S2, HAS_R>(s, y0, x0, s20, r0),
                     o1 = degree_epilogue<HAS_S2, HAS_R>(s, y1, x1, s21, r1);
        s.out[row0 + l0] = o0;
        s.out[row0 + l1] = o1;
        if (DOT) acc = fma(o1, s.dotv[row0 + l1], __dmul_rn(o0, s.dotv[row0 + l0]));  // as two acc += steps
    } else
#endif
    {
        if (a0) {
            const double o = pat_row<HAS_S2, HAS_R>(A, s, sv, sx, st, ent, sidx, row0, l0, p0, x0, s20, r0);
            s.out[row0 + l0] = o;
            if (DOT) acc = o * s.dotv[row0 + l0];
        }
        if (a1) {
            const double o = pat_row<HAS_S2, HAS_R>(A, s, sv, sx, st, ent, sidx, row0, l1, p1, x1, s21, r1);
            s.out[row0 + l1] = o;
            if (DOT) acc += o * s.dotv[row0 + l1];
        }
    }
    if (DOT) {
        acc = block_sum<PAT_THREADS>(acc, red);
        if (threadIdx.x == 0) s.partials[blockIdx.x] = acc;
    }
}

// Ring kernel (the default for staged tiles; NPC_CSR_RING=0 -> k_csr_pat_stage): every operand
// of a tile's row sums is in shared memory before the sums start, so the compute phase has no
// global-memory round trip.  Per tile the host precomputes (pattern_ring_table):
//   * a copy list of <= RING_MAXD - 1 bulk copies (cp.async.bulk, one mbarrier): the tile's table,
//     its pattern ids, its own-value columns, the values of mirrors in EARLIER tiles -- near ones
//     (a 3D grid's -N for the first rows of a tile) as a "gap" directly in front of the column
//     they come from, so D[col_p + o + lr] addresses both halves, far ones (-N^2) as a window of
//     the earlier tile's column -- and the x windows; lanes of warp 0 issue one copy each, so the
//     first byte is requested one global load after the CTA starts;
//   * a table of entries {xb, vb}: x = D[xb + lr], value = D[vb + lr] for row lr of the tile --
//     one branch-free form for own values, in-tile, near and far mirrors.
// Two rows per thread (lr = tid, tid + PAT_THREADS) summed in one loop when their patterns have
// the same length.  Same values in the same order as the plain form: bitwise the same results.
// NS = 1: one tile per CTA (grid = tiles), 3 CTAs per SM, each CTA's copies in flight while the
// other CTAs compute.  NS > 1 (A/B, NPC_RING_NS): persistent CTAs walking tiles blockIdx.x +
// i * gridDim.x through NS stages, the copies of tile i + NS issued as tile i's sums finish.
static constexpr int RING_MAXD = 32;  // int4 copy descriptors per tile at most (header + copies)
static constexpr int RING_GAP_MAX = PAT_TILE;  // near earlier-tile mirrors held as a column gap
static constexpr int RING_STAGE_MAX = 110 * 1024;  // bytes of one stage

struct RingDev {
    const double *vals;          // own values (tile-ELL blocks, as PatDev::vals)
    const int *tbl;              // concatenated per-tile ring tables (16-byte aligned each)
    const unsigned char *pat;    // pattern id per row
    const int4 *desc;            // dstride descriptors per tile: {ncopies, bytes} + {kind, dst, src, bytes}
    int n;
    int dstride;                 // 16, or 32 when some tile needs more than 15 copies
};

#ifndef NPC_RING_WAIT_NS
#define NPC_RING_WAIT_NS 1000
#endif
// Warp 0: the bulk copies of one tile into a stage (x = the input vector of this step), from the
// tile's descriptor block d (lane 0: header {ncopies, bytes, has an odd x tail}; lanes 1..: one
// copy each).  part 0: everything; part 1: the barrier's arrive and the copies that do not read
// x; part 2: the x windows (a tile with an odd x tail takes part 0 only: its tail store must
// precede the arrive).
// WIDE = 0: stride 16 (every tile <= 15 copies); 1: stride 32; -1: the operator's A.dstride
template <int WIDE = -1>
__device__ __forceinline__ int4 ring_desc(const RingDev &A, int tile, int lane) {
    if (WIDE == 0) return lane < 16 ? A.desc[(size_t)tile * 16 + lane] : make_int4(0, 0, 0, 0);
    // lanes 0..15 always (the common case: <= 15 copies); 16..31 only for a tile with more
    const int4 *p = A.desc + (size_t)tile * (WIDE == 1 ? 32 : A.dstride);
    int4 d = lane < 16 ? p[lane] : make_int4(0, 0, 0, 0);
    if (A.dstride > 16 && __shfl_sync(0xffffffffu, d.x, 0) > 15 && lane >= 16) d = p[lane];
    return d;
}
__device__ __forceinline__ void ring_issue_d(const int4 &d, const RingDev &A, const double *x, unsigned char *st,
                                             uint64_t *bar, int lane, uint64_t vals_policy, bool hint, int part) {
    if (part == 0 && lane > 0 && d.x == 4) *reinterpret_cast<double *>(st + d.y) = x[d.z];  // odd x tail
    if (part != 2) {
        __syncwarp();
        if (lane == 0) mbar_arrive_expect_tx(bar, (uint32_t)d.y);
        __syncwarp();
    }
    if (lane == 0 || d.w <= 0) return;
    if (d.x == 1) {
        if (part != 1) bulk_g2s(st + d.y, x + d.z, (uint32_t)d.w, bar);
    } else if (part != 2) {
        if (d.x == 0 && hint) {
            bulk_g2s_evict_first(st + d.y, A.vals + d.z, (uint32_t)d.w, bar, vals_policy);  // any L2 policy
        } else {
            const void *src = d.x == 0 ? (const void *)(A.vals + d.z)
                              : d.x == 2 ? (const void *)(A.tbl + d.z)
                                         : (const void *)(A.pat + d.z);
            bulk_g2s(st + d.y, src, (uint32_t)d.w, bar);
        }
    }
}
template <int WIDE = -1>
__device__ __forceinline__ void ring_issue(const RingDev &A, const double *x, int tile, unsigned char *st, uint64_t *bar,
                                           int lane, uint64_t vals_policy, bool hint) {
    ring_issue_d(ring_desc<WIDE>(A, tile, lane), A, x, st, bar, lane, vals_policy, hint, 0);
}

// Per-row streams of a tile (s_{j-2}, r, the dot operand), loaded ahead into registers.
template <int R>
struct RingRows {
    double s2[R], r[R], v[R];
};
// dot_src (DOT): 0 = load dotv, 1 = dotv is the input x (taken from its staged window),
// 2 = dotv is r (taken from the r stream): the dot operand then costs no extra stream
template <bool HAS_S2, bool HAS_R, bool DOT, int R>
__device__ __forceinline__ void ring_load_rows(const double *s2, const double *r, const double *dotv, int row0,
                                               int nrows, RingRows<R> &q, int dot_src = 0) {
    constexpr int NT = PAT_TILE / R;
#pragma unroll
    for (int k = 0; k < R; ++k) {
        const int l = threadIdx.x + k * NT;
        q.s2[k] = q.r[k] = q.v[k] = 0.0;
        if (l < nrows) {
            if (HAS_S2) q.s2[k] = s2[row0 + l];
            if (HAS_R) q.r[k] = r[row0 + l];
            if (DOT && dot_src == 0) q.v[k] = dotv[row0 + l];
        }
    }
}

// The row sums and epilogue of one staged tile (every operand in shared memory).
template <bool HAS_S2, bool HAS_R, bool DOT, int R>
__device__ __forceinline__ void ring_tile(const StepArgs &s, const unsigned char *st8, int tbl_bytes, int row0,
                                          int nrows, const RingRows<R> &cur, double &acc, int dot_src = 0) {
    constexpr int NT = PAT_TILE / R;
    const int *st = reinterpret_cast<const int *>(st8);
    const unsigned char *sp = st8 + tbl_bytes;
    const char *Db = reinterpret_cast<const char *>(sp + PAT_TILE);  // D; entries are byte offsets
    const int2 *E = reinterpret_cast<const int2 *>(st + st[1]);
    const int *ps = st + 4;
    const int x0b = st[2];
    auto ld = [](const char *p, int off) { return *reinterpret_cast<const double *>(p + off); };
    int eb[R], ne[R];
    const char *Dr[R];
    double y[R];
    bool same = true;
#pragma unroll
    for (int k = 0; k < R; ++k) {
        const int l = threadIdx.x + k * NT;
        const int p = l < nrows ? sp[l] : 0;
        eb[k] = ps[p];
        ne[k] = l < nrows ? ps[p + 1] - eb[k] : 0;
        Dr[k] = Db + 8 * l;
        y[k] = 0.0;
        same = same && ne[k] == ne[0];
    }
    if (same) {  // every row in one loop (the common case: one pattern length)
#pragma unroll 2
        for (int e = 0; e < ne[0]; ++e) {
#pragma unroll
            for (int k = 0; k < R; ++k) {
                const int2 u = E[eb[k] + e];
                y[k] = fma(ld(Dr[k], u.y), ld(Dr[k], u.x), y[k]);
            }
        }
    } else {
#pragma unroll
        for (int k = 0; k < R; ++k)
            for (int e = 0; e < ne[k]; ++e) {
                const int2 u = E[eb[k] + e];
                y[k] = fma(ld(Dr[k], u.y), ld(Dr[k], u.x), y[k]);
            }
    }
#pragma unroll
    for (int k = 0; k < R; ++k) {
        const int l = threadIdx.x + k * NT;
        if (l < nrows) {
            const double xv = ld(Dr[k], x0b);
            const double o = degree_epilogue<HAS_S2, HAS_R>(s, y[k], xv, cur.s2[k], cur.r[k]);
            s.out[row0 + l] = o;
            if (DOT) acc = fma(o, dot_src == 1 ? xv : dot_src == 2 ? cur.r[k] : cur.v[k], acc);
        }
    }
}

// R rows per thread (lr = tid + q * PAT_TILE / R), summed in one interleaved loop when their
// patterns have the same length.
template <bool HAS_S2, bool HAS_R, bool DOT, int NS, int R, int WIDE = 0>
__global__ void __launch_bounds__(PAT_TILE / R, NS == 1 ? 1536 * 2 / PAT_TILE : 1)
    k_csr_pat_ring(RingDev A, StepArgs s, const int *__restrict__ tiles, int ntl, int stage_bytes, int tbl_bytes) {
    constexpr int NT = PAT_TILE / R;  // threads
    extern __shared__ __align__(16) unsigned char rg_smem[];
    __shared__ uint64_t full[NS];
    __shared__ double red[NT / 32];
    if (s.done && *s.done) return;  // uniform, before any copy is issued
    const int lane = threadIdx.x & 31;
    const bool issuer = threadIdx.x < 32;
    if (threadIdx.x == 0) {
        for (int b = 0; b < NS; ++b) mbar_init(&full[b], 1);
        fence_mbar_init();
    }
    __syncthreads();
    // NS = 1: grid = tiles, one each
    const int nmine = NS == 1 ? 1 : ntl > (int)blockIdx.x ? (ntl - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
    auto tile_of = [&](int i) {
        const int q = (int)blockIdx.x + i * (int)gridDim.x;
        return tiles ? tiles[q] : q;
    };
    if (issuer)
        for (int i = 0; i < NS && i < nmine; ++i)
            ring_issue<WIDE>(A, s.x, tile_of(i), rg_smem + (size_t)(i % NS) * stage_bytes, &full[i % NS], lane, 0,
                             false);
    RingRows<R> cur;
    const int dot_src = !DOT ? 0 : s.dotv == s.x ? 1 : (HAS_R && s.dotv == s.r) ? 2 : 0;
    auto rows_of = [&](int i, RingRows<R> &q) {
        const int row0 = tile_of(i) * PAT_TILE;
        ring_load_rows<HAS_S2, HAS_R, DOT, R>(s.s2, s.r, s.dotv, row0, min(PAT_TILE, A.n - row0), q, dot_src);
    };
    if (nmine > 0) rows_of(0, cur);
    double acc = 0.0;
    for (int i = 0; i < nmine; ++i) {
        RingRows<R> nxt;
        if (NS > 1 && i + 1 < nmine) rows_of(i + 1, nxt);
        const int b = i % NS;
        const int row0 = tile_of(i) * PAT_TILE, nrows = min(PAT_TILE, A.n - row0);
        mbar_wait_sleep(&full[b], (uint32_t)((i / NS) & 1), NPC_RING_WAIT_NS);
        ring_tile<HAS_S2, HAS_R, DOT, R>(s, rg_smem + (size_t)b * stage_bytes, tbl_bytes, row0, nrows, cur, acc,
                                         dot_src);
        if (NS > 1) {
            cur = nxt;
            if (i + NS < nmine) {
                __syncthreads();  // every row of stage b summed: it can be refilled
                if (issuer)
                    ring_issue<WIDE>(A, s.x, tile_of(i + NS), rg_smem + (size_t)b * stage_bytes, &full[b], lane, 0,
                                     false);
            }
        }
    }
    if (DOT) {
        acc = block_sum<NT>(acc, red);
        if (threadIdx.x == 0) s.partials[blockIdx.x] = acc;
        if (NS > 1 && blockIdx.x == 0)  // persistent grid: the slots of the tiles beyond the grid read as 0
            for (int k = gridDim.x + threadIdx.x; k < ntl; k += NT) s.partials[k] = 0.0;
    }
}

// ---------------------------------------------------------------- two degrees per pass (L2 wavefront)
// Temporal blocking for the pattern form without any grid geometry: one launch computes s_j
// (step s1) and s_{j+1} (step s2) for every tile.  Work items are taken in ticket order (an
// atomic counter, so a taken item only ever waits on items taken before it): s_j of tile u,
// interleaved with s_{j+1} of tile u - L.  s_{j+1} of tile t reads s_j through its x windows,
// i.e. tiles deps[t].x .. deps[t].y; the CTA's warp 0 waits until those tiles' epoch flags show
// this launch (release/acquire), then copies them.  With the lag L larger than that reach plus
// the items in flight, the wait is normally already satisfied, and tile t's own values, s_{j-1}
// and r -- read by s_j of tile t only L tiles earlier -- come from L2 the second time: per two
// degrees HBM sees the matrix once and five vectors (s_{j-1}, s_{j-2}, r read; s_j, s_{j+1}
// written) instead of the matrix twice and eight vectors.  Same sums and epilogues as two
// k_csr_pat_ring launches: bitwise equal.  The ticket counter is never reset: every launch
// takes exactly 2 x tiles tickets (or none, when the PCG's done flag is set), so ticket / (2
// tiles) numbers the launch -- the epoch the flags carry (graph-replay safe, no host state).
struct WaveState {
    unsigned long long ticket;  // items taken over all launches: launch = ticket / (2 ntiles)
    unsigned pticket, pepoch;   // persistent form: items taken in this launch, launch number
};
#ifndef NPC_WAVE_HINTS
#define NPC_WAVE_HINTS 1
#endif
#ifndef NPC_WAVE_SLEEP_NS
#define NPC_WAVE_SLEEP_NS 500
#endif
#ifndef NPC_WAVE_NOWAIT  // A/B only (results may be wrong): no dependency wait
#define NPC_WAVE_NOWAIT 0
#endif
template <bool DOT>
__global__ void __launch_bounds__(PAT_THREADS, 1536 / PAT_THREADS)
    k_csr_pat_wave(RingDev A, StepArgs s1, StepArgs s2, int ntl, int L, int stage_bytes, int tbl_bytes,
                   WaveState *ws, unsigned *flags, const int2 *__restrict__ deps) {
    constexpr int R = 2;
    extern __shared__ __align__(16) unsigned char rg_smem[];
    __shared__ uint64_t full;
    __shared__ double red[PAT_THREADS / 32];
    __shared__ int sh_item;
    __shared__ unsigned sh_ep;
    if (s1.done && *s1.done) return;  // uniform, before a ticket is taken
    const int lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        mbar_init(&full, 1);
        fence_mbar_init();
        const unsigned long long tk = atomicAdd(&ws->ticket, 1ull), per = 2ull * (unsigned long long)ntl;
        sh_item = (int)(tk % per);
        sh_ep = (unsigned)(tk / per) + 1u;  // this launch's flag value
    }
    __syncthreads();
    const int item = sh_item;
    const unsigned ep = sh_ep;
    // item -> (role, tile): s_j of tiles 0 .. L'-1, then pairs (s_j of u, s_{j+1} of u - L), then
    // the remaining s_{j+1}
    const int Lp = min(L, ntl), n2 = max(0, ntl - L);
    int role, tile;
    if (item < Lp) {
        role = 0, tile = item;
    } else if (item - Lp < 2 * n2) {
        const int k = (item - Lp) >> 1;
        role = (item - Lp) & 1;
        tile = role == 0 ? L + k : k;
    } else {
        role = 1, tile = n2 + (item - Lp - 2 * n2);
    }
    const StepArgs &s = role == 0 ? s1 : s2;
    const double *x = role == 0 ? s1.x : s1.out;   // s_{j-1} / s_j
    const double *s2v = role == 0 ? s1.s2 : s1.x;  // s_{j-2} / s_{j-1}
    const int row0 = tile * PAT_TILE, nrows = min(PAT_TILE, A.n - row0);
    if (threadIdx.x < 32) {
        uint64_t pol = 0;
        if (NPC_WAVE_HINTS) {
            if (role == 0)
                asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
            else
                asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
        }
        // the copies that do not read s_j go out before the dependency wait
        const int4 d = ring_desc(A, tile, lane);
        const bool tail = __shfl_sync(0xffffffffu, d.z, 0) != 0;
        if (!tail) ring_issue_d(d, A, x, rg_smem, &full, lane, pol, NPC_WAVE_HINTS != 0, 1);
        if (role == 1 && !NPC_WAVE_NOWAIT) {  // s_j of every tile this one's x windows cover must be complete
            const int2 dp = deps[tile];
            bool ok;
            // relaxed loads, all in flight together (an acquire per load would serialise them),
            // then one acquire fence once every flag shows this launch
            do {
                ok = true;
                for (int base = dp.x; base <= dp.y; base += 256) {
                    unsigned f[8];
#pragma unroll
                    for (int k = 0; k < 8; ++k) {
                        const int t = base + lane + 32 * k;
                        f[k] = ep;
                        if (t <= dp.y) asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(f[k]) : "l"(flags + t));
                    }
#pragma unroll
                    for (int k = 0; k < 8; ++k) ok = ok && (int)(f[k] - ep) >= 0;
                }
                ok = __all_sync(0xffffffffu, ok);
                if (!ok) __nanosleep(NPC_WAVE_SLEEP_NS);
            } while (!ok);
            asm volatile("fence.acq_rel.gpu;" ::: "memory");
            asm volatile("fence.proxy.async.global;" ::: "memory");  // generic-proxy writes -> bulk copies
        }
        ring_issue_d(d, A, x, rg_smem, &full, lane, pol, NPC_WAVE_HINTS != 0, tail ? 0 : 2);
    }
    RingRows<R> cur;
    const bool dot = DOT && role == 1;
    if (dot)
        ring_load_rows<true, true, true, R>(s2v, s.r, s.dotv, row0, nrows, cur);
    else
        ring_load_rows<true, true, false, R>(s2v, s.r, nullptr, row0, nrows, cur);
    double acc = 0.0;
    mbar_wait_sleep(&full, 0, NPC_RING_WAIT_NS);
    if (dot)
        ring_tile<true, true, true, R>(s, rg_smem, tbl_bytes, row0, nrows, cur, acc);
    else
        ring_tile<true, true, false, R>(s, rg_smem, tbl_bytes, row0, nrows, cur, acc);
    if (DOT && role == 1) {
        acc = block_sum<PAT_THREADS>(acc, red);  // uniform over the CTA (role is)
        if (threadIdx.x == 0) s2.partials[tile] = acc;
    }
    __syncthreads();  // every row of this item stored
    if (threadIdx.x == 0) {
        if (role == 0) {
            asm volatile("fence.proxy.async.global;" ::: "memory");
            asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(flags + tile), "r"(ep) : "memory");
        }
    }
}

// Persistent form of the wave pass (NPC_WAVE_PERSIST=1 with NPC_CSR_WAVE=1): 3 CTAs per SM of
// 16 consumer warps + 1 producer warp.  The producer takes the NEXT item's ticket, publishes it
// and, for an s_{j+1} item, polls its dependency flags (and fences) while the consumers still
// sum the current item; once they release the stage it issues the next item's copies at once.
// So the acquire latency of the dependency check is off the critical path.  k_wave_begin resets
// the per-launch ticket and advances the epoch (one thread, before every launch).
__global__ void k_wave_begin(WaveState *ws) {
    ws->pticket = 0;
    ws->pepoch += 1;
}
template <bool DOT>
__global__ void __maxnreg__(40)
    k_csr_pat_wave_p(RingDev A, StepArgs s1, StepArgs s2, int ntl, int L, int tbl_bytes, WaveState *ws,
                     unsigned *flags, const int2 *__restrict__ deps) {
    constexpr int R = 2, NCW = PAT_THREADS / 32;
    extern __shared__ __align__(16) unsigned char rg_smem[];
    __shared__ uint64_t full, empty, info_bar[2];
    __shared__ int info[2][2];  // {role, tile} of items i (slot i % 2); role -1: no more items
    __shared__ double red[NCW];
    if (s1.done && *s1.done) return;  // uniform
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        mbar_init(&full, 1);
        mbar_init(&empty, NCW);
        mbar_init(&info_bar[0], 1);
        mbar_init(&info_bar[1], 1);
        fence_mbar_init();
    }
    __syncthreads();
    const unsigned ep = *reinterpret_cast<volatile unsigned *>(&ws->pepoch);
    const int per = 2 * ntl;
    auto map_item = [&](int item, int L, int &role, int &tile) {
        const int l0 = min(L, ntl), n2 = max(0, ntl - L);
        if (item < l0) {
            role = 0, tile = item;
        } else if (item - l0 < 2 * n2) {
            const int k = (item - l0) >> 1;
            role = (item - l0) & 1;
            tile = role == 0 ? L + k : k;
        } else {
            role = 1, tile = n2 + (item - l0 - 2 * n2);
        }
    };
    if (warp == NCW) {
        // ---------------- producer
        uint64_t pol0 = 0, pol1 = 0;
        if (NPC_WAVE_HINTS) {
            asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol0));
            asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol1));
        }
        for (int i = 0;; ++i) {
            int item = 0;
            if (lane == 0) item = (int)atomicAdd(&ws->pticket, 1u);
            item = __shfl_sync(0xffffffffu, item, 0);
            int role = -1, tile = 0;
            if (item < per) map_item(item, L, role, tile);
            if (lane == 0) {
                info[i & 1][0] = role;
                info[i & 1][1] = tile;
                mbar_arrive(&info_bar[i & 1]);
            }
            if (role < 0) break;  // the consumers leave on the published role
            const double *x = role == 0 ? s1.x : s1.out;
            const int4 d = ring_desc(A, tile, lane);
            if (role == 1) {  // s_j of the tiles this one's x windows cover: while the consumers sum
                const int2 dp = deps[tile];
                bool ok;
                do {
                    ok = true;
                    for (int base = dp.x; base <= dp.y; base += 256) {
                        unsigned f[8];
#pragma unroll
                        for (int k = 0; k < 8; ++k) {
                            const int t = base + lane + 32 * k;
                            f[k] = ep;
                            if (t <= dp.y) asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(f[k]) : "l"(flags + t));
                        }
#pragma unroll
                        for (int k = 0; k < 8; ++k) ok = ok && (int)(f[k] - ep) >= 0;
                    }
                    ok = __all_sync(0xffffffffu, ok);
                    if (!ok) __nanosleep(NPC_WAVE_SLEEP_NS);
                } while (!ok);
                asm volatile("fence.acq_rel.gpu;" ::: "memory");
                asm volatile("fence.proxy.async.global;" ::: "memory");
            }
            if (i > 0) mbar_wait(&empty, (uint32_t)((i - 1) & 1));  // the consumers left the stage
            ring_issue_d(d, A, x, rg_smem, &full, lane, role == 0 ? pol0 : pol1, NPC_WAVE_HINTS != 0, 0);
        }
    } else {
        // ---------------- consumers
        for (int i = 0;; ++i) {
            mbar_wait(&info_bar[i & 1], (uint32_t)((i >> 1) & 1));
            const int role = info[i & 1][0], tile = info[i & 1][1];
            if (role < 0) break;
            const StepArgs &s = role == 0 ? s1 : s2;
            const double *s2v = role == 0 ? s1.s2 : s1.x;
            const int row0 = tile * PAT_TILE, nrows = min(PAT_TILE, A.n - row0);
            RingRows<R> cur;
            const bool dot = DOT && role == 1;
            if (dot)
                ring_load_rows<true, true, true, R>(s2v, s.r, s.dotv, row0, nrows, cur);
            else
                ring_load_rows<true, true, false, R>(s2v, s.r, nullptr, row0, nrows, cur);
            mbar_wait_sleep(&full, (uint32_t)(i & 1), NPC_RING_WAIT_NS);
            double a = 0.0;
            if (dot)
                ring_tile<true, true, true, R>(s, rg_smem, tbl_bytes, row0, nrows, cur, a);
            else
                ring_tile<true, true, false, R>(s, rg_smem, tbl_bytes, row0, nrows, cur, a);
            if (dot) {  // this tile's partial, as block_sum<PAT_THREADS> (consumers only: named barrier 1)
                a = warp_sum(a);
                if (lane == 0) red[warp] = a;
                asm volatile("bar.sync 1, %0;" ::"r"(PAT_THREADS));
                if (warp == 0) {
                    double t = lane < NCW ? red[lane] : 0.0;
                    t = warp_sum(t);
                    if (lane == 0) s2.partials[tile] = t;
                }
            }
            if (role == 0) {  // every row stored -> the tile's flag
                asm volatile("bar.sync 1, %0;" ::"r"(PAT_THREADS));
                if (threadIdx.x == 0) {
                    asm volatile("fence.proxy.async.global;" ::: "memory");
                    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(flags + tile), "r"(ep) : "memory");
                }
            }
            if (dot) asm volatile("bar.sync 1, %0;" ::"r"(PAT_THREADS));  // red[] reused next item
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty);
        }
    }
}

class CsrOperator : public Operator {
  public:
    DevBuf rowptr, cols, vals;
    DevBuf codes, dict, dict_off, tptr, roff;  // coded form (see the file comment)
    bool coded = false;
    // pattern form (k_csr_pat_step): own values in `vals` (tile-ELL blocks), block pointers in
    // `tptr`, and per-row pattern ids + per-tile pattern tables here
    bool pattern = false;
    DevBuf pat, tbl, tbl_off;
    DevBuf tbl2, tbl2_off;  // staged kernel tables (k_csr_pat_stage)
    int xspan_max = 0, tbl2_max = 0;
    size_t smem_stage = 0;
    DevBuf rtbl, rdesc;      // ring kernel: per-tile tables and copy descriptors (k_csr_pat_ring)
    bool ring = false;
    int ring_ns = 1;         // stages per CTA (1: one tile per CTA; A/B NPC_RING_NS=2)
    int ring_rpt = 2;        // rows per thread (A/B NPC_RING_RPT=4)
    int ring_ctas = 0;       // resident CTAs per SM of the persistent form (queried at the first launch)
    int ring_stage = 0, ring_tbl_bytes = 0;
    long long ring_tbl_ints = 0;  // stored (deduplicated) ring-table words
    long long ring_desc_bytes = 0;  // descriptor bytes the kernels read per application
    int ring_dstride = 16;
    // two degrees per pass (k_csr_pat_wave): per-tile x-window reach, epoch flags, ticket state
    DevBuf wdeps, wflags, wstate;
    int wave_lag = 0, ring_span = 0;
    bool wave = false, wave_persist = false;
    struct PatTiles {  // a tile list split by kernel: staged / unstaged
        DevBuf staged, unstaged;
        int ns = 0, nu = 0;
        bool identity = false;  // staged == [0, ns): launch without a tile list
    } pt_all, pt_interior;
    DevBuf cvals;  // full CSR values for the cluster-resident kernels (pattern form only)
    const double *csr_vals() const { return pattern ? cvals.as<double>() : vals.as<double>(); }
    long long own_nnz = 0, tbl_total = 0;
    int tbl_max = 0;
    long long dict_total = 0;
    DevBuf tiles_interior, tiles_boundary;
    int ntiles = 0, n_interior = 0, n_boundary = 0;
    int vspan_max = 0, cspan_max = 0;
    size_t smem_bytes = 0;
    bool staged = true;
    long long nnz = 0;
    HaloPlan plan;
    HaloRuntime halo;
    bool multi = false;

    int num_partials() const override { return std::max(ntiles, 1); }

    double bytes_per_step(bool has_s2, bool has_r) const override {
        // values + column ids (or codes + dictionaries) + row pointers once, x once (perfect
        // gather reuse), write out, read s_{j-2} and r when present.
        double b = matrix_bytes() + 2.0 * 8.0 * n_local;
        if (has_s2) b += 8.0 * n_local;
        if (has_r) b += 8.0 * n_local;
        return b;
    }

    double matrix_bytes() const override {
        if (pattern && ring)  // own values (incl. ELL padding), pattern ids, shared tables, copy descriptors
            return (double)own_nnz * 8.0 + (double)n_local + (double)ring_tbl_ints * 4.0 + (double)ring_desc_bytes;
        if (pattern)  // own values (incl. ELL padding), pattern ids, tables, tile pointers
            return (double)own_nnz * 8.0 + (double)n_local + (double)tbl_total * 4.0 + (double)(ntiles + 1) * 8.0;
        if (coded)  // values + codes, dictionaries + their offsets, tile pointers, 16-bit row offsets
            return (double)nnz * 9.0 + (double)dict_total * 4.0 + (double)(ntiles + 1) * 8.0 +
                   (double)n_local * 2.0;
        return (double)nnz * 12.0 + (double)(n_local + 1) * 4.0;
    }

    template <bool ST, bool H2, bool HR, bool DT, bool GH>
    npc_status launch_t(const StepArgs &s, const int *tl, int nt, double *partials) {
        if (pattern) return launch_p<H2, HR, DT, GH>(s, tl, nt, partials);
        return coded ? launch_c<ST, H2, HR, DT, GH, true>(s, tl, nt, partials)
                     : launch_c<ST, H2, HR, DT, GH, false>(s, tl, nt, partials);
    }
    template <bool ST, bool H2, bool HR, bool DT, bool GH, bool CD>
    npc_status launch_c(const StepArgs &s, const int *tl, int nt, double *partials) {
        if (nt <= 0) return NPC_SUCCESS;
        CsrDev A{rowptr.as<int>(), cols.as<int>(), vals.as<double>(), n_local,
                 GH ? halo.ghost_buf.as<double>() : nullptr, codes.as<unsigned char>(), dict.as<int>(),
                 dict_off.as<int>(), tptr.as<int>(), roff.as<unsigned short>()};
        StepArgs a = s;
        a.partials = partials;
        auto kern = k_csr_step<ST, H2, HR, DT, GH, CD>;
        size_t sm = ST ? smem_bytes : 0;
        if (sm > 48 * 1024) NPC_TRY(allow_max_dynamic_smem(kern));
        kern<<<nt, CD ? CSR_TILE_CODED : CSR_TILE, sm, ctx->stream>>>(A, a, tl, vspan_max);
        NPC_LAUNCH_CHECK();
        return NPC_SUCCESS;
    }

    template <bool H2, bool HR, bool DT, bool GH>
    npc_status launch_p(const StepArgs &s, const int *tl, int nt, double *partials) {
        if (nt <= 0) return NPC_SUCCESS;
        PatDev A{vals.as<double>(), tptr.as<int>(), pat.as<unsigned char>(), tbl.as<int>(), tbl_off.as<int>(),
                 n_local, GH ? halo.ghost_buf.as<double>() : nullptr, nullptr, nullptr};
        StepArgs a = s;
        a.partials = partials;
        auto kern = k_csr_pat_step<H2, HR, DT, GH>;
        if (smem_bytes > 48 * 1024) NPC_TRY(allow_max_dynamic_smem(kern));
        kern<<<nt, PAT_TILE, smem_bytes, ctx->stream>>>(A, a, tl, vspan_max, tbl_max);
        NPC_LAUNCH_CHECK();
        return NPC_SUCCESS;
    }

    // opt every pattern-form kernel variant into large dynamic shared memory up front
    template <bool H2, bool HR, bool DT>
    npc_status prepare3() {
        NPC_TRY(allow_max_dynamic_smem(k_csr_pat_stage<H2, HR, DT>));
        NPC_TRY(allow_max_dynamic_smem(k_csr_pat_ring<H2, HR, DT, 1, 2>));
        NPC_TRY(allow_max_dynamic_smem(k_csr_pat_ring<H2, HR, DT, 1, 2, 1>));
        NPC_TRY(allow_max_dynamic_smem(k_csr_pat_ring<H2, HR, DT, 2, 2>));
        NPC_TRY(allow_max_dynamic_smem(k_csr_pat_ring<H2, HR, DT, 1, 4>));
        NPC_TRY(allow_max_dynamic_smem(k_csr_pat_ring<H2, HR, DT, 2, 4>));
        NPC_TRY(allow_max_dynamic_smem(k_csr_pat_step<H2, HR, DT, false>));
        return allow_max_dynamic_smem(k_csr_pat_step<H2, HR, DT, true>);
    }
    npc_status prepare_kernels() {
        NPC_TRY(allow_max_dynamic_smem(k_csr_pat_wave<true>));
        NPC_TRY(allow_max_dynamic_smem(k_csr_pat_wave<false>));
        NPC_TRY(allow_max_dynamic_smem(k_csr_pat_wave_p<true>));
        NPC_TRY(allow_max_dynamic_smem(k_csr_pat_wave_p<false>));
        NPC_TRY((prepare3<true, true, true>()));
        NPC_TRY((prepare3<true, true, false>()));
        NPC_TRY((prepare3<true, false, true>()));
        NPC_TRY((prepare3<true, false, false>()));
        NPC_TRY((prepare3<false, true, true>()));
        NPC_TRY((prepare3<false, true, false>()));
        NPC_TRY((prepare3<false, false, true>()));
        return prepare3<false, false, false>();
    }

    template <bool H2, bool HR, bool DT>
    npc_status launch_stage(const StepArgs &s, const int *tl, int nt, double *partials) {
        if (nt <= 0) return NPC_SUCCESS;
        PatDev A{vals.as<double>(), tptr.as<int>(), pat.as<unsigned char>(), tbl.as<int>(), tbl_off.as<int>(),
                 n_local, nullptr, tbl2.as<int>(), tbl2_off.as<int>()};
        StepArgs a = s;
        a.partials = partials;
        auto kern = k_csr_pat_stage<H2, HR, DT>;
        if (smem_stage > 48 * 1024) NPC_TRY(allow_max_dynamic_smem(kern));
        kern<<<nt, PAT_THREADS, smem_stage, ctx->stream>>>(A, a, tl, vspan_max, xspan_max);
        NPC_LAUNCH_CHECK();
        return NPC_SUCCESS;
    }
    template <bool H2, bool HR, bool DT, int NS, int R, int WIDE = 0>
    npc_status launch_ring_ns(const StepArgs &s, const int *tl, int nt, double *partials) {
        RingDev A{vals.as<double>(), rtbl.as<int>(), pat.as<unsigned char>(), rdesc.as<int4>(), n_local, ring_dstride};
        StepArgs a = s;
        a.partials = partials;
        auto kern = k_csr_pat_ring<H2, HR, DT, NS, R, WIDE>;
        const size_t sm = (size_t)NS * ring_stage;
        int grid = nt;
        if (NS > 1) {
            if (ring_ctas == 0) {  // resident CTAs per SM at this stage size
                int occ = 0;
                NPC_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, PAT_TILE / R, sm));
                ring_ctas = std::max(1, occ);
            }
            grid = std::min(nt, ctx->num_sms * ring_ctas);
        }
        kern<<<grid, PAT_TILE / R, sm, ctx->stream>>>(A, a, tl, nt, ring_stage, ring_tbl_bytes);
        NPC_LAUNCH_CHECK();
        return NPC_SUCCESS;
    }
    template <bool H2, bool HR, bool DT>
    npc_status launch_ring(const StepArgs &s, const int *tl, int nt, double *partials) {
        if (nt <= 0) return NPC_SUCCESS;
        if (ring_dstride > 16) return launch_ring_ns<H2, HR, DT, 1, 2, 1>(s, tl, nt, partials);  // > 15 copies
        if (ring_rpt == 4)
            return ring_ns == 2 ? launch_ring_ns<H2, HR, DT, 2, 4>(s, tl, nt, partials)
                                : launch_ring_ns<H2, HR, DT, 1, 4>(s, tl, nt, partials);
        return ring_ns == 2 ? launch_ring_ns<H2, HR, DT, 2, 2>(s, tl, nt, partials)
                            : launch_ring_ns<H2, HR, DT, 1, 2>(s, tl, nt, partials);
    }
    npc_status launch_stage_any(const StepArgs &s, const int *tl, int nt, double *partials) {
        const bool h2 = s.s2 != nullptr, hr = s.r != nullptr, dt = s.dotv != nullptr;
        if (ring) {
            if (h2 && hr && dt) return launch_ring<true, true, true>(s, tl, nt, partials);
            if (h2 && hr) return launch_ring<true, true, false>(s, tl, nt, partials);
            if (h2 && dt) return launch_ring<true, false, true>(s, tl, nt, partials);
            if (h2) return launch_ring<true, false, false>(s, tl, nt, partials);
            if (hr && dt) return launch_ring<false, true, true>(s, tl, nt, partials);
            if (hr) return launch_ring<false, true, false>(s, tl, nt, partials);
            if (dt) return launch_ring<false, false, true>(s, tl, nt, partials);
            return launch_ring<false, false, false>(s, tl, nt, partials);
        }
        if (h2 && hr && dt) return launch_stage<true, true, true>(s, tl, nt, partials);
        if (h2 && hr) return launch_stage<true, true, false>(s, tl, nt, partials);
        if (h2 && dt) return launch_stage<true, false, true>(s, tl, nt, partials);
        if (h2) return launch_stage<true, false, false>(s, tl, nt, partials);
        if (hr && dt) return launch_stage<false, true, true>(s, tl, nt, partials);
        if (hr) return launch_stage<false, true, false>(s, tl, nt, partials);
        if (dt) return launch_stage<false, false, true>(s, tl, nt, partials);
        return launch_stage<false, false, false>(s, tl, nt, partials);
    }
    // A tile set of the pattern form: staged tiles first (their partial slots first), then the
    // rest through k_csr_pat_step.  x must be 16-byte aligned for the window copies; otherwise
    // every tile takes k_csr_pat_step.
    npc_status launch_pattern_set(const StepArgs &s, const PatTiles &t, double *partials) {
        const bool aligned = ((uintptr_t)s.x & 15) == 0;
        const int *sl = t.identity ? nullptr : t.staged.as<int>();
        if (aligned)
            NPC_TRY(launch_stage_any(s, sl, t.ns, partials));
        else if (t.ns > 0)
            NPC_TRY(launch(s, t.staged.as<int>(), t.ns, partials, false));
        return launch(s, t.unstaged.as<int>(), t.nu, partials ? partials + t.ns : nullptr, false);
    }

    template <bool H2, bool HR, bool DT>
    npc_status launch_g(const StepArgs &s, const int *tl, int nt, double *partials, bool ghost) {
        if (staged) {
            if (ghost) return launch_t<true, H2, HR, DT, true>(s, tl, nt, partials);
            return launch_t<true, H2, HR, DT, false>(s, tl, nt, partials);
        }
        if (ghost) return launch_t<false, H2, HR, DT, true>(s, tl, nt, partials);
        return launch_t<false, H2, HR, DT, false>(s, tl, nt, partials);
    }

    npc_status launch(const StepArgs &s, const int *tl, int nt, double *partials, bool ghost) {
        const bool h2 = s.s2 != nullptr, hr = s.r != nullptr, dt = s.dotv != nullptr;
        if (h2 && hr && dt) return launch_g<true, true, true>(s, tl, nt, partials, ghost);
        if (h2 && hr) return launch_g<true, true, false>(s, tl, nt, partials, ghost);
        if (h2 && dt) return launch_g<true, false, true>(s, tl, nt, partials, ghost);
        if (h2) return launch_g<true, false, false>(s, tl, nt, partials, ghost);
        if (hr && dt) return launch_g<false, true, true>(s, tl, nt, partials, ghost);
        if (hr) return launch_g<false, true, false>(s, tl, nt, partials, ghost);
        if (dt) return launch_g<false, false, true>(s, tl, nt, partials, ghost);
        return launch_g<false, false, false>(s, tl, nt, partials, ghost);
    }

    bool supports_step2() const override { return pattern && ring && wave && ring_ns == 1; }
    int num_partials2() const override { return std::max(ntiles, 1); }
    double bytes_per_step2() const override { return matrix_bytes() + 5.0 * 8.0 * n_local; }
    npc_status step2(const StepArgs &s1, const StepArgs &s2) override {
        if (!s1.x || !s1.s2 || !s1.r || !s2.r || !s1.out || !s2.out) {
            set_error("CSR step2: x, s_{j-2}, r and both outputs are required");
            return NPC_ERR_INVALID_ARGUMENT;
        }
        if (((uintptr_t)s1.x & 15) || ((uintptr_t)s1.out & 15)) {  // window copies need 16-byte aligned inputs
            NPC_TRY(step(s1));
            StepArgs t = s2;
            t.x = s1.out;
            t.s2 = s1.x;
            return step(t);
        }
        RingDev A{vals.as<double>(), rtbl.as<int>(), pat.as<unsigned char>(), rdesc.as<int4>(), n_local, ring_dstride};
        if (wave_persist) {
            k_wave_begin<<<1, 1, 0, ctx->stream>>>(wstate.as<WaveState>());
            NPC_LAUNCH_CHECK();
            auto gop = [&](auto kern) -> npc_status {
                const int grid = std::min(2 * ntiles, ctx->num_sms * (1536 / PAT_THREADS));
                kern<<<grid, PAT_THREADS + 32, ring_stage, ctx->stream>>>(A, s1, s2, ntiles, wave_lag, ring_tbl_bytes,
                                                                         wstate.as<WaveState>(), wflags.as<unsigned>(),
                                                                         wdeps.as<int2>());
                NPC_LAUNCH_CHECK();
                return NPC_SUCCESS;
            };
            return s2.dotv ? gop(k_csr_pat_wave_p<true>) : gop(k_csr_pat_wave_p<false>);
        }
        auto go = [&](auto kern) -> npc_status {
            kern<<<2 * ntiles, PAT_THREADS, ring_stage, ctx->stream>>>(A, s1, s2, ntiles, wave_lag, ring_stage,
                                                                      ring_tbl_bytes, wstate.as<WaveState>(),
                                                                      wflags.as<unsigned>(), wdeps.as<int2>());
            NPC_LAUNCH_CHECK();
            return NPC_SUCCESS;
        };
        return s2.dotv ? go(k_csr_pat_wave<true>) : go(k_csr_pat_wave<false>);
    }

    SmallCsrPlan small;  // cluster-resident polynomial (single rank, n <= 16384)
    bool supports_fused_poly() const override {
        return small.cl_size > 0 && !getenv("NPC_NO_CLUSTER");
    }
    npc_status apply_poly_fused(const double *r, double *z, const double *coef_dev, int k, double tb,
                                const double *dotv, double *partials, int *nparts, const int *done) override {
        SmallCsrDev A{rowptr.as<int>(), cols.as<int>(), csr_vals(), n_local, small.R, small.nnz_cta};
        if (dotv && nparts) *nparts = small.cl_size;
        return launch_csr_poly_cluster(ctx, A, small.cl_size, small.threads, small.smem, r, z, coef_dev, k, tb, dotv,
                                       partials, done);
    }

    bool supports_fused_lanczos() const override { return supports_fused_pcg(); }
    npc_status lanczos_fused(const double *v0, int m, double *alphas, double *betas, int *steps) override {
        SmallCsrDev A{rowptr.as<int>(), cols.as<int>(), csr_vals(), n_local, small.R, small.nnz_cta};
        return launch_csr_lanczos_cluster(ctx, A, small, v0, m, alphas, betas, steps);
    }
    bool supports_fused_pcg() const override {
        return supports_fused_poly() && small.smem_pcg > 0;
    }
    npc_status pcg_fused(const double *b, double *x, const double *coef_dev, int k, double tb, int use_poly,
                         double tol2b, int maxit, ClusterPcgOut *out, double *history) override {
        SmallCsrDev A{rowptr.as<int>(), cols.as<int>(), csr_vals(), n_local, small.R, small.nnz_cta};
        return launch_csr_pcg_cluster(ctx, A, small, b, x, coef_dev, k, tb, use_poly, tol2b, maxit, out, history);
    }

    npc_status step(const StepArgs &s) override {
        if (n_local == 0 && !multi) return NPC_SUCCESS;
        // a rank without rows still joins the halo exchange and writes zero dot partials
        // (num_partials() >= 1 of them are read)
        const bool zero_parts = multi && ntiles == 0 && s.dotv;
        if (pattern) {
            if (!multi || ctx->nranks == 1) {
                if (zero_parts) return launch_fill(ctx, s.partials, 0.0, num_partials());
                return launch_pattern_set(s, pt_all, s.partials);
            }
            NPC_TRY(halo_start(ctx, plan, halo, s.x));
            NPC_TRY(launch_pattern_set(s, pt_interior, s.partials));
            NPC_TRY(halo_wait(ctx, halo));
            if (zero_parts) return launch_fill(ctx, s.partials, 0.0, num_partials());
            return launch(s, tiles_boundary.as<int>(), n_boundary, s.partials ? s.partials + n_interior : nullptr,
                          true);
        }
        if (zero_parts) {
            if (ctx->nranks > 1) {
                NPC_TRY(halo_start(ctx, plan, halo, s.x));
                NPC_TRY(halo_wait(ctx, halo));
            }
            return launch_fill(ctx, s.partials, 0.0, num_partials());
        }
        // single rank, or a 1-rank distributed context (no halo; with more ranks the exchange
        // is collective for the local transport even when this rank's plan is empty)
        if (!multi || ctx->nranks == 1) return launch(s, nullptr, ntiles, s.partials, false);
        // halo of x -> ghost slots on the comm stream, interior tiles meanwhile
        NPC_TRY(halo_start(ctx, plan, halo, s.x));
        NPC_TRY(launch(s, tiles_interior.as<int>(), n_interior, s.partials, false));
        NPC_TRY(halo_wait(ctx, halo));
        return launch(s, tiles_boundary.as<int>(), n_boundary, s.partials ? s.partials + n_interior : nullptr, true);
    }
};

// Validate CSR invariants: rowptr monotone from 0, column ids in range and
// strictly ascending within a row, values finite.
static npc_status validate_csr(int n, long long ncols, const int *rowptr, const int *colidx, const double *vals) {
    if (rowptr[0] != 0) {
        set_error("CSR: rowptr[0] = %d (must be 0)", rowptr[0]);
        return NPC_ERR_DIMENSION;
    }
    for (int i = 0; i < n; ++i)  // monotone first: the row ranges below are then valid
        if (rowptr[i + 1] < rowptr[i]) {
            set_error("CSR: rowptr not monotone at row %d", i);
            return NPC_ERR_DIMENSION;
        }
    // rows checked in parallel chunks; the first offending row (lowest index) is reported
    std::vector<long long> bad(64, -1);
    std::vector<int> why(64, 0);
    host_parallel_for(n, [&](long long b, long long e, int t) {
        for (long long i = b; i < e; ++i)
            for (int p = rowptr[i]; p < rowptr[i + 1]; ++p) {
                int w = 0;
                if (colidx[p] < 0 || colidx[p] >= ncols) w = 1;
                else if (p > rowptr[i] && colidx[p] <= colidx[p - 1]) w = 2;
                else if (!std::isfinite(vals[p])) w = 3;
                if (w) {
                    bad[t] = i;
                    why[t] = w;
                    return;
                }
            }
    });
    for (int t = 0; t < 64; ++t)
        if (bad[t] >= 0) {
            const char *msg[] = {"", "column out of range", "columns not strictly ascending", "non-finite value"};
            set_error("CSR: %s in row %lld", msg[why[t]], bad[t]);
            return NPC_ERR_DIMENSION;
        }
    return NPC_SUCCESS;
}

npc_status validate_csr_desc(Context *ctx, const npc_operator_desc *d) {
    if (!d->rowptr || (!d->colidx && d->n_local > 0) || (!d->vals && d->n_local > 0)) {
        set_error("CSR: null array");
        return NPC_ERR_INVALID_ARGUMENT;
    }
    (void)ctx;
    return validate_csr(d->n_local, d->n_global, d->rowptr, d->colidx, d->vals);
}

// Convert global column ids to local ids ([0,n) owned, n + ghost slot otherwise).
npc_status localize_columns(Context *ctx, const npc_operator_desc *d, HaloPlan &plan, std::vector<int> &local_cols) {
    const int n = d->n_local;
    const long long nnz = d->rowptr[n];
    local_cols.resize((size_t)nnz);
    if (!ctx->distributed()) {
        host_parallel_for(nnz, [&](long long b, long long e, int) {
            std::memcpy(local_cols.data() + b, d->colidx + b, sizeof(int) * (size_t)(e - b));
        });
        return NPC_SUCCESS;
    }
    // partition: gather every rank's row_begin (collective)
    std::vector<long long> starts;
    NPC_TRY(ctx->tr->allgather_i64(ctx, d->row_begin, starts));
    starts.push_back(d->n_global);
    for (int q = 0; q < ctx->nranks; ++q)
        if (starts[q + 1] < starts[q]) {
            set_error("row blocks must be assigned to ranks in global row order");
            return NPC_ERR_DIMENSION;
        }
    NPC_TRY(halo_plan_local(n, d->rowptr, d->colidx, ctx->nranks, starts.data(), ctx->rank, plan));
    NPC_TRY(halo_plan_exchange(ctx, d->row_begin, plan));
    const long long r0 = d->row_begin, r1 = d->row_begin + n;
    for (long long p = 0; p < nnz; ++p) {
        long long c = d->colidx[p];
        if (c >= r0 && c < r1)
            local_cols[p] = (int)(c - r0);
        else {
            auto it = std::lower_bound(plan.ghost_ids.begin(), plan.ghost_ids.end(), c);
            local_cols[p] = n + (int)(it - plan.ghost_ids.begin());
        }
    }
    return NPC_SUCCESS;
}


// Host side of the pattern form.  Returns false (caller falls back to the coded/plain form)
// when a tile has more than 256 distinct patterns, a table longer than PAT_TBL_MAX words, a row
// with more than 256 own values, ELL padding above 1/8 of the own values, or a block larger
// than the shared-memory budget.
struct PatHost {
    std::unique_ptr<double[]> vals;  // own values, tile-ELL blocks (own_nnz + 8 padding)
    std::vector<int> tptr, tbl, tbl_off;
    std::vector<unsigned char> pat;
    int vspan_max = 0, tbl_max = 0;
    long long own_nnz = 0;  // stored values, padding included
    // staged kernel: per-tile table [nwin, entry offset, npat, 0 | nwin x {ga, len, sbase, tail}
    // | npat + 1 entry starts | (pad to 4) | entries {xb, vb, o, pos}], and which tiles stage
    std::vector<int> tbl2, tbl2_off;
    std::vector<char> stage;
    int xspan_max = 0, tbl2_max = 0;
    // ring kernel (k_csr_pat_ring): per-tile tables (16-byte aligned), RING_MAXD int4 copy
    // descriptors per tile, the stage size and its table region; ring = every staged tile has one
    std::vector<int> rtbl, rdesc, rdeps;
    int ring_stage = 0, ring_tbl_bytes = 0, ring_span = 0, ring_dstride = 16;
    bool ring = false;
};

// x windows + decoded entries of one tile for k_csr_pat_stage (see there).  pstart/pent: the
// tile's patterns as built by build_pattern.  Returns the table, or an empty vector when the
// tile's windows do not fit the shared-memory budget (it then runs k_csr_pat_step).
static std::vector<int> pattern_stage_table(int n, int row0, int nrows, int own_block, const std::vector<int> &pstart,
                                            const std::vector<int> &pent, int *xspan) {
    const int nrs = (nrows + 1) & ~1;  // column stride of the tile's own block (even)
    const int np = (int)pstart.size() - 1;
    std::vector<int> offs(1, 0);  // offset 0 always: the epilogue's x[row] comes from its window
    for (int w : pent) offs.push_back((w & 1) ? (w >> 9) : (w >> 1));
    std::sort(offs.begin(), offs.end());
    offs.erase(std::unique(offs.begin(), offs.end()), offs.end());
    struct Win { long long a, b; };
    std::vector<Win> win;
    for (int o : offs) {  // [row0 + o, row0 + o + nrows) clipped to the owned x, merged
        const long long a = std::max<long long>(0, (long long)row0 + o),
                        b = std::min<long long>(n, (long long)row0 + o + nrows);
        if (a >= b) continue;
        if (!win.empty() && a <= win.back().b + 64)
            win.back().b = std::max(win.back().b, b);
        else
            win.push_back({a, b});
    }
    std::vector<int> t(4, 0), wdesc;
    int sb = 0;
    for (auto &w : win) {  // TMA part [ga, ga + len) even-aligned; an odd last element as a tail
        const long long ga = w.a & ~1LL;
        long long bt = (w.b + 1) & ~1LL;
        int tail = 0;
        if (bt > n) {
            bt = w.b - 1;
            tail = 1;
        }
        const int len = (int)(bt - ga);
        wdesc.insert(wdesc.end(), {(int)ga, len, sb, tail});
        sb += (len + tail + 1) & ~1;
    }
    *xspan = sb;
    t[0] = (int)win.size();
    t.insert(t.end(), wdesc.begin(), wdesc.end());
    const int sidx = (int)t.size();
    t.resize(sidx + np + 1);
    while (t.size() % 4) t.push_back(0);
    t[1] = (int)t.size();
    t[2] = np;
    {  // header slot 3: x base of offset 0 (x[row0 + lr] = sx[t[3] + lr])
        int wi = 0;
        while (wi + 1 < (int)win.size() && win[wi + 1].a <= row0) ++wi;
        t[3] = wdesc[4 * wi + 2] + (row0 - wdesc[4 * wi]);
    }
    for (int q = 0; q < np; ++q) {
        t[sidx + q] = (int)(t.size() - t[1]) / 4;
        int k = 0;
        for (int e = pstart[q]; e < pstart[q + 1]; ++e) {
            const int w = pent[e];
            const int o = (w & 1) ? (w >> 9) : (w >> 1);
            const long long c0 = (long long)row0 + o;  // column of the tile's first row
            int wi = 0;
            while (wi + 1 < (int)win.size() && win[wi + 1].a <= std::max<long long>(c0, 0)) ++wi;
            const int xb = wdesc[4 * wi + 2] + (int)(c0 - wdesc[4 * wi]);
            if (w & 1) {
                const int pos = (w >> 1) & 255;
                t.insert(t.end(), {xb, pos * nrs + o, o, pos});
            } else {
                t.insert(t.end(), {xb, k * nrs, 0, 0});
                ++k;
            }
        }
    }
    t[sidx + np] = (int)(t.size() - t[1]) / 4;
    if ((size_t)own_block * 8 + (size_t)sb * 8 + t.size() * 4 > (size_t)PAT_STAGE_SMEM) return {};
    return t;
}

// Ring-kernel table of one staged tile (see k_csr_pat_ring).  tb: the tile's pattern table as
// built by build_pattern ([np + 1 starts][entry words]); prow: the pattern id of each row.
// Shared-memory stage: [table][pattern ids][D], D = own-value columns (column p preceded by its
// gap G_p: values of column p of the previous tile's last G_p rows), far mirror windows, x
// windows.  Copies carry a region (0 table, 1 pattern ids, 2 D in doubles) fixed up once the
// table region's size is known.  Returns false when the tile needs more copies than a
// descriptor holds or a mirror the layout cannot address (the operator then keeps
// k_csr_pat_stage).
#ifndef NPC_AB_NOZWIN
#define NPC_AB_NOZWIN 0
#endif
struct RingCopy {
    int kind, region, dst, src, bytes;  // kind: 0 vals, 1 x, 2 table, 3 pattern ids, 4 x tail
};
struct RingTile {
    std::vector<int> tbl;
    std::vector<RingCopy> cp;
    int dbl = 0;
    int dep_lo = 0, dep_hi = -1;  // tiles of x the tile's windows cover (two-degree pass)
};

static bool pattern_ring_table(int n, int t, const std::vector<int> &tptr, const std::vector<int> &twidth,
                               const std::vector<int> &tb, const unsigned char *prow, RingTile &rt) {
    const int T = PAT_TILE, r0 = t * T, nr = std::min(T, n - r0), nrs = (nr + 1) & ~1, W = twidth[t];
    const int np = tb[0] - 1;
    std::vector<int> lmin((size_t)np, INT_MAX), lmax((size_t)np, -1);
    for (int lr = 0; lr < nr; ++lr) {
        const int q = prow[lr];
        lmin[q] = std::min(lmin[q], lr);
        lmax[q] = std::max(lmax[q], lr);
    }
    // x windows: [r0 + o, r0 + o + nr) for every distinct offset, clipped and merged
    std::vector<int> offs(1, 0);
    for (int e = np + 1; e < (int)tb.size(); ++e) offs.push_back((tb[e] & 1) ? (tb[e] >> 9) : (tb[e] >> 1));
    std::sort(offs.begin(), offs.end());
    offs.erase(std::unique(offs.begin(), offs.end()), offs.end());
    struct Win { long long a, b; };
    std::vector<Win> win;
    for (int o : offs) {
        const long long a = std::max<long long>(0, (long long)r0 + o), b = std::min<long long>(n, (long long)r0 + o + nr);
        if (a >= b) continue;
        if (!win.empty() && a <= win.back().b + 64)
            win.back().b = std::max(win.back().b, b);
        else
            win.push_back({a, b});
    }
    struct XW { int ga, len, sb, tail; };
    std::vector<XW> xw;
    int xs = 0;
    for (auto &w : win) {
        const long long ga = w.a & ~1LL;
        long long bt = (w.b + 1) & ~1LL;
        int tail = 0;
        if (bt > n) bt = w.b - 1, tail = 1;
        xw.push_back({(int)ga, (int)(bt - ga), xs, tail});
        xs += ((int)(bt - ga) + tail + 1) & ~1;
    }
    auto xwin_of = [&](long long c) {
        int wi = 0;
        while (wi + 1 < (int)win.size() && win[wi + 1].a <= std::max<long long>(c, 0)) ++wi;
        return wi;
    };
    // mirror classes: 0 in tile / near (column gap), 1 far (window)
    std::vector<int> G((size_t)W, 0);
    struct Far { long long lo, hi; int pos; };
    std::vector<Far> far;
    std::vector<char> cls(tb.size(), 0);
    for (int q = 0; q < np; ++q)
        for (int e = tb[q]; e < tb[q + 1]; ++e) {
            const int w = tb[e];
            if (!(w & 1)) continue;
            const int o = w >> 9, pos = (w >> 1) & 255;
            const long long cmin = (long long)r0 + lmin[q] + o, cmax = (long long)r0 + lmax[q] + o;
            if (cmin >= r0) {
                if (pos >= W) return false;
            } else if (r0 - cmin <= RING_GAP_MAX && pos < W && t > 0 && pos < twidth[t - 1]) {
                G[pos] = std::max(G[pos], (int)(r0 - cmin));
            } else if (cmax < r0) {
                cls[e] = 1;
                far.push_back({cmin, cmax, pos});
            } else {
                return false;
            }
        }
    for (int &g : G) g = (g + 1) & ~1;
    std::sort(far.begin(), far.end(), [](const Far &a, const Far &b) { return a.pos != b.pos ? a.pos < b.pos : a.lo < b.lo; });
    std::vector<Far> fw;  // merged far windows, [lo, hi) even-aligned
    for (auto &f : far) {
        if (!fw.empty() && fw.back().pos == f.pos && f.lo <= fw.back().hi + 64)
            fw.back().hi = std::max(fw.back().hi, (f.hi + 2) & ~1LL);
        else
            fw.push_back({f.lo & ~1LL, (f.hi + 2) & ~1LL, f.pos});
    }
    // D layout
    std::vector<int> col((size_t)W);
    int off = 0;
    for (int p = 0; p < W; ++p) {
        off += G[p];
        col[p] = off;
        off += nrs;
    }
    std::vector<int> fwb(fw.size());
    for (size_t k = 0; k < fw.size(); ++k) fwb[k] = off, off += (int)(fw[k].hi - fw[k].lo);
    const int xbase = off;
    rt.dbl = off + xs;
    // copies
    rt.cp.clear();
    rt.cp.push_back({2, 0, 0, -1, 0});                     // table (source and size filled below)
    rt.cp.push_back({3, 1, 0, r0, (nr + 15) & ~15});       // pattern ids
    for (int p = 0; p < W;) {                              // own columns, in runs without gaps
        int p1 = p;
        while (p1 + 1 < W && G[p1 + 1] == 0) ++p1;
        rt.cp.push_back({0, 2, col[p], tptr[t] + p * nrs, (p1 - p + 1) * nrs * 8});
        p = p1 + 1;
    }
    for (int p = 0; p < W; ++p)  // gaps: column p of the previous (full) tile's last G_p rows
        if (G[p]) rt.cp.push_back({0, 2, col[p] - G[p], tptr[t - 1] + p * T + (T - G[p]), G[p] * 8});
    for (size_t k = 0; k < fw.size(); ++k)  // far windows, one copy per source tile
        for (long long c = fw[k].lo; c < fw[k].hi && !NPC_AB_NOZWIN;) {
            const int tj = (int)(c / T);
            const long long ce = std::min<long long>(fw[k].hi, (long long)(tj + 1) * T);
            if (fw[k].pos < twidth[tj])
                rt.cp.push_back({0, 2, fwb[k] + (int)(c - fw[k].lo), tptr[tj] + fw[k].pos * T + (int)(c - (long long)tj * T),
                                 (int)(ce - c) * 8});
            c = ce;
        }
    rt.dep_lo = INT_MAX, rt.dep_hi = -1;
    for (auto &w : xw) {
        // A/B only (results wrong): drop the x windows that do not contain the tile's own rows
        if (NPC_AB_NOZWIN && (w.ga + w.len <= r0 || w.ga >= r0 + nr)) continue;
        if (w.len) rt.cp.push_back({1, 2, xbase + w.sb, w.ga, w.len * 8});
        if (w.tail) rt.cp.push_back({4, 2, xbase + w.sb + w.len, w.ga + w.len, 0});
        if (w.len + w.tail > 0) {
            rt.dep_lo = std::min(rt.dep_lo, w.ga / T);
            rt.dep_hi = std::max(rt.dep_hi, (w.ga + w.len + w.tail - 1) / T);
        }
    }
    if ((int)rt.cp.size() > RING_MAXD - 1) return false;
    // table: [np, entry start, x0 base, nrs][np + 1 starts (entries)][pad][entries {xb, vb}]
    std::vector<int> &o = rt.tbl;
    o.assign(4, 0);
    o[0] = np;
    o[3] = nrs;
    {
        const int wi = xwin_of(r0);
        o[2] = 8 * (xbase + xw[wi].sb + (r0 - xw[wi].ga));
    }
    const int sidx = 4;
    o.resize(sidx + np + 1);
    if (o.size() & 1) o.push_back(0);
    o[1] = (int)o.size();
    for (int q = 0; q < np; ++q) {
        o[sidx + q] = (int)(o.size() - o[1]) / 2;
        int k = 0;
        for (int e = tb[q]; e < tb[q + 1]; ++e) {
            const int w = tb[e];
            const int of = (w & 1) ? (w >> 9) : (w >> 1);
            const long long c0 = (long long)r0 + of;
            const int wi = xwin_of(c0);
            const int xb = xbase + xw[wi].sb + (int)(c0 - xw[wi].ga);
            int vb;
            if (!(w & 1)) {
                vb = col[k++];
            } else if (!cls[e]) {
                vb = col[(w >> 1) & 255] + of;
            } else {
                const int pos = (w >> 1) & 255;
                const long long cmin = (long long)r0 + lmin[q] + of;
                size_t f = 0;
                while (!(fw[f].pos == pos && fw[f].lo <= cmin && cmin < fw[f].hi)) ++f;
                vb = fwb[f] + (int)((long long)r0 + of - fw[f].lo);
            }
            o.push_back(8 * xb);  // byte offsets into D
            o.push_back(8 * vb);
        }
    }
    o[sidx + np] = (int)(o.size() - o[1]) / 2;
    while (o.size() % 4) o.push_back(0);
    rt.cp[0].bytes = (int)o.size() * 4;
    return true;
}

// Phase wall times of operator creation on stderr (NPC_CREATE_TIMES=1; profiling only).
struct CreateTimer {
    bool on = getenv("NPC_CREATE_TIMES") != nullptr;
    std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
    void mark(const char *what) {
        if (!on) return;
        const auto now = std::chrono::steady_clock::now();
        fprintf(stderr, "npc create: %-28s %8.1f ms\n", what, std::chrono::duration<double, std::milli>(now - t).count());
        t = now;
    }
};

static bool build_pattern(int n, long long row_begin, const int *rowptr, const int *gcol, const int *lcols,
                          const double *vals, bool mirror, bool stage, PatHost &ph) {
    const long long nnz = rowptr[n];
    CreateTimer tm;
    // 1. mirror partners: a_ij (j < i, owned) whose transpose a_ji exists with the
    //    bitwise-identical value (then a_ji is an upper entry of row j, hence always own);
    // 2. (same pass, the row still in cache) the index of every own entry within its row's own
    //    list -- mirror positions refer to it
    std::unique_ptr<int[]> partner_buf(new int[(size_t)std::max<long long>(nnz, 1)]);
    int *partner = partner_buf.get();
    std::unique_ptr<unsigned char[]> opos_buf(new unsigned char[(size_t)std::max<long long>(nnz, 1)]);
    unsigned char *opos = opos_buf.get();
    std::unique_ptr<int[]> rown_buf(new int[(size_t)std::max(n, 1)]);
    int *rown = rown_buf.get();
    std::vector<char> bad(64, 0);
    host_parallel_for(n, [&](long long b, long long e, int t) {
            for (long long i = b; i < e; ++i) {
                int k = 0;
                for (int p = rowptr[i]; p < rowptr[i + 1]; ++p) {
                    int pp = -1;
                    const int c = lcols[p];
                    if (mirror && c < i && c >= 0 && i - c < PAT_MIRROR_MAX_OFF) {  // ghosts: c >= n > i
                        const int *lo = gcol + rowptr[c], *hi = gcol + rowptr[c + 1];
                        const int *q = std::lower_bound(lo, hi, (int)(row_begin + i));
                        if (q != hi && *q == row_begin + i &&
                            std::memcmp(&vals[q - gcol], &vals[p], sizeof(double)) == 0)
                            pp = (int)(q - gcol);
                    }
                    partner[p] = pp;
                    opos[p] = 0;
                    if (pp < 0) {
                        if (k > 255) bad[t] = 1;
                        opos[p] = (unsigned char)k++;
                    }
                }
                rown[i] = k;
            }
        });
    for (char c : bad)
        if (c) return false;
    tm.mark("partners + own positions");
    // 2b. a row with fewer own values than its tile's widest row streams ELL padding anyway: its
    //     mirrors of EARLIER tiles (farthest first) become own values in those slots -- the same
    //     bytes, one L2 read (or ring-kernel copy) less; bitwise the same values and order
    if (mirror && !getenv("NPC_CSR_NOFILL")) {
        host_parallel_for(ceil_div(n, PAT_TILE), [&](long long t0, long long t1, int) {
            for (long long t = t0; t < t1; ++t) {
                const int r0 = (int)t * PAT_TILE, r1 = std::min(n, r0 + PAT_TILE);
                int w = 0;
                for (int i = r0; i < r1; ++i) w = std::max(w, rown[i]);
                for (int i = r0; i < r1; ++i) {
                    if (rown[i] >= w) continue;
                    for (int p = rowptr[i]; p < rowptr[i + 1] && rown[i] < w; ++p)
                        if (partner[p] >= 0 && lcols[p] < r0) partner[p] = -1, ++rown[i];
                    int k = 0;
                    for (int p = rowptr[i]; p < rowptr[i + 1]; ++p) opos[p] = partner[p] < 0 ? (unsigned char)k++ : 0;
                }
            }
        }, 64);
    }
    tm.mark("padding fill");
    // 3. per tile: patterns (deduplicated by hash, then by words), ELL width, tables
    const int ntiles = ceil_div(n, PAT_TILE);
    std::vector<std::vector<int>> ttbl((size_t)ntiles);
    std::vector<int> twidth((size_t)ntiles, 0), txs((size_t)ntiles, 0);
    std::vector<std::vector<int>> ttbl2((size_t)ntiles);
    ph.pat.assign((size_t)std::max(n, 1), 0);
    std::vector<char> ok((size_t)ntiles, 1);
    host_parallel_for(ntiles, [&](long long t0, long long t1, int) {
        std::vector<int> words, pstart, pent;
        std::vector<unsigned long long> phash;
        for (long long t = t0; t < t1; ++t) {
            const int r0 = (int)t * PAT_TILE, r1 = std::min(n, r0 + PAT_TILE);
            phash.clear();
            pstart.assign(1, 0);
            pent.clear();
            int wmax = 0;
            for (int i = r0; i < r1 && ok[t]; ++i) {
                words.clear();
                unsigned long long h = 1469598103934665603ull;
                for (int p = rowptr[i]; p < rowptr[i + 1]; ++p) {
                    const int o = lcols[p] - i;
                    int w;
                    if (partner[p] >= 0)
                        w = (int)((unsigned)o << 9) | ((int)opos[partner[p]] << 1) | 1;
                    else
                        w = (int)((unsigned)o << 1);
                    words.push_back(w);
                    h = (h ^ (unsigned)w) * 1099511628211ull;
                }
                h ^= words.size();
                int id = -1;
                for (int q = 0; q < (int)phash.size() && id < 0; ++q)
                    if (phash[q] == h && pstart[q + 1] - pstart[q] == (int)words.size() &&
                        std::equal(words.begin(), words.end(), pent.begin() + pstart[q]))
                        id = q;
                if (id < 0) {
                    if (phash.size() == 256) {
                        ok[t] = 0;
                        break;
                    }
                    id = (int)phash.size();
                    phash.push_back(h);
                    pent.insert(pent.end(), words.begin(), words.end());
                    pstart.push_back((int)pent.size());
                }
                ph.pat[i] = (unsigned char)id;
                wmax = std::max(wmax, rown[i]);
            }
            if (!ok[t]) continue;
            const int np = (int)phash.size();
            std::vector<int> &tb = ttbl[t];  // [np + 1 absolute starts][entries]
            tb.resize((size_t)np + 1 + pent.size());
            for (int q = 0; q <= np; ++q) tb[q] = np + 1 + pstart[q];
            std::copy(pent.begin(), pent.end(), tb.begin() + np + 1);
            if ((int)tb.size() > PAT_TBL_MAX) ok[t] = 0;
            twidth[t] = wmax;
            bool ghost = false;  // tiles with ghost columns run k_csr_pat_step (x not windowed)
            for (int p = rowptr[r0]; p < rowptr[r1] && !ghost; ++p) ghost = lcols[p] >= n;
            if (!ghost && stage) {
                const int nr = r1 - r0;
                ttbl2[t] = pattern_stage_table(n, r0, nr, wmax * ((nr + 1) & ~1), pstart, pent, &txs[t]);
            }
        }
    }, 64);
    for (char c : ok)
        if (!c) return false;
    ph.tptr.assign((size_t)ntiles + 1, 0);
    ph.tbl_off.assign((size_t)ntiles + 1, 0);
    long long real = 0;
    for (int i = 0; i < n; ++i) real += rown[i];
    for (int t = 0; t < ntiles; ++t) {
        const int nr = std::min(PAT_TILE, n - t * PAT_TILE);
        const long long blk = (long long)twidth[t] * ((nr + 1) & ~1);  // even column stride: 16-byte aligned
        if (ph.tptr[t] + blk > INT_MAX) return false;
        ph.tptr[t + 1] = ph.tptr[t] + (int)blk;
        ph.tbl_off[t + 1] = ph.tbl_off[t] + (int)ttbl[t].size();
        ph.vspan_max = std::max(ph.vspan_max, (int)blk);
        ph.tbl_max = std::max(ph.tbl_max, (int)ttbl[t].size());
    }
    ph.own_nnz = ph.tptr[ntiles];
    if (8 * (ph.own_nnz - real) > real + 8LL * ntiles) return false;  // ELL padding above 1/8
    ph.tbl_max = (ph.tbl_max + 3) & ~3;
    if ((size_t)ph.vspan_max * 8 + (size_t)ph.tbl_max * 4 > (size_t)CSR_MAX_SMEM) return false;
    ph.tbl.resize((size_t)ph.tbl_off[ntiles]);
    ph.stage.assign((size_t)ntiles, 0);
    ph.tbl2_off.assign((size_t)ntiles + 1, 0);
    for (int t = 0; t < ntiles; ++t) {
        if (ttbl2[t].empty()) ttbl2[t] = {0, 4, 0, 0};  // unstaged tile: an empty header
        else ph.stage[t] = 1, ph.xspan_max = std::max(ph.xspan_max, txs[t]);
        ph.tbl2_off[t + 1] = ph.tbl2_off[t] + (int)ttbl2[t].size();
        ph.tbl2_max = std::max(ph.tbl2_max, (int)ttbl2[t].size());
    }
    ph.tbl2.resize((size_t)ph.tbl2_off[ntiles]);
    for (int t = 0; t < ntiles; ++t) std::copy(ttbl2[t].begin(), ttbl2[t].end(), ph.tbl2.begin() + ph.tbl2_off[t]);
    tm.mark("patterns + stage tables");
    // 4. ring-kernel tables: every staged tile gets one, or the operator keeps k_csr_pat_stage
    if (stage && !getenv("NPC_CSR_NORING")) {
        std::vector<RingTile> rts((size_t)ntiles);
        std::vector<char> rok((size_t)ntiles, 1);
        host_parallel_for(ntiles, [&](long long t0, long long t1, int) {
            for (long long t = t0; t < t1; ++t)
                if (ph.stage[t])
                    rok[t] = pattern_ring_table(n, (int)t, ph.tptr, twidth, ttbl[t], ph.pat.data() + t * PAT_TILE, rts[t]);
        }, 64);
        ph.ring = std::all_of(rok.begin(), rok.end(), [](char c) { return c != 0; });
        if (ph.ring) {
            // tables are tile-relative: tiles with the same row patterns share one (a 3D grid's
            // interior tiles all do), so the stored tables stay L2-resident
            size_t tmax = 0, dmax = 0;
            std::vector<long long> toff((size_t)ntiles, 0);
            std::unordered_map<unsigned long long, std::vector<int>> seen;  // hash -> tiles stored
            long long total_ints = 0;
            for (int t = 0; t < ntiles; ++t) {
                tmax = std::max(tmax, rts[t].tbl.size());
                dmax = std::max(dmax, (size_t)rts[t].dbl);
                if (!ph.stage[t]) continue;
                unsigned long long h = 1469598103934665603ull;
                for (int v : rts[t].tbl) h = (h ^ (unsigned)v) * 1099511628211ull;
                auto &cand = seen[h];
                int same = -1;
                for (int u : cand)
                    if (rts[u].tbl == rts[t].tbl) same = u;
                if (same >= 0) {
                    toff[t] = toff[same];
                } else {
                    toff[t] = total_ints;
                    total_ints += (long long)rts[t].tbl.size();
                    cand.push_back(t);
                }
            }
            ph.ring_tbl_bytes = (int)(((tmax * 4) + 15) & ~(size_t)15);
            const size_t stage = ((size_t)ph.ring_tbl_bytes + PAT_TILE + dmax * 8 + 127) & ~(size_t)127;
            ph.ring = stage <= (size_t)RING_STAGE_MAX && total_ints < INT_MAX;
            ph.ring_stage = (int)stage;
            if (ph.ring) {
                ph.rtbl.assign((size_t)total_ints + 4, 0);
                for (auto &kv : seen)
                    for (int u : kv.second) std::copy(rts[u].tbl.begin(), rts[u].tbl.end(), ph.rtbl.begin() + toff[u]);
                size_t most = 0;
                for (int t = 0; t < ntiles; ++t) most = std::max(most, rts[t].cp.size());
                ph.ring_dstride = most > 15 ? 32 : 16;
                ph.rdesc.assign((size_t)ntiles * ph.ring_dstride * 4, 0);
                ph.rdeps.assign((size_t)ntiles * 2, 0);
                for (int t = 0; t < ntiles; ++t) {
                    ph.rdeps[2 * t] = std::min(rts[t].dep_lo, t);
                    ph.rdeps[2 * t + 1] = std::max(rts[t].dep_hi, t);
                    ph.ring_span = std::max(ph.ring_span, ph.rdeps[2 * t + 1] - t);
                }
                host_parallel_for(ntiles, [&](long long t0, long long t1, int) {
                    for (long long t = t0; t < t1; ++t) {
                        if (!ph.stage[t]) continue;
                        int *dd = ph.rdesc.data() + (size_t)t * ph.ring_dstride * 4;
                        long long total = 0;
                        for (size_t k = 0; k < rts[t].cp.size(); ++k) {
                            const RingCopy &c = rts[t].cp[k];
                            const int dst = c.region == 0 ? c.dst
                                            : c.region == 1 ? ph.ring_tbl_bytes + c.dst
                                                            : ph.ring_tbl_bytes + PAT_TILE + c.dst * 8;
                            int *q = dd + 4 * (k + 1);
                            q[0] = c.kind, q[1] = dst, q[2] = c.kind == 2 ? (int)toff[t] : c.src, q[3] = c.bytes;
                            total += c.bytes;
                        }
                        dd[0] = (int)rts[t].cp.size();
                        dd[1] = (int)total;
                        dd[2] = std::any_of(rts[t].cp.begin(), rts[t].cp.end(), [](const RingCopy &c) { return c.kind == 4; });
                    }
                }, 256);
            }
        }
    }
    tm.mark("ring tables");
    ph.vals.reset(new double[(size_t)ph.own_nnz + 8]);
    std::fill(ph.vals.get() + ph.own_nnz, ph.vals.get() + ph.own_nnz + 8, 0.0);
    host_parallel_for(ntiles, [&](long long t0, long long t1, int) {
        for (long long t = t0; t < t1; ++t) {
            std::copy(ttbl[t].begin(), ttbl[t].end(), ph.tbl.begin() + ph.tbl_off[t]);
            const int r0 = (int)t * PAT_TILE, r1 = std::min(n, r0 + PAT_TILE), nrs = (r1 - r0 + 1) & ~1;
            double *blk = ph.vals.get() + ph.tptr[t];
            std::fill(blk, ph.vals.get() + ph.tptr[t + 1], 0.0);  // ELL padding
            for (int i = r0; i < r1; ++i)
                for (int p = rowptr[i]; p < rowptr[i + 1]; ++p)
                    if (partner[p] < 0) blk[(size_t)opos[p] * nrs + (i - r0)] = vals[p];
        }
    }, 64);
    tm.mark("tile-ELL values");
    return true;
}

// Upload a pattern-form operator (PatHost from build_pattern) and build its tile lists.
static npc_status finish_pattern_operator(Context *ctx, const npc_operator_desc *d, CsrOperator &op, PatHost &ph,
                                          const int *lcols) {
    const int n = d->n_local;
    op.ntiles = ceil_div(n, PAT_TILE);
    op.own_nnz = ph.own_nnz;
    op.tbl_total = (long long)ph.tbl.size();
    op.vspan_max = ph.vspan_max;
    op.tbl_max = ph.tbl_max;
    op.smem_bytes = (size_t)ph.vspan_max * 8 + (size_t)ph.tbl_max * 4;
    op.staged = true;
    std::vector<int> ti, tb;
    for (int t = 0; t < op.ntiles; ++t) {
        const int r0 = t * PAT_TILE, r1 = std::min(n, r0 + PAT_TILE);
        bool ghost = false;
        if (op.multi)
            for (int p = d->rowptr[r0]; p < d->rowptr[r1] && !ghost; ++p) ghost = lcols[p] >= n;
        (ghost ? tb : ti).push_back(t);
    }
    op.n_interior = (int)ti.size();
    op.n_boundary = (int)tb.size();
    op.xspan_max = ph.xspan_max;
    op.tbl2_max = (ph.tbl2_max + 3) & ~3;
    op.smem_stage = ((size_t)ph.vspan_max + (size_t)ph.xspan_max) * 8 + (size_t)op.tbl2_max * 4;
    op.ring = ph.ring;
    if (op.ring) {
        op.ring_stage = ph.ring_stage;
        op.ring_tbl_bytes = ph.ring_tbl_bytes;
        op.ring_tbl_ints = (long long)ph.rtbl.size();
        op.ring_dstride = ph.ring_dstride;
        for (int t = 0; t < op.ntiles; ++t)
            if (ph.stage[t]) op.ring_desc_bytes += ph.rdesc[(size_t)t * ph.ring_dstride * 4] > 15 ? 512 : 256;
        if (const char *e = getenv("NPC_RING_NS")) op.ring_ns = std::min(2, std::max(1, atoi(e)));
        if (const char *e = getenv("NPC_RING_RPT")) op.ring_rpt = atoi(e) == 4 ? 4 : 2;
        if ((size_t)op.ring_ns * op.ring_stage > 227 * 1024) op.ring_ns = 1;
        NPC_TRY(op.rtbl.alloc(sizeof(int) * ph.rtbl.size()));
        NPC_TRY(op.rdesc.alloc(sizeof(int) * ph.rdesc.size()));
        NPC_CUDA_TRY(cudaMemcpy(op.rtbl.p, ph.rtbl.data(), sizeof(int) * ph.rtbl.size(), cudaMemcpyHostToDevice));
        NPC_CUDA_TRY(cudaMemcpy(op.rdesc.p, ph.rdesc.data(), sizeof(int) * ph.rdesc.size(), cudaMemcpyHostToDevice));
        // the two-degree pass (opt-in NPC_CSR_WAVE=1): single rank, every tile staged.  Measured on
        // config 3 (profiles/r02_wave_ab.md): DRAM per pair 1.21 GB instead of 2.17 GB, but the pass
        // is then bound by its doubled L2 / bulk-copy volume and the dependency waits (p_50 10.0 ms
        // vs 8.7 ms one degree per pass)
        op.ring_span = ph.ring_span;
        op.wave = !op.multi && ph.rdeps.size() == (size_t)op.ntiles * 2 && getenv("NPC_NO_STEP2") == nullptr &&
                  getenv("NPC_CSR_WAVE") != nullptr;
        for (int t = 0; t < op.ntiles && op.wave; ++t) op.wave = ph.stage[t] != 0;
        if (op.wave) {
            NPC_TRY(op.wdeps.alloc(sizeof(int) * ph.rdeps.size()));
            NPC_TRY(op.wflags.alloc(sizeof(unsigned) * op.ntiles));
            NPC_TRY(op.wstate.alloc(sizeof(WaveState)));
            NPC_CUDA_TRY(cudaMemcpy(op.wdeps.p, ph.rdeps.data(), sizeof(int) * ph.rdeps.size(), cudaMemcpyHostToDevice));
            NPC_CUDA_TRY(cudaMemset(op.wflags.p, 0, sizeof(unsigned) * op.ntiles));
            NPC_CUDA_TRY(cudaMemset(op.wstate.p, 0, sizeof(WaveState)));
            // lag: the x-window reach plus the items in flight (3 CTAs per SM, half of them s_j)
            op.wave_persist = getenv("NPC_WAVE_PERSIST") != nullptr;
            // persistent: each CTA holds its current and its next item
            op.wave_lag = op.ring_span + ctx->num_sms * 3 / (op.wave_persist ? 1 : 2) + 64;
            if (const char *e = getenv("NPC_WAVE_LAG")) op.wave_lag = std::max(op.ring_span + 1, atoi(e));
        }
    }
    auto split = [&](const std::vector<int> &list, CsrOperator::PatTiles &pt) -> npc_status {
        std::vector<int> st, un;
        for (int t : list) (ph.stage[t] ? st : un).push_back(t);
        pt.ns = (int)st.size();
        pt.nu = (int)un.size();
        pt.identity = true;
        for (int q = 0; q < pt.ns && pt.identity; ++q) pt.identity = st[q] == q;
        NPC_TRY(pt.staged.alloc(sizeof(int) * std::max<size_t>(st.size(), 1)));
        NPC_TRY(pt.unstaged.alloc(sizeof(int) * std::max<size_t>(un.size(), 1)));
        if (!st.empty()) NPC_CUDA_TRY(cudaMemcpy(pt.staged.p, st.data(), sizeof(int) * st.size(), cudaMemcpyHostToDevice));
        if (!un.empty()) NPC_CUDA_TRY(cudaMemcpy(pt.unstaged.p, un.data(), sizeof(int) * un.size(), cudaMemcpyHostToDevice));
        return NPC_SUCCESS;
    };
    {
        std::vector<int> all((size_t)op.ntiles);
        for (int t = 0; t < op.ntiles; ++t) all[t] = t;
        NPC_TRY(split(all, op.pt_all));
        if (op.multi) NPC_TRY(split(ti, op.pt_interior));
    }
    NPC_TRY(op.tbl2.alloc(sizeof(int) * std::max<size_t>(ph.tbl2.size(), 1)));
    NPC_TRY(op.tbl2_off.alloc(sizeof(int) * ph.tbl2_off.size()));
    if (!ph.tbl2.empty())
        NPC_CUDA_TRY(cudaMemcpy(op.tbl2.p, ph.tbl2.data(), sizeof(int) * ph.tbl2.size(), cudaMemcpyHostToDevice));
    NPC_CUDA_TRY(cudaMemcpy(op.tbl2_off.p, ph.tbl2_off.data(), sizeof(int) * ph.tbl2_off.size(), cudaMemcpyHostToDevice));
    if (!op.multi && !plan_csr_poly_cluster(n, d->rowptr, op.small)) op.small = SmallCsrPlan{};
    NPC_TRY(op.prepare_kernels());  // before any launch can happen inside a PCG graph capture
    // the cluster-resident small-operator kernels read the plain arrays
    if (op.small.cl_size > 0) {
        NPC_TRY(op.rowptr.alloc(sizeof(int) * (n + 1)));
        NPC_TRY(op.cols.alloc(sizeof(int) * (op.nnz + 8)));
        NPC_TRY(op.cvals.alloc(sizeof(double) * (op.nnz + 8)));
        NPC_CUDA_TRY(cudaMemcpy(op.rowptr.p, d->rowptr, sizeof(int) * (n + 1), cudaMemcpyHostToDevice));
        NPC_CUDA_TRY(cudaMemcpy(op.cols.p, lcols, sizeof(int) * op.nnz, cudaMemcpyHostToDevice));
        NPC_CUDA_TRY(cudaMemcpy(op.cvals.p, d->vals, sizeof(double) * op.nnz, cudaMemcpyHostToDevice));
    }
    const size_t nvals = (size_t)ph.own_nnz + 8;
    NPC_TRY(op.vals.alloc(sizeof(double) * nvals));
    NPC_TRY(op.tptr.alloc(sizeof(int) * ph.tptr.size()));
    NPC_TRY(op.pat.alloc(ph.pat.size() + 16));  // bulk copies of a tile's ids round up to 16 bytes
    NPC_TRY(op.tbl.alloc(sizeof(int) * std::max<size_t>(ph.tbl.size(), 1)));
    NPC_TRY(op.tbl_off.alloc(sizeof(int) * ph.tbl_off.size()));
    NPC_CUDA_TRY(cudaMemcpy(op.vals.p, ph.vals.get(), sizeof(double) * nvals, cudaMemcpyHostToDevice));
    NPC_CUDA_TRY(cudaMemcpy(op.tptr.p, ph.tptr.data(), sizeof(int) * ph.tptr.size(), cudaMemcpyHostToDevice));
    NPC_CUDA_TRY(cudaMemcpy(op.pat.p, ph.pat.data(), ph.pat.size(), cudaMemcpyHostToDevice));
    if (!ph.tbl.empty())
        NPC_CUDA_TRY(cudaMemcpy(op.tbl.p, ph.tbl.data(), sizeof(int) * ph.tbl.size(), cudaMemcpyHostToDevice));
    NPC_CUDA_TRY(cudaMemcpy(op.tbl_off.p, ph.tbl_off.data(), sizeof(int) * ph.tbl_off.size(), cudaMemcpyHostToDevice));
    if (op.multi) {
        NPC_TRY(op.tiles_interior.alloc(sizeof(int) * std::max<size_t>(ti.size(), 1)));
        NPC_TRY(op.tiles_boundary.alloc(sizeof(int) * std::max<size_t>(tb.size(), 1)));
        if (!ti.empty())
            NPC_CUDA_TRY(cudaMemcpy(op.tiles_interior.p, ti.data(), sizeof(int) * ti.size(), cudaMemcpyHostToDevice));
        if (!tb.empty())
            NPC_CUDA_TRY(cudaMemcpy(op.tiles_boundary.p, tb.data(), sizeof(int) * tb.size(), cudaMemcpyHostToDevice));
        NPC_TRY(halo_setup(ctx, op.plan, op.halo));
    }
    return NPC_SUCCESS;
}

npc_status make_csr_operator(Context *ctx, const npc_operator_desc *d, std::unique_ptr<Operator> &out) {
    CreateTimer tm;
    NPC_TRY(validate_csr_desc(ctx, d));
    auto op = std::make_unique<CsrOperator>();
    op->ctx = ctx;
    op->kind = NPC_OP_CSR;
    op->n_local = d->n_local;
    op->n_global = d->n_global;
    op->row_begin = d->row_begin;
    const int n = d->n_local;
    const long long nnz = d->rowptr[n];
    op->nnz = nnz;
    // single rank: the caller's column ids are already local (no 4 B/nnz copy)
    std::vector<int> lvec;
    const int *lcols = d->colidx;
    if (ctx->distributed()) {
        NPC_TRY(localize_columns(ctx, d, op->plan, lvec));
        lcols = lvec.data();
    }
    op->multi = ctx->distributed();
    tm.mark("validate + localize");
    if (!getenv("NPC_CSR_PLAIN") && !getenv("NPC_CSR_CODED") && nnz > 0) {
        PatHost ph;
        if (build_pattern(n, d->row_begin, d->rowptr, d->colidx, lcols, d->vals, !getenv("NPC_CSR_NOMIRROR"),
                          !getenv("NPC_CSR_NOSTAGE"), ph)) {
            op->pattern = true;
            tm.mark("build_pattern");
            NPC_TRY(finish_pattern_operator(ctx, d, *op, ph, lcols));
            tm.mark("uploads + tile lists");
            out = std::move(op);
            return NPC_SUCCESS;
        }
    }
    // the values upload (the largest array) runs on a helper thread while the host builds the
    // column form; joined before any return
    NPC_TRY(op->vals.alloc(sizeof(double) * (nnz + 8)));
    NPC_CUDA_TRY(cudaMemset(op->vals.as<double>() + nnz, 0, sizeof(double) * 8));
    cudaError_t up_err = cudaSuccess;
    struct Joiner {
        std::thread t;
        ~Joiner() {
            if (t.joinable()) t.join();
        }
    } up;
    if (nnz) {
        const int dev = ctx->device;
        up.t = std::thread([&up_err, &op, d, nnz, dev]() {
            up_err = cudaSetDevice(dev);
            if (up_err == cudaSuccess)
                up_err = cudaMemcpy(op->vals.p, d->vals, sizeof(double) * nnz, cudaMemcpyHostToDevice);
        });
    }
    // coded column ids: per tile of CSR_TILE_CODED rows, the distinct offsets col - row (<= 256,
    // first-seen order) and a byte per entry; any tile with more -> the plain form on CSR_TILE rows
    const int ntc = ceil_div(n, CSR_TILE_CODED);
    std::vector<std::vector<int>> tdict((size_t)ntc);
    std::vector<unsigned char> hcodes;
    bool coded = !getenv("NPC_CSR_PLAIN") && nnz > 0;
    if (coded) {
        hcodes.assign((size_t)nnz + 16, 0);
        std::vector<char> ok((size_t)ntc, 1);
        host_parallel_for(ntc, [&](long long t0, long long t1, int) {
            // offset -> code by a small open-addressing table (codes in first-seen order; the
            // kernel only indexes the dictionary, so it needs no particular order)
            constexpr int HB = 10, HS = 1 << HB;  // 1,024 slots >= 4 x CSR_DICT_MAX
            std::vector<int> key(HS), val(HS);
            std::vector<long long> stamp(HS, -1);
            for (long long t = t0; t < t1; ++t) {
                const int r0 = (int)t * CSR_TILE_CODED, r1 = std::min(n, r0 + CSR_TILE_CODED);
                if (d->rowptr[r1] - d->rowptr[r0] > 65535) {  // 16-bit row offsets
                    ok[t] = 0;
                    continue;
                }
                std::vector<int> &offs = tdict[t];
                bool fits = true;
                for (int r = r0; r < r1 && fits; ++r)
                    for (int p = d->rowptr[r]; p < d->rowptr[r + 1]; ++p) {
                        const int o = lcols[p] - r;
                        unsigned h = ((unsigned)o * 2654435761u) >> (32 - HB);
                        while (stamp[h] == t && key[h] != o) h = (h + 1) & (HS - 1);
                        if (stamp[h] != t) {
                            if ((int)offs.size() == CSR_DICT_MAX) {
                                fits = false;
                                break;
                            }
                            stamp[h] = t;
                            key[h] = o;
                            val[h] = (int)offs.size();
                            offs.push_back(o);
                        }
                        hcodes[p] = (unsigned char)val[h];
                    }
                if (!fits) {
                    ok[t] = 0;
                    offs.clear();
                }
            }
        });
        for (char c : ok) coded = coded && c;
    }
    op->coded = coded;
    const int TILE = coded ? CSR_TILE_CODED : CSR_TILE;
    // tiles, spans, interior/boundary split
    op->ntiles = ceil_div(n, TILE);
    std::vector<int> ti, tb;
    for (int t = 0; t < op->ntiles; ++t) {
        int r0 = t * TILE, r1 = std::min(n, r0 + TILE);
        int pb = d->rowptr[r0], pe = d->rowptr[r1];
        op->vspan_max = std::max(op->vspan_max, ((pe + 1) & ~1) - (pb & ~1));
        op->cspan_max = std::max(op->cspan_max, ((pe + 3) & ~3) - (pb & ~3));
        bool ghost = false;
        if (op->multi)
            for (int p = pb; p < pe && !ghost; ++p) ghost = lcols[p] >= n;
        (ghost ? tb : ti).push_back(t);
    }
    op->vspan_max = (op->vspan_max + 1) & ~1;
    int cbspan_max = 0;
    if (coded)
        for (int t = 0; t < op->ntiles; ++t) {
            const int pb = d->rowptr[t * TILE], pe = d->rowptr[std::min(n, (t + 1) * TILE)];
            cbspan_max = std::max(cbspan_max, ((pe + 15) & ~15) - (pb & ~15));
        }
    op->smem_bytes = (size_t)op->vspan_max * 8 + (coded ? (size_t)cbspan_max : (size_t)op->cspan_max * 4) + 16;
    op->staged = op->smem_bytes <= (size_t)CSR_MAX_SMEM;
    op->n_interior = (int)ti.size();
    op->n_boundary = (int)tb.size();
    if (!op->multi && !plan_csr_poly_cluster(n, d->rowptr, op->small)) op->small = SmallCsrPlan{};
    // upload (arrays padded so the aligned bulk copies never read past the allocation); the
    // int32 column ids only where a kernel reads them (plain form, cluster-resident kernels)
    const bool need_cols = !coded || op->small.cl_size > 0;
    const long long ncols = need_cols ? nnz : 0;
    const int nrp = need_cols ? n + 1 : 1;  // the coded kernel reads tile pointers + 16-bit offsets
    NPC_TRY(op->rowptr.alloc(sizeof(int) * nrp));
    NPC_TRY(op->cols.alloc(sizeof(int) * (ncols + 8)));
    NPC_CUDA_TRY(cudaMemcpy(op->rowptr.p, d->rowptr, sizeof(int) * nrp, cudaMemcpyHostToDevice));
    NPC_CUDA_TRY(cudaMemset(op->cols.as<int>() + ncols, 0, sizeof(int) * 8));
    if (ncols) NPC_CUDA_TRY(cudaMemcpy(op->cols.p, lcols, sizeof(int) * ncols, cudaMemcpyHostToDevice));
    if (coded) {
        std::vector<int> doff((size_t)op->ntiles + 1, 0), dall;
        for (int t = 0; t < op->ntiles; ++t) doff[t + 1] = doff[t] + (int)tdict[t].size();
        dall.reserve((size_t)doff[op->ntiles]);
        for (auto &v : tdict) dall.insert(dall.end(), v.begin(), v.end());
        op->dict_total = (long long)dall.size();
        NPC_TRY(op->codes.alloc(hcodes.size()));
        NPC_TRY(op->dict.alloc(sizeof(int) * std::max<size_t>(dall.size(), 1)));
        NPC_TRY(op->dict_off.alloc(sizeof(int) * doff.size()));
        NPC_CUDA_TRY(cudaMemcpy(op->codes.p, hcodes.data(), hcodes.size(), cudaMemcpyHostToDevice));
        if (!dall.empty())
            NPC_CUDA_TRY(cudaMemcpy(op->dict.p, dall.data(), sizeof(int) * dall.size(), cudaMemcpyHostToDevice));
        NPC_CUDA_TRY(cudaMemcpy(op->dict_off.p, doff.data(), sizeof(int) * doff.size(), cudaMemcpyHostToDevice));
        std::vector<int> tp((size_t)op->ntiles + 1);
        std::vector<unsigned short> ro((size_t)std::max(n, 1));
        for (int t = 0; t <= op->ntiles; ++t) tp[t] = d->rowptr[std::min(n, t * CSR_TILE_CODED)];
        for (int r = 0; r < n; ++r) ro[r] = (unsigned short)(d->rowptr[r] - tp[r / CSR_TILE_CODED]);
        NPC_TRY(op->tptr.alloc(sizeof(int) * tp.size()));
        NPC_TRY(op->roff.alloc(sizeof(unsigned short) * ro.size()));
        NPC_CUDA_TRY(cudaMemcpy(op->tptr.p, tp.data(), sizeof(int) * tp.size(), cudaMemcpyHostToDevice));
        NPC_CUDA_TRY(cudaMemcpy(op->roff.p, ro.data(), sizeof(unsigned short) * ro.size(), cudaMemcpyHostToDevice));
    }
    if (op->multi) {
        NPC_TRY(op->tiles_interior.alloc(sizeof(int) * std::max<size_t>(ti.size(), 1)));
        NPC_TRY(op->tiles_boundary.alloc(sizeof(int) * std::max<size_t>(tb.size(), 1)));
        if (!ti.empty())
            NPC_CUDA_TRY(cudaMemcpy(op->tiles_interior.p, ti.data(), sizeof(int) * ti.size(), cudaMemcpyHostToDevice));
        if (!tb.empty())
            NPC_CUDA_TRY(cudaMemcpy(op->tiles_boundary.p, tb.data(), sizeof(int) * tb.size(), cudaMemcpyHostToDevice));
        NPC_TRY(halo_setup(ctx, op->plan, op->halo));
    }
    if (up.t.joinable()) up.t.join();
    NPC_CUDA_TRY(up_err);
    out = std::move(op);
    return NPC_SUCCESS;
}

}  // namespace npc

// ---------------------------------------------------------------- host-only layout check
// npc_pattern_check (include/npc.h): the pattern form and ring layout of a single-rank CSR
// matrix built exactly as npc_create_operator builds them, and y = A x evaluated ON THE HOST by
// replaying every ring tile's copy descriptors into a stage buffer (pre-filled with NaN bytes,
// so a sum that reads a byte no copy wrote is caught) and summing its rows from the entry table
// in the kernel's order (fma chain).  Alignment, bounds and byte counts of every copy are
// checked as the bulk-copy engine requires.  Tiles without a ring layout are summed from the
// CSR arrays in stored order.  A test hook for the host logic; no GPU, no context.
namespace npc {
static npc_status pattern_check_impl(int n, const int *rowptr, const int *colidx, const double *vals, const double *x,
                                     double *y, long long *info) {
    NPC_TRY(validate_csr(n, n, rowptr, colidx, vals));
    const int *lcols = colidx;
    PatHost ph;
    for (int k = 0; k < 8; ++k) info[k] = 0;
    if (!build_pattern(n, 0, rowptr, colidx, lcols, vals, !getenv("NPC_CSR_NOMIRROR"), !getenv("NPC_CSR_NOSTAGE"), ph)) {
        set_error("npc_pattern_check: the matrix does not take the pattern form");
        return NPC_ERR_UNSUPPORTED;
    }
    const int ntiles = ceil_div(n, PAT_TILE);
    info[0] = 1;
    info[1] = ph.ring ? 1 : 0;
    info[2] = ntiles;
    info[5] = ph.ring_stage;
    info[6] = (long long)ph.rtbl.size();
    info[7] = ph.own_nnz;
    auto fail = [&](const char *what, int t, int k) {
        set_error("npc_pattern_check: tile %d copy %d: %s", t, k, what);
        return NPC_ERR_INTERNAL;
    };
    std::vector<unsigned char> stage(ph.ring ? (size_t)ph.ring_stage : 0);
    for (int t = 0; t < ntiles; ++t) {
        const int r0 = t * PAT_TILE, nr = std::min(PAT_TILE, n - r0);
        if (!(ph.ring && ph.stage[t])) {
            for (int i = r0; i < r0 + nr; ++i) {
                double s = 0.0;
                for (int p = rowptr[i]; p < rowptr[i + 1]; ++p) s = std::fma(vals[p], x[colidx[p]], s);
                y[i] = s;
            }
            continue;
        }
        ++info[3];
        std::fill(stage.begin(), stage.end(), (unsigned char)0xFF);  // NaN doubles
        const int *dd = ph.rdesc.data() + (size_t)t * ph.ring_dstride * 4;
        const int nc = dd[0];
        info[4] = std::max<long long>(info[4], nc);
        if (nc < 0 || nc > RING_MAXD - 1) return fail("copy count", t, 0);
        long long total = 0;
        for (int k = 1; k <= nc; ++k) {
            const int kind = dd[4 * k], dst = dd[4 * k + 1], src = dd[4 * k + 2], bytes = dd[4 * k + 3];
            if (kind == 4) {  // odd x tail: one double stored by a thread
                if (dst % 8 || dst < 0 || dst + 8 > ph.ring_stage || src < 0 || src >= n) return fail("tail", t, k);
                std::memcpy(&stage[dst], &x[src], 8);
                continue;
            }
            if (dst % 16 || bytes % 16 || bytes <= 0 || dst < 0 || dst + bytes > ph.ring_stage)
                return fail("destination alignment / bounds", t, k);
            const unsigned char *s8 = nullptr;
            long long sbyte = 0, slen = 0;
            if (kind == 0) s8 = reinterpret_cast<const unsigned char *>(ph.vals.get()), sbyte = 8LL * src, slen = 8LL * (ph.own_nnz + 8);
            else if (kind == 1) s8 = reinterpret_cast<const unsigned char *>(x), sbyte = 8LL * src, slen = 8LL * n;
            else if (kind == 2) s8 = reinterpret_cast<const unsigned char *>(ph.rtbl.data()), sbyte = 4LL * src, slen = 4LL * (long long)ph.rtbl.size();
            else if (kind == 3) s8 = ph.pat.data(), sbyte = src, slen = (long long)ph.pat.size() + 16;
            else return fail("kind", t, k);
            if (sbyte % 16 || sbyte < 0 || sbyte + bytes > slen) return fail("source alignment / bounds", t, k);
            const long long avail = kind == 3 ? (long long)ph.pat.size() : slen;  // the id array is padded on the GPU
            std::memcpy(&stage[dst], s8 + sbyte, (size_t)std::max<long long>(0, std::min<long long>(bytes, avail - sbyte)));
            total += bytes;
        }
        if (total != dd[1]) return fail("header byte count", t, 0);
        const int *st = reinterpret_cast<const int *>(stage.data());
        const int ent = st[1], x0b = st[2];
        const unsigned char *sp = stage.data() + ph.ring_tbl_bytes;
        const unsigned char *Db = sp + PAT_TILE;
        const long long dlen = (long long)ph.ring_stage - ph.ring_tbl_bytes - PAT_TILE;
        auto ld = [&](long long off, double *v) {
            if (off < 0 || off + 8 > dlen || off % 8) return false;
            std::memcpy(v, Db + off, 8);
            return true;
        };
        for (int lr = 0; lr < nr; ++lr) {
            const int p = sp[lr];
            if (p >= st[0]) return fail("pattern id", t, lr);
            double s = 0.0, xv, vv;
            for (int e = st[4 + p]; e < st[4 + p + 1]; ++e) {
                const int ux = st[ent + 2 * e], uy = st[ent + 2 * e + 1];
                if (!ld(ux + 8LL * lr, &xv) || !ld(uy + 8LL * lr, &vv)) return fail("entry offset", t, lr);
                s = std::fma(vv, xv, s);
            }
            if (!ld(x0b + 8LL * lr, &xv) || std::memcmp(&xv, &x[r0 + lr], 8) != 0) return fail("x[row] window", t, lr);
            y[r0 + lr] = s;
        }
    }
    return NPC_SUCCESS;
}
}  // namespace npc

extern "C" npc_status npc_pattern_check(int n, const int *rowptr, const int *colidx, const double *vals,
                                        const double *x, double *y, long long *info) {
    using namespace npc;
    if (!(n >= 0 && rowptr && x && y && info && (rowptr[n] == 0 || (colidx && vals)))) {
        set_error("npc_pattern_check: null argument");
        return NPC_ERR_INVALID_ARGUMENT;
    }
    try {
        return pattern_check_impl(n, rowptr, colidx, vals, x, y, info);
    } catch (const std::bad_alloc &) {
        set_error("npc_pattern_check: host out of memory");
        return NPC_ERR_OUT_OF_MEMORY;
    }
}
