/*
 * npc.h -- C ABI of libnpc: the xi-modified Newton-Chebyshev polynomial preconditioner
 * z = p_k(A) r applied inside Preconditioned Conjugate Gradient, on NVIDIA B200 (sm_100a).
 *
 * Method: arXiv 2208.01339 (PAPER.md in the reference tree).  The problem statement is
 * "solve A x = b, A SPD, only y = A x available"; p_k(A) r is
 * Alg. 2 with theta replaced by theta_bar = theta (1 + xi) (Eq. thetamod,
 * PAPER.md:328; delta unchanged -- DESIGN.md reading A1); PCG is PAPER.md:122-123 with the
 * paper's counter laws (Table tab11).
 *
 * Conventions (all entry points):
 *  - Every call returns npc_status and never aborts or exits; npc_last_error(ctx) returns
 *    the message of the last failing call made on ctx (through ctx or a handle created
 *    from it), npc_last_error(NULL) that of the last failing call on this thread (including
 *    calls that failed before a context was known, e.g. on a NULL handle).
 *  - Pointers named *_dev are CUDA device pointers owned by the CALLER, on the context's
 *    device, holding fp64 values of the rank's n_local owned rows (contiguous, 8-byte
 *    aligned; 16-byte alignment is faster).  Everything else (operator storage, work
 *    vectors, coefficient tables) is owned by the library handle and freed by destroy.
 *  - Host arrays passed to npc_create_operator are COPIED; the caller may free them after.
 *  - All work is enqueued on the context's stream; calls that return values to the host
 *    (estimate_spectrum, pcg_solve) synchronise that stream, the others do not.
 *  - Handles are immutable after creation except for their work vectors; one host thread
 *    at a time may use a context and the handles created from it.
 *  - Multi-rank (nranks > 1): one process per GPU, rows partitioned in contiguous blocks
 *    (row_begin, n_local) in global row order.  Calls marked COLLECTIVE must be made by
 *    every rank in the same order.
 */
#ifndef NPC_H
#define NPC_H

#if defined(__GNUC__)
#define NPC_API __attribute__((visibility("default")))
#else
#define NPC_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    NPC_SUCCESS = 0,
    NPC_ERR_INVALID_ARGUMENT = 1,   /* null handle/pointer, degree < 0, xi < 0, lmin <= 0, ... */
    NPC_ERR_DIMENSION = 2,          /* CSR invariants violated, sizes inconsistent            */
    NPC_ERR_DEGENERATE_INTERVAL = 3,/* lmin == lmax: delta = 0, Chebyshev undefined (A10)       */
    NPC_ERR_NOT_CONVERGED = 4,      /* maxit reached; x holds the last iterate, stats filled  */
    NPC_ERR_BREAKDOWN = 5,          /* <r,z> <= 0 or <p,Ap> <= 0 (operator or poly not SPD)    */
    NPC_ERR_CUDA = 6,
    NPC_ERR_NCCL = 7,
    NPC_ERR_OUT_OF_MEMORY = 8,
    NPC_ERR_UNSUPPORTED = 9,
    NPC_ERR_INTERNAL = 10           /* a host-side layout check failed (npc_pattern_check)     */
} npc_status;

typedef struct npc_context_s *npc_context;
typedef struct npc_operator_s *npc_operator;
typedef struct npc_poly_s *npc_poly;

/* ---- context --------------------------------------------------------------------------
 * device: CUDA ordinal.  nranks/rank: 1/0 for a single GPU; for nranks > 1,
 * nccl_unique_id points to the 128-byte ncclUniqueId produced by npc_get_unique_id on rank
 * 0 and broadcast by the caller (e.g. torch.distributed); COLLECTIVE in that case.
 * A context created with a transport -- any nccl_unique_id, or npc_context_create_local --
 * is DISTRIBUTED even at nranks == 1: operators take the multi-rank descriptor contract
 * (global column ids, row_begin/n_global) and every operator and solver runs its multi-rank
 * path (halo plans, NCCL collectives captured into the PCG graphs, ||r||^2 allreduced on a
 * side stream overlapping the next p_k(A) r), with empty halos on one rank.  nranks == 1 without a unique id is the
 * single-GPU path (device-side convergence test, fused small-operator kernels).
 * cuda_stream: a cudaStream_t to enqueue on, or NULL for a library-owned stream.        */
NPC_API npc_status npc_context_create(int device, int nranks, int rank, const void *nccl_unique_id,
                              void *cuda_stream, npc_context *out);
/* Testing/emulation transport: the nranks ranks are host threads of THIS process (each
 * calls this with the same group name and its rank; COLLECTIVE).  Collectives go through
 * host barriers and device-to-device copies, so several ranks may share one GPU; nothing is
 * captured into CUDA graphs.  Same numerics as NCCL (sums in rank order).                */
NPC_API npc_status npc_context_create_local(int device, int nranks, int rank, const char *group,
                                    void *cuda_stream, npc_context *out);
NPC_API npc_status npc_context_destroy(npc_context ctx);
/* Global reductions of npc_pcg_solve on a DISTRIBUTED context (no effect otherwise), SURVEY
 * §8(a) a5/a6; the paper's point is that the preconditioner itself needs none
 * (PAPER.md:18-20, 1234-1237).
 *   0 (default): one allreduce of {gamma, delta} on the critical path and a second, 1-scalar
 *      allreduce of ||r_{i+1}||^2 on a side stream that overlaps the next p_k(A) r; the exit
 *      is seen about one allreduce latency into that application (stats.reductions = 2/iter).
 *   1: ONE allreduce of {gamma, delta, ||r_i||^2} per iteration (the north star's form); the
 *      exit is seen only after u = p_k(A) r and w = A u of the next iteration exist, so each
 *      solve computes one extra (k+1)-application block, counted in stats.op_applications
 *      ((iters+1)(k+1)); same iterates and iteration count as form 0.
 * NPC_PCG_FUSED_ALLREDUCE=1 in the environment sets the default of new distributed contexts. */
NPC_API npc_status npc_context_set_fused_allreduce(npc_context ctx, int enable);
NPC_API npc_status npc_get_unique_id(void *out128);
/* Message of the last failing call on ctx (ctx != NULL) or on the calling thread (NULL);
 * "" if none.  The pointer stays valid until the next failing call on the same context /
 * thread (or until npc_context_destroy).                                                   */
NPC_API const char *npc_last_error(npc_context ctx);
/* Version string, e.g. "npc 0.1 sm_100a". */
NPC_API const char *npc_version(void);
/* Number of CUDA kernels this library has launched in the process so far (all contexts). */
NPC_API unsigned long long npc_launch_count(void);

/* ---- in-library kernel timing (CUDA events on the context stream) ------------------------
 * When enabled, the library brackets its launches with CUDA events and accumulates device
 * milliseconds and launch counts per class until the next get (which resets):
 *   0 fused degree steps of p_k(A) r        1 operator applications outside p_k (w = A u,
 *   2 PCG vector update                        Lanczos A q, true residual)
 *   3 reductions and scalar kernels          4 other vector kernels (Lanczos, copies)
 * get synchronises the context stream.                                                     */
#define NPC_TIMING_CLASSES 5
NPC_API npc_status npc_context_set_timing(npc_context ctx, int enable);
NPC_API npc_status npc_context_get_timing(npc_context ctx, double *ms_out, long long *launches_out);

/* ---- operators ------------------------------------------------------------------------- */
typedef enum {
    NPC_OP_CSR = 0,      /* general sparse, CSR (configs 1, 3); tile-staged fused kernel   */
    NPC_OP_SELL = 1,     /* general sparse given as CSR, stored as SELL-C-sigma (config 4)  */
    NPC_OP_STENCIL = 2,  /* constant-coefficient 2D 5-point / 3D 7-point Dirichlet (config 2)*/
    NPC_OP_SCHUR = 3,    /* S = tridiag(-1, 2 + c, -1) + B^T D^{-1} B, never assembled (cfg 5)*/
    NPC_OP_CALLBACK = 4, /* user y = A x on the device; recurrence in a separate kernel      */
    NPC_OP_DFN = 5       /* the paper's DFN Schur complement S_u (Alg. 3), optionally Jacobi-
                            scaled by D_S (Alg. 4)                                           */
} npc_op_kind;

/* User operator: y_dev = A x_dev for this rank's n_local rows, enqueued on cuda_stream.
 * Return 0 on success; any other value makes the calling npc_* function fail. */
typedef int (*npc_apply_fn)(void *user, const double *x_dev, double *y_dev, void *cuda_stream);

typedef struct {
    npc_op_kind kind;
    long long n_global;          /* global number of rows (== n_local when nranks == 1)    */
    long long row_begin;         /* first global row owned by this rank                   */
    int n_local;                 /* rows owned by this rank                               */
    /* CSR / SELL: this rank's rows; rowptr[n_local+1] (rowptr[0] == 0), colidx = GLOBAL
     * column ids in [0, n_global), ascending within a row, vals fp64 (no NaN/Inf).        */
    const int *rowptr;
    const int *colidx;
    const double *vals;
    int sell_C;                  /* SELL chunk height; 0 -> 32 (only 32 is supported)       */
    int sell_sigma;              /* SELL sorting window; 0 -> 256; 1 -> no sorting          */
    /* STENCIL: grid nx * ny * nz_global (dim 3) or nx * ny (dim 2, nz = 1), row index
     * i = x + nx*(y + ny*z); this rank owns planes [z_begin, z_begin + nz_local).
     * y_i = diag*x_i + offdiag * sum of the existing neighbours (homogeneous Dirichlet). */
    int stencil_dim, nx, ny, nz_global, z_begin, nz_local;
    double diag, offdiag;
    /* SCHUR: c[n_local] (diagonal shift of the tridiagonal block over the rank's trace rows),
     * B rows [b_row_begin, b_row_begin + b_n_local) as CSR with GLOBAL column ids (trace
     * unknowns, 0..4 entries per row), d[b_n_local] > 0.  The B rows a rank owns are free
     * (any block); with nranks > 1 each application all-gathers v, applies the rank's B rows
     * and reduce-scatters B^T D^-1 B v to the trace-row owners.      */
    const double *c;
    long long b_rows_global;
    long long b_row_begin;
    int b_n_local;
    const int *b_rowptr;
    const int *b_colidx;
    const double *b_vals;
    const double *d;
    /* CALLBACK */
    npc_apply_fn apply;
    void *user;
    /* DFN (§4.2, Eq. schur):  S_u = G^u - a B^T A^-1 C - a C^T A^-1 B
     *                                        + C^T A^-1 G^h A^-1 C,   n_local = n^u.
     * A (n^h x n^h) SPD and G^h (n^h x n^h) SPSD must be block-diagonal over the dfn_nblk
     * fracture blocks [dfn_hblk[f], dfn_hblk[f+1]) (dfn_hblk[0] = 0, dfn_hblk[nblk] = n^h,
     * at most 8192 rows per block); C and B (n^h x n^u), G^u (n^u x n^u), all CSR with
     * column ids ascending or not (copied).  The library factorises every block of A
     * (banded Cholesky, band = the block's bandwidth in the given ordering).  dfn_scaled = 1
     * makes the operator D_S^{-1/2} S_u D_S^{-1/2}, D_S = diag(S_u) by Alg. 4 (PAPER.md:
     * 812-841), computed at create; NPC_ERR_DIMENSION if a block of A is not SPD or an entry
     * of D_S is not positive.
     * nranks > 1 (COLLECTIVE; the paper's DSMat partition): each rank passes
     * its consecutive whole fracture blocks -- dfn_nh / dfn_nblk / dfn_hblk local, h rows in
     * rank order, the column ids of A and G^h GLOBAL h ids -- and the u rows [row_begin,
     * row_begin + n_local) those fractures own: every column of C in its rows must be an owned
     * u row (C is fracture-local), else NPC_ERR_UNSUPPORTED.  B and G^u columns are GLOBAL u
     * ids of any rank; the library gathers the B^T entries and D_S of other ranks at create
     * and exchanges halos of x (u space) and of A^-1-products (h space) per application.     */
    long long dfn_nh;
    int dfn_nblk;
    const int *dfn_hblk;
    const int *a_rowptr, *a_colidx;
    const double *a_vals;
    const int *gh_rowptr, *gh_colidx;
    const double *gh_vals;
    const int *c_rowptr, *c_colidx;
    const double *c_vals;
    const int *bm_rowptr, *bm_colidx;
    const double *bm_vals;
    const int *gu_rowptr, *gu_colidx;
    const double *gu_vals;
    double dfn_alpha;
    int dfn_scaled;
} npc_operator_desc;

/* Create an operator (COLLECTIVE when nranks > 1: builds the halo plan).  Validates the
 * CSR invariants (NPC_ERR_DIMENSION), uploads and converts (CSR -> tile metadata and, when
 * every 256-row tile has <= 256 distinct column offsets, 1-byte dictionary codes for the
 * column ids; CSR -> sigma-sorted SELL-32; B -> D^{-1/2} B).                                */
NPC_API npc_status npc_create_operator(npc_context ctx, const npc_operator_desc *desc, npc_operator *out);
NPC_API npc_status npc_destroy_operator(npc_operator op);
/* Bytes of operator data one application streams in the format the library stored (e.g. a
 * CSR operator: 8 B values + 1 B codes per nonzero + dictionaries + row pointers when coded,
 * 12 B per nonzero + row pointers otherwise); the roofline numerator of the fused kernels. */
NPC_API npc_status npc_operator_matrix_bytes(npc_operator op, double *bytes);
/* y_dev = A x_dev (one application; halo exchange included).  */
NPC_API npc_status npc_apply_operator(npc_operator op, const double *x_dev, double *y_dev);

/* ---- spectrum estimate (replaces the paper's DACG) ---------------------
 * nsteps-step Lanczos (no reorthogonalisation) from v0_dev, or, when v0_dev is NULL, from the
 * counter-hash vector uniform[-1,1) (splitmix64 of `seed` and the GLOBAL row index + 1, so
 * every partition draws the same vector; workloads.lanczos_start(n, seed=...) is the same
 * generator; NPC_DEFAULT_SEED = 0x5EED is the library's and the tests' default).  seed is
 * ignored when v0_dev != NULL.  The wall time of the call is kept on the operator and
 * reported as part of npc_pcg_stats.setup_seconds by solves with a poly set after it.
 * *lmin = smallest Ritz value of T_s (an over-estimate of lambda_min: harmless for the
 * polynomial); *lmax = theta_max + rho, the largest Ritz value plus its residual norm
 * rho = beta_s |e_s^T s| -- an upper estimate of lambda_max, because an interval that misses
 * the top of the spectrum makes p_k(A) grow like T_{k+1} there (reading A11).
 * Stops early (and succeeds, rho = 0) on an exact invariant subspace.  COLLECTIVE.
 * The _ex variant writes {theta_min, theta_max, rho, steps taken} to out4 (host).          */
#define NPC_DEFAULT_SEED 0x5EEDull
NPC_API npc_status npc_estimate_spectrum(npc_operator op, int nsteps, const double *v0_dev,
                                 unsigned long long seed, double *lmin, double *lmax);
NPC_API npc_status npc_estimate_spectrum_ex(npc_operator op, int nsteps, const double *v0_dev,
                                    unsigned long long seed, double *out4);

/* ---- polynomial preconditioner (Alg. 2) --------------------------------
 * degree k >= 0 (k applications of A per npc_apply_poly), interval [lmin, lmax] with
 * 0 < lmin < lmax (lmin == lmax -> NPC_ERR_DEGENERATE_INTERVAL), xi >= 0 (Eq. thetamod).
 * Coefficients are computed once on the host (Eq. rhocheb).                                */
NPC_API npc_status npc_set_poly(npc_operator op, int degree, double lmin, double lmax, double xi,
                        npc_poly *out);
/* Newton variant (Alg. 1): P_0 r = zeta_0 r, P_{j+1} r = zeta_{j+1}(2 P_j r
 * - P_j A P_j r), degree 2^nlev - 1 (0 <= nlev <= 16), zeta_0 = 1/theta_bar and zeta_1 with
 * alpha' = theta_bar - delta (reading A1; equal to Chebyshev of the same degree,
 * PAPER.md:296-306).  Usable wherever an npc_poly is (apply, PCG); the recursion keeps
 * 2 (nlev - 1) work vectors and is not fused across levels, so Chebyshev is the fast path.  */
NPC_API npc_status npc_set_poly_newton(npc_operator op, int nlev, double lmin, double lmax, double xi,
                               npc_poly *out);
/* Low-rank spectral correction (Sec. "Low-rank acceleration"):
 *     P = p_k(A) + V (V^T A V)^{-1} V^T,
 * V_dev = p vectors of the rank's n_local rows, vector j at V_dev + j*n_local (caller-owned,
 * copied), 0 <= p <= 16; p = 0 removes the correction.  Typically V holds approximate
 * leftmost eigenvectors (npc_ritz_vectors): on an exact eigenvector the preconditioned
 * eigenvalue mu_j becomes mu_j + 1 (Eq. plusone).  Setup applies A p times and forms
 * V^T A V (Cholesky-inverted on the host): NPC_ERR_BREAKDOWN if it is not SPD.  Each later
 * application of the poly adds one p-vector reduction (V^T r; one allreduce of p scalars when
 * nranks > 1).  Applies to Chebyshev and Newton polys.  COLLECTIVE.                         */
NPC_API npc_status npc_poly_set_lowrank(npc_poly poly, int p, const double *V_dev);
/* Approximate leftmost eigenvectors: nsteps-step Lanczos with FULL reorthogonalisation
 * (stores nsteps+1 basis vectors on the device) from v0_dev or, when NULL, the counter-hash
 * start of npc_estimate_spectrum with NPC_DEFAULT_SEED; the Ritz pairs of the p smallest Ritz values of T_nsteps
 * are written to theta_out[p] (host, ascending) and V_dev (p vectors of n_local rows, vector
 * j at V_dev + j*n_local, caller-owned, unit 2-norm).  1 <= p <= 16, p <= nsteps <= 4096.
 * NPC_ERR_BREAKDOWN if the Krylov space is exhausted before p steps.  COLLECTIVE.          */
NPC_API npc_status npc_ritz_vectors(npc_operator op, int nsteps, int p, const double *v0_dev, double *V_dev,
                                    double *theta_out);
NPC_API npc_status npc_destroy_poly(npc_poly poly);
/* z_dev = p_k(A) r_dev: exactly k operator applications, no reductions, no host sync.
 * z_dev must not alias r_dev.                                                              */
NPC_API npc_status npc_apply_poly(npc_poly poly, const double *r_dev, double *z_dev);

/* ---- PCG ----------------------------------------------------------------------------------
 * Solve A x = b with PCG preconditioned by poly (NULL -> plain CG), single-reduction
 * (Chronopoulos-Gear) form with the dot products fused into the producing kernels.
 * x_dev: in = x0, out = solution.  Stops when ||r_i|| / ||b|| <= tol on the recursive
 * residual; then the true residual is formed and, if above tol, replaces r and PCG
 * restarts from the current x (at most 50 times; readings A5, A23).  tol in (0,1), maxit >= 1.
 * b == 0 -> x = 0, iters = 0, NPC_SUCCESS.  COLLECTIVE.                                     */
typedef struct {
    int iters;                   /* x updates                                               */
    int converged;
    long long op_applications;   /* every A application, including those inside p_k: k+1
                                    per iteration, +1 if x0 != 0, +1 per true residual; a
                                    distributed solve's application cut short by the
                                    overlapped convergence check is not counted             */
    long long reductions;        /* global reduction points (allreduces when distributed):
                                    1 per iteration (2 when distributed: gamma/delta, and
                                    ||r||^2 on the side stream) + 1 per V^T r of a low-rank
                                    correction, +1 each for ||b||, ||r_0||, true residual   */
    double relres_recursive;     /* ||r_iters|| / ||b|| (recursive residual)                */
    double relres_true;          /* ||b - A x|| / ||b|| of the returned x                   */
    double setup_seconds;        /* the preconditioner's setup, reported separately as the
                                    paper does for its eigenvalue estimate:
                                    wall time of the last npc_estimate_spectrum on the
                                    operator before npc_set_poly + that npc_set_poly (0 for
                                    plain CG); not part of solve_seconds                    */
    double solve_seconds;        /* wall time of the call                                   */
    double *history;             /* optional caller HOST buffer of length maxit + 1, or NULL:
                                    history[i] = ||r_i|| / ||b||, i = 0..iters               */
} npc_pcg_stats;

NPC_API npc_status npc_pcg_solve(npc_poly poly, npc_operator op, const double *b_dev, double *x_dev,
                         double tol, int maxit, npc_pcg_stats *stats);

/* ---- host-only helpers (no GPU needed) ----------------------------------------------------
 * Halo plan of a contiguous row-block partition, exposed for host-side tests of the
 * multi-rank path: given this rank's CSR rows (GLOBAL column ids) and the partition
 * row_starts[nranks + 1], writes the number of ghost columns and, if ghost_ids != NULL
 * (capacity *n_ghost), the ascending global ids of the ghost columns, and the per-rank
 * ghost counts recv_counts[nranks].  Returns NPC_ERR_DIMENSION on invalid input.          */
NPC_API npc_status npc_halo_plan(int n_local, const int *rowptr, const int *colidx, int nranks,
                         const long long *row_starts, int rank, int *n_ghost,
                         long long *ghost_ids, int *recv_counts);
/* Layout check of the CSR operator's pattern form (op_csr.cu, Alg. 2's
 * operator application): builds the storage a single-rank
 * npc_create_operator would build for the n x n CSR matrix (rowptr[n + 1], colidx, vals: HOST
 * arrays, read only, column ids ascending within a row) and evaluates y = A x ON THE HOST
 * (x, y: host arrays of n doubles) by replaying every ring-kernel tile's bulk-copy
 * descriptors into a staging buffer pre-filled with NaN bytes and summing each row from the
 * tile's entry table in the kernel's order (an fma chain in ascending column order); tiles
 * without a ring layout are summed from the CSR arrays.  Every copy's 16-byte alignment,
 * bounds and the header's byte count are checked.  info[8] (host) receives {pattern form,
 * ring layout, tiles, ring tiles, most copies in a tile, stage bytes, stored ring-table
 * words, stored own values}.  Returns NPC_ERR_UNSUPPORTED when the matrix does not take the
 * pattern form, NPC_ERR_DIMENSION on invalid CSR, NPC_ERR_INTERNAL (message in
 * npc_last_error) when the layout violates a check.  Honours the NPC_CSR_* layout knobs.    */
NPC_API npc_status npc_pattern_check(int n, const int *rowptr, const int *colidx, const double *vals,
                             const double *x, double *y, long long *info);
/* Chebyshev coefficients as used by the kernels: for j = 1..k the fused degree step is
 * s_j = a_j (A s_{j-1}) + b_j s_{j-1} + c_j s_{j-2} + d_j r with s_0 = r / theta_bar,
 * s_{-1} = 0.  Writes theta_bar, delta, sigma and the 4*k table coef[4*(j-1) + {0,1,2,3}]. */
NPC_API npc_status npc_poly_coefficients(int degree, double lmin, double lmax, double xi,
                                 double *theta_bar, double *delta, double *sigma, double *coef);

#ifdef __cplusplus
}
#endif
#endif /* NPC_H */
