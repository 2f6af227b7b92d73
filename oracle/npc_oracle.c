/*
 * npc_oracle.c -- plain, slow, obviously-correct CPU fp64 ORACLE for the hot path of
 * arXiv 2208.01339: the xi-modified Chebyshev polynomial preconditioner
 * p_m(A) r (Alg. 2) inside textbook PCG, plus the Lanczos spectrum estimate that replaces
 * the paper's DACG, and the Newton variant (Alg. 1) for cross-checks.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  It shares no code, header,
 * table or constant with the CUDA path (paper_2208_01339_b200/csrc), and neither side
 * includes the other.
 *
 * Rules followed: fp64 everywhere; no blocking, fusion or reordering beyond what the
 * cited algorithm states; sums run in index order.  Row loops of an operator application
 * may be split across OpenMP threads (each row is still summed sequentially in stored
 * order, so the result is independent of the thread count), and so may element-wise
 * vector loops (independent entries, bitwise the same result); inner products are
 * sequential.  Built with -O2 -fno-fast-math -ffp-contract=off.
 *
 * Pins (tests/test_oracle_pins.py) -- every function below is pinned; none is
 * "parity unpinned":
 *   orc_op_apply         P3 (1D-Laplacian eigenvectors), P11 (x*=1), dense comparisons
 *   orc_cheb_params/rho  P7 (SPEC worked values), P8 (rho closed form)
 *   orc_cheb_apply       P1 (Table tab:epsil eigenvalues), P3, P4 (spectrum bound), P6
 *   orc_newton_apply     P5 (Newton == Chebyshev), P12 (Fig. 1 values)
 *   orc_lanczos          P9 (n steps reproduce the spectrum; config-1 Ritz bracket)
 *   orc_pcg              P2 (Table tab:epsil iterations), P6, P10 (counter laws), P11, P15
 *   orc_lowrank_setup/apply  P14 (Eq. plusone on exact eigenvectors), P15 (dense P, symmetry)
 *   orc_lanczos_full     P16 (n steps: exact spectrum and eigenvectors of a dense SPD matrix)
 *   orc_dfn_setup/apply  P17 (Alg. 3 == dense Eq. schur, symmetry, Alg. 4 == diag, unit
 *                        diagonal after scaling, SPD), P18 (end-to-end block system residual)
 */
#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* ------------------------------------------------------------------------------------ */
/* Operators (O1).  Kinds: 0 = CSR, 1 = constant-coefficient Dirichlet stencil, 2 = Schur  */
/* S = tridiag(-1, 2 + c, -1) + B^T D^{-1} B (BASELINE config 5).                          */
/* ------------------------------------------------------------------------------------ */
typedef struct {
    int kind;
    long n;
    /* CSR */
    const int *rowptr, *colidx;
    const double *vals;
    /* stencil */
    int dim, nx, ny, nz;
    double diag, offdiag;
    /* Schur */
    const double *c;          /* length n */
    long nb;                  /* rows of B */
    const int *browptr, *bcolidx;
    const double *bvals, *d;  /* d: length nb */
    double *tmp;              /* length nb, scratch owned by the caller */
    /* DFN Schur complement (kind 3): S_u = G^u - a B^T A^-1 C - a C^T A^-1 B + C^T A^-1 G^h A^-1 C
     * (Eq. schur), n = n^u; A, G^h block-diagonal over nblk fracture blocks
     * (hblk[nblk+1] row offsets into the n^h head unknowns); C, B are n^h x n^u.          */
    long nh;
    int nblk;
    const int *hblk;
    const int *Arp, *Aci;   const double *Av;
    const int *Ghrp, *Ghci; const double *Ghv;
    const int *Crp, *Cci;   const double *Cv;
    const int *Brp, *Bci;   const double *Bv;
    const int *Gurp, *Guci; const double *Guv;
    double alpha;
    int scaled;               /* 1: apply D_S^{-1/2} S_u D_S^{-1/2}    */
    double *Lfac;             /* per-block dense Cholesky factors (orc_dfn_setup)          */
    long *Loff;
    double *ds;               /* D_S = diag(S_u) by Alg. 4 (orc_dfn_setup)                 */
    double *dwork;            /* 7 n^h + n^u scratch                                       */
} orc_op;

int orc_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* y_i = sum_j a_ij x_j, stored (ascending column) order. PAPER.md:899-901 (SpMV). */
static void csr_apply(const orc_op *A, const double *x, double *y) {
    long i;
#pragma omp parallel for schedule(static)
    for (i = 0; i < A->n; i++) {
        double s = 0.0;
        for (int p = A->rowptr[i]; p < A->rowptr[i + 1]; p++) s += A->vals[p] * x[A->colidx[p]];
        y[i] = s;
    }
}

/* Constant-coefficient 2D 5-point / 3D 7-point operator with homogeneous Dirichlet
 * boundaries (reading A13): y_i = diag*x_i + offdiag * sum over existing neighbours,
 * neighbours visited in ascending index order (z-1, y-1, x-1, x+1, y+1, z+1). */
static void stencil_apply(const orc_op *A, const double *x, double *y) {
    const long nx = A->nx, ny = A->ny, nz = (A->dim == 3) ? A->nz : 1;
    long i;
#pragma omp parallel for schedule(static)
    for (i = 0; i < A->n; i++) {
        long ix = i % nx, iy = (i / nx) % ny, iz = i / (nx * ny);
        double s = 0.0;
        if (A->dim == 3 && iz > 0) s += x[i - nx * ny];
        if (iy > 0) s += x[i - nx];
        if (ix > 0) s += x[i - 1];
        if (ix < nx - 1) s += x[i + 1];
        if (iy < ny - 1) s += x[i + nx];
        if (A->dim == 3 && iz < nz - 1) s += x[i + nx * ny];
        y[i] = A->diag * x[i] + A->offdiag * s;
    }
}

/* S x = C x + B^T (D^{-1} (B x)), two passes with a sequential scatter (O1, config 5;
 * the "global product - local inverse - transposed product" shape of Alg. 3,
 * PAPER.md:794-810, with D standing in for A). */
static void schur_apply(const orc_op *A, const double *x, double *y) {
    long i, q;
    const long n = A->n;
#pragma omp parallel for schedule(static)
    for (q = 0; q < A->nb; q++) {
        double s = 0.0;
        for (int p = A->browptr[q]; p < A->browptr[q + 1]; p++) s += A->bvals[p] * x[A->bcolidx[p]];
        A->tmp[q] = s / A->d[q];
    }
#pragma omp parallel for schedule(static)
    for (i = 0; i < n; i++) {
        double s = (2.0 + A->c[i]) * x[i];
        if (i > 0) s -= x[i - 1];
        if (i < n - 1) s -= x[i + 1];
        y[i] = s;
    }
    for (q = 0; q < A->nb; q++)
        for (int p = A->browptr[q]; p < A->browptr[q + 1]; p++) y[A->bcolidx[p]] += A->bvals[p] * A->tmp[q];
}

/* ------------------------------------------------------------------------------------ */
/* DFN Schur complement (O9).                                     */
/* ------------------------------------------------------------------------------------ */
/* y = M x for an m-row CSR matrix */
static void csr_mv(long m, const int *rp, const int *ci, const double *v, const double *x, double *y) {
    for (long i = 0; i < m; i++) {
        double s = 0.0;
        for (int p = rp[i]; p < rp[i + 1]; p++) s += v[p] * x[ci[p]];
        y[i] = s;
    }
}
/* y = M^T x (M: m rows, ncol columns), sequential scatter */
static void csr_mtv(long m, long ncol, const int *rp, const int *ci, const double *v, const double *x, double *y) {
    for (long j = 0; j < ncol; j++) y[j] = 0.0;
    for (long i = 0; i < m; i++)
        for (int p = rp[i]; p < rp[i + 1]; p++) y[ci[p]] += v[p] * x[i];
}
/* Solve L u = v (lower) then L^T t = u block by block with the dense per-block factors:
 * t = (L_A L_A^T)^{-1} v (Alg. 3 steps 3-4, 5-6, 9-10). */
static void dfn_solve_block(const orc_op *A, int f, const double *v, double *t) {
    {
        const long h0 = A->hblk[f], m = A->hblk[f + 1] - h0;
        const double *L = A->Lfac + A->Loff[f];
        for (long i = 0; i < m; i++) {                       /* L u = v */
            double s = v[h0 + i];
            for (long k = 0; k < i; k++) s -= L[i * m + k] * t[h0 + k];
            t[h0 + i] = s / L[i * m + i];
        }
        for (long i = m - 1; i >= 0; i--) {                  /* L^T t = u */
            double s = t[h0 + i];
            for (long k = i + 1; k < m; k++) s -= L[k * m + i] * t[h0 + k];
            t[h0 + i] = s / L[i * m + i];
        }
    }
}
static void dfn_solve(const orc_op *A, const double *v, double *t) {
    for (int f = 0; f < A->nblk; f++) dfn_solve_block(A, f, v, t);
}
/* Alg. 3 with the scalar alpha of Eq. schur (reading A8: the algorithm as
 * printed omits alpha).  y = S_u r. */
static void dfn_apply_unscaled(const orc_op *A, const double *r, double *y) {
    const long nh = A->nh, nu = A->n;
    double *v = A->dwork, *z = v + nh, *t = z + nh, *w = t + nh, *u = w + nh, *q = u + nh, *zu = q + nh;
    csr_mv(nh, A->Crp, A->Cci, A->Cv, r, v);                  /* 1: v = C r            */
    csr_mv(nh, A->Brp, A->Bci, A->Bv, r, z);                  /* 2: z = B r            */
    dfn_solve(A, v, t);                                      /* 3-4: t = A^-1 v       */
    dfn_solve(A, z, w);                                      /* 5-6: w = A^-1 z       */
    csr_mv(nu, A->Gurp, A->Guci, A->Guv, r, zu);              /* 7: z = G^u r ...      */
    csr_mtv(nh, nu, A->Brp, A->Bci, A->Bv, t, y);            /*    - a B^T t          */
    for (long i = 0; i < nu; i++) zu[i] -= A->alpha * y[i];
    csr_mtv(nh, nu, A->Crp, A->Cci, A->Cv, w, y);            /*    - a C^T w          */
    for (long i = 0; i < nu; i++) zu[i] -= A->alpha * y[i];
    csr_mv(nh, A->Ghrp, A->Ghci, A->Ghv, t, v);               /* 8: v = G^h t          */
    dfn_solve(A, v, q);                                      /* 9-10: w = A^-1 v      */
    csr_mtv(nh, nu, A->Crp, A->Cci, A->Cv, q, y);            /* 11: y = z + C^T w     */
    for (long i = 0; i < nu; i++) y[i] += zu[i];
}
static void dfn_apply(const orc_op *A, const double *x, double *y) {
    if (!A->scaled) { dfn_apply_unscaled(A, x, y); return; }
    const long nu = A->n;
    double *xs = A->dwork + 7 * A->nh;                        /* D^{-1/2} x            */
    for (long i = 0; i < nu; i++) xs[i] = x[i] / sqrt(A->ds[i]);
    dfn_apply_unscaled(A, xs, y);
    for (long i = 0; i < nu; i++) y[i] /= sqrt(A->ds[i]);
}

/* Setup: dense Cholesky A_f = L_f L_f^T of every diagonal block of A (PAPER.md:782-785,
 * "the exact Cholesky factorization of A"), then D_S = diag(S_u) by Alg. 4
 * with alpha: Z = (L_A L_A^T)^{-1} C, T = G^h Z - 2 alpha B, (D_S)_i = G^u_ii + z_i^T t_i,
 * one column at a time (z_i = A^{-1} c_i by dfn_solve on a dense n^h vector).
 * Returns 0, -1 (A block not SPD), -2 (A not block-diagonal), -3 (D_S entry <= 0). */
int orc_dfn_setup(orc_op *A) {
    const long nh = A->nh, nu = A->n;
    A->Loff = (long *)malloc(sizeof(long) * (A->nblk + 1));
    A->Loff[0] = 0;
    for (int f = 0; f < A->nblk; f++) {
        const long m = A->hblk[f + 1] - A->hblk[f];
        A->Loff[f + 1] = A->Loff[f] + m * m;
    }
    A->Lfac = (double *)calloc(A->Loff[A->nblk] > 0 ? A->Loff[A->nblk] : 1, sizeof(double));
    A->ds = (double *)malloc(sizeof(double) * (nu > 0 ? nu : 1));
    A->dwork = (double *)malloc(sizeof(double) * (7 * nh + nu + 1));
    for (int f = 0; f < A->nblk; f++) {
        const long h0 = A->hblk[f], m = A->hblk[f + 1] - h0;
        double *L = A->Lfac + A->Loff[f];
        for (long i = 0; i < m; i++)                          /* dense copy of A_f     */
            for (int p = A->Arp[h0 + i]; p < A->Arp[h0 + i + 1]; p++) {
                const long j = A->Aci[p] - h0;
                if (j < 0 || j >= m) return -2;
                L[i * m + j] = A->Av[p];
            }
        for (long j = 0; j < m; j++) {                        /* column Cholesky        */
            double d = L[j * m + j];
            for (long k = 0; k < j; k++) d -= L[j * m + k] * L[j * m + k];
            if (!(d > 0.0)) return -1;
            L[j * m + j] = sqrt(d);
            for (long i = j + 1; i < m; i++) {
                double s = L[i * m + j];
                for (long k = 0; k < j; k++) s -= L[i * m + k] * L[j * m + k];
                L[i * m + j] = s / L[j * m + j];
            }
            for (long i = 0; i < j; i++) L[i * m + j] = 0.0;  /* keep the strict upper part zero */
        }
    }
    /* Alg. 4, column i of C and B: gather them from the CSR rows once (CSC by counting) */
    int *ccnt = (int *)calloc(nu + 1, sizeof(int)), *bcnt = (int *)calloc(nu + 1, sizeof(int));
    for (long p = 0; p < A->Crp[nh]; p++) ccnt[A->Cci[p] + 1]++;
    for (long p = 0; p < A->Brp[nh]; p++) bcnt[A->Bci[p] + 1]++;
    for (long i = 0; i < nu; i++) { ccnt[i + 1] += ccnt[i]; bcnt[i + 1] += bcnt[i]; }
    int *crow = (int *)malloc(sizeof(int) * (A->Crp[nh] + 1)), *brow = (int *)malloc(sizeof(int) * (A->Brp[nh] + 1));
    double *cval = (double *)malloc(sizeof(double) * (A->Crp[nh] + 1)), *bval = (double *)malloc(sizeof(double) * (A->Brp[nh] + 1));
    int *cf = (int *)malloc(sizeof(int) * (nu + 1)), *bf = (int *)malloc(sizeof(int) * (nu + 1));
    memcpy(cf, ccnt, sizeof(int) * (nu + 1)); memcpy(bf, bcnt, sizeof(int) * (nu + 1));
    for (long i = 0; i < nh; i++) {
        for (int p = A->Crp[i]; p < A->Crp[i + 1]; p++) { crow[cf[A->Cci[p]]] = (int)i; cval[cf[A->Cci[p]]++] = A->Cv[p]; }
        for (int p = A->Brp[i]; p < A->Brp[i + 1]; p++) { brow[bf[A->Bci[p]]] = (int)i; bval[bf[A->Bci[p]]++] = A->Bv[p]; }
    }
    /* A is block-diagonal, so z_i = A^{-1} c_i vanishes outside the blocks that column i of C
     * touches: only those blocks are solved and summed (the rest of z_i stays 0). */
    double *cz = A->dwork, *z = cz + nh, *gz = z + nh;
    int *fblk = (int *)malloc(sizeof(int) * (nh > 0 ? nh : 1)), *touched = (int *)calloc(A->nblk + 1, sizeof(int));
    for (int f = 0; f < A->nblk; f++) for (long i = A->hblk[f]; i < A->hblk[f + 1]; i++) fblk[i] = f;
    for (long i = 0; i < nh; i++) { cz[i] = 0.0; z[i] = 0.0; }
    int st = 0;
    for (long c = 0; c < nu && !st; c++) {
        for (int p = ccnt[c]; p < ccnt[c + 1]; p++) cz[crow[p]] = cval[p];   /* c_i (dense)  */
        double zt = 0.0;                                                      /* z_i^T t_i    */
        for (int p = ccnt[c]; p < ccnt[c + 1]; p++) {
            const int f = fblk[crow[p]];
            if (touched[f]) continue;
            touched[f] = 1;
            dfn_solve_block(A, f, cz, z);                                     /* z_i = A^-1 c_i */
            for (long i = A->hblk[f]; i < A->hblk[f + 1]; i++) {              /* G^h z_i      */
                double g = 0.0;
                for (int q = A->Ghrp[i]; q < A->Ghrp[i + 1]; q++) g += A->Ghv[q] * z[A->Ghci[q]];
                zt += z[i] * g;
            }
        }
        for (int p = bcnt[c]; p < bcnt[c + 1]; p++) zt -= 2.0 * A->alpha * z[brow[p]] * bval[p];
        double gii = 0.0;
        for (int p = A->Gurp[c]; p < A->Gurp[c + 1]; p++) if (A->Guci[p] == c) gii += A->Guv[p];
        A->ds[c] = gii + zt;
        if (!(A->ds[c] > 0.0)) st = -3;
        for (int p = ccnt[c]; p < ccnt[c + 1]; p++) {                         /* reset z_i, c_i */
            const int f = fblk[crow[p]];
            cz[crow[p]] = 0.0;
            if (!touched[f]) continue;
            touched[f] = 0;
            for (long i = A->hblk[f]; i < A->hblk[f + 1]; i++) z[i] = 0.0;
        }
    }
    free(fblk); free(touched); (void)gz;
    free(ccnt); free(bcnt); free(crow); free(brow); free(cval); free(bval); free(cf); free(bf);
    return st;
}

void orc_dfn_free(orc_op *A) {
    free(A->Lfac); free(A->Loff); free(A->ds); free(A->dwork);
    A->Lfac = NULL; A->Loff = NULL; A->ds = NULL; A->dwork = NULL;
}

int orc_op_apply(const orc_op *A, const double *x, double *y) {
    switch (A->kind) {
        case 0: csr_apply(A, x, y); return 0;
        case 1: stencil_apply(A, x, y); return 0;
        case 2: schur_apply(A, x, y); return 0;
        case 3: if (!A->Lfac) return -1; dfn_apply(A, x, y); return 0;
        default: return -1;
    }
}

/* ------------------------------------------------------------------------------------ */
/* Coefficients (O3).  PAPER.md:240-252 (theta, delta, sigma; Eq. rhocheb) and Eq.       */
/* thetamod PAPER.md:328: theta_bar = theta (1 + xi); delta unchanged (reading A1).       */
/* ------------------------------------------------------------------------------------ */
int orc_cheb_params(double alpha, double beta, double xi, double *theta_bar, double *delta, double *sigma) {
    if (!(alpha > 0.0) || !(beta >= alpha) || !(xi >= 0.0)) return -1;
    double theta = (beta + alpha) / 2.0;
    *delta = (beta - alpha) / 2.0;
    *theta_bar = theta * (1.0 + xi);
    if (*delta == 0.0) return -2;              /* degenerate interval (A10) */
    *sigma = *theta_bar / *delta;
    return 0;
}

/* rho_0 = 1/sigma, rho_k = 1/(2 sigma - rho_{k-1}), k = 1..m (Eq. rhocheb). */
void orc_cheb_rho(double sigma, int m, double *rho) {
    rho[0] = 1.0 / sigma;
    for (int k = 1; k <= m; k++) rho[k] = 1.0 / (2.0 * sigma - rho[k - 1]);
}

/* ------------------------------------------------------------------------------------ */
/* p_m(A) r by Alg. 2 verbatim (O4).  work: 3n doubles.                 */
/* ------------------------------------------------------------------------------------ */
int orc_cheb_apply(const orc_op *A, int m, double alpha, double beta, double xi,
                   const double *r, double *rhat, double *work) {
    double theta_bar, delta, sigma;
    int st = orc_cheb_params(alpha, beta, xi, &theta_bar, &delta, &sigma);
    if (st) return st;
    const long n = A->n;
    double *rho = (double *)malloc(sizeof(double) * (m + 1));
    orc_cheb_rho(sigma, m, rho);                         /* step 1 */
    double *x_old = work, *x = work + n, *z = work + 2 * n;
    long i;
#pragma omp parallel for schedule(static)
    for (i = 0; i < n; i++) x_old[i] = r[i] / theta_bar;  /* step 2 */
    if (m == 0) {
        memcpy(rhat, x_old, sizeof(double) * n);
        free(rho);
        return 0;
    }
    orc_op_apply(A, r, z);                               /* step 3: x = 2 rho_1/delta (2r - A r/theta) */
#pragma omp parallel for schedule(static)
    for (i = 0; i < n; i++) x[i] = (2.0 * rho[1] / delta) * (2.0 * r[i] - z[i] / theta_bar);
    for (int k = 2; k <= m; k++) {                       /* step 4 */
        orc_op_apply(A, x, z);
#pragma omp parallel for schedule(static)
        for (i = 0; i < n; i++) z[i] = (2.0 / delta) * (r[i] - z[i]);                       /* step 5 */
#pragma omp parallel for schedule(static)
        for (i = 0; i < n; i++) rhat[i] = rho[k] * (2.0 * sigma * x[i] - rho[k - 1] * x_old[i] + z[i]); /* step 6 */
#pragma omp parallel for schedule(static)
        for (i = 0; i < n; i++) { x_old[i] = x[i]; x[i] = rhat[i]; }   /* step 7 */
    }
    memcpy(rhat, x, sizeof(double) * n);
    free(rho);
    return 0;
}

/* ------------------------------------------------------------------------------------ */
/* Newton / Hotelling polynomial (O7, cross-check only), Alg. 1 PAPER.md:190-210.         */
/* zeta_0 = 1/theta_bar; zeta_1 = 2/(1 + 2 a' zeta_0 - (a' zeta_0)^2) with a' = theta_bar */
/* - delta = alpha + xi theta (reading A1); zeta_i = 2/(1 + 2 zeta_{i-1} - zeta_{i-1}^2).  */
/* P_0 r = zeta_0 r;  P_{j+1} r = zeta_{j+1} (2 P_j r - P_j A P_j r).                    */
/* ------------------------------------------------------------------------------------ */
int orc_newton_zeta(double alpha, double beta, double xi, int nlev, double *zeta) {
    double theta_bar, delta, sigma;
    int st = orc_cheb_params(alpha, beta, xi, &theta_bar, &delta, &sigma);
    if (st == -1) return st;
    double ap = theta_bar - (beta - alpha) / 2.0;
    zeta[0] = 1.0 / theta_bar;
    if (nlev >= 1) zeta[1] = 2.0 / (1.0 + 2.0 * ap * zeta[0] - (ap * zeta[0]) * (ap * zeta[0]));
    for (int i = 2; i <= nlev; i++) zeta[i] = 2.0 / (1.0 + 2.0 * zeta[i - 1] - zeta[i - 1] * zeta[i - 1]);
    return 0;
}

static void newton_rec(const orc_op *A, const double *zeta, int j, const double *r, double *out, double *work) {
    const long n = A->n;
    long i;
    if (j == 0) {
        for (i = 0; i < n; i++) out[i] = zeta[0] * r[i];
        return;
    }
    double *pr = work, *apr = work + n, *papr = work + 2 * n, *sub = work + 3 * n;
    newton_rec(A, zeta, j - 1, r, pr, sub);          /* P_{j-1} r      */
    orc_op_apply(A, pr, apr);                         /* A P_{j-1} r    */
    newton_rec(A, zeta, j - 1, apr, papr, sub);      /* P_{j-1} A P_{j-1} r */
    for (i = 0; i < n; i++) out[i] = zeta[j] * (2.0 * pr[i] - papr[i]);
}

/* work: 3 n nlev + n doubles */
int orc_newton_apply(const orc_op *A, int nlev, double alpha, double beta, double xi,
                     const double *r, double *out, double *work) {
    double zeta[64];
    if (nlev < 0 || nlev > 60) return -1;
    int st = orc_newton_zeta(alpha, beta, xi, nlev, zeta);
    if (st) return st;
    newton_rec(A, zeta, nlev, r, out, work);
    return 0;
}

/* ------------------------------------------------------------------------------------ */
/* Lanczos (O2; replaces the paper's DACG, per the north star).         */
/* q1 = v0/||v0||, beta_0 = 0; for j = 1..m: w = A q_j - beta_{j-1} q_{j-1};               */
/* alpha_j = <q_j, w>; w -= alpha_j q_j; beta_j = ||w||; stop if beta_j == 0;              */
/* q_{j+1} = w / beta_j.  No reorthogonalisation.  Returns the number of steps taken;     */
/* T is tridiag(beta_1..beta_{s-1}; alpha_1..alpha_s).  work: 3n doubles.                 */
/* ------------------------------------------------------------------------------------ */
static double dot(long n, const double *a, const double *b) {
    double s = 0.0;
    for (long i = 0; i < n; i++) s += a[i] * b[i];
    return s;
}

/* ------------------------------------------------------------------------------------ */
/* Low-rank spectral correction (O8), PAPER.md:483-508 (Sec. "Low-rank acceleration"):    */
/*     P = P_0 + V (V^T A V)^{-1} V^T,   V = [v_1 .. v_p]  (n x p, column j at V + j n),  */
/* P_0 = p_m(A) (Alg. 2).  Setup: G = V^T A V formed entry by entry (G_ab = <v_a, A v_b>),*/
/* then its Cholesky factor G = L L^T (plain row-by-row algorithm, L lower, p x p         */
/* row-major).  Apply: s = V^T r; solve L y = s, L^T c = y; out = p_m(A) r + V c.         */
/* ------------------------------------------------------------------------------------ */
int orc_lowrank_setup(const orc_op *A, int p, const double *V, double *L, double *work) {
    const long n = A->n;
    double *G = (double *)malloc(sizeof(double) * p * p);
    for (int b = 0; b < p; b++) {
        orc_op_apply(A, V + (long)b * n, work);
        for (int a = 0; a < p; a++) G[a * p + b] = dot(n, V + (long)a * n, work);
    }
    for (int a = 0; a < p * p; a++) L[a] = 0.0;
    for (int i = 0; i < p; i++) {            /* Cholesky: L_ii = sqrt(G_ii - sum_k L_ik^2) ... */
        for (int j = 0; j <= i; j++) {
            double t = G[i * p + j];
            for (int k = 0; k < j; k++) t -= L[i * p + k] * L[j * p + k];
            if (i == j) {
                if (!(t > 0.0)) { free(G); return -1; }   /* V^T A V not SPD */
                L[i * p + i] = sqrt(t);
            } else {
                L[i * p + j] = t / L[j * p + j];
            }
        }
    }
    free(G);
    return 0;
}

/* c = (L L^T)^{-1} V^T r, out += V c.  c: p doubles of scratch. */
static void lowrank_add(long n, int p, const double *V, const double *L, const double *r, double *out, double *c) {
    for (int a = 0; a < p; a++) c[a] = dot(n, V + (long)a * n, r);          /* s = V^T r */
    for (int i = 0; i < p; i++) {                                             /* L y = s */
        double t = c[i];
        for (int k = 0; k < i; k++) t -= L[i * p + k] * c[k];
        c[i] = t / L[i * p + i];
    }
    for (int i = p - 1; i >= 0; i--) {                                        /* L^T c = y */
        double t = c[i];
        for (int k = i + 1; k < p; k++) t -= L[k * p + i] * c[k];
        c[i] = t / L[i * p + i];
    }
    for (int a = 0; a < p; a++)                                               /* out += V c */
        for (long i = 0; i < n; i++) out[i] += V[(long)a * n + i] * c[a];
}

int orc_lowrank_apply(const orc_op *A, int m, double alpha, double beta, double xi, int p, const double *V,
                      const double *L, const double *r, double *out, double *work) {
    int st = orc_cheb_apply(A, m, alpha, beta, xi, r, out, work);
    if (st) return st;
    double *c = (double *)malloc(sizeof(double) * (p > 0 ? p : 1));
    lowrank_add(A->n, p, V, L, r, out, c);
    free(c);
    return 0;
}

/* Lanczos with full reorthogonalisation (classical Gram-Schmidt applied twice against all */
/* previous basis vectors), keeping the basis Q (m+1 vectors, column j at Q + j n) for     */
/* Ritz vectors (O8 helper: approximate leftmost eigenvectors for V).  Returns the steps.  */
int orc_lanczos_full(const orc_op *A, int m, const double *v0, double *alphas, double *betas, double *Q,
                     double *w) {
    const long n = A->n;
    double nv = sqrt(dot(n, v0, v0));
    if (!(nv > 0.0)) return -1;
    long i;
    for (i = 0; i < n; i++) Q[i] = v0[i] / nv;
    int j;
    for (j = 0; j < m; j++) {
        double *q = Q + (long)j * n;
        orc_op_apply(A, q, w);
        alphas[j] = dot(n, q, w);
        for (int pass = 0; pass < 2; pass++)
            for (int l = 0; l <= j; l++) {
                const double h = dot(n, Q + (long)l * n, w);
                for (i = 0; i < n; i++) w[i] -= h * Q[(long)l * n + i];
            }
        double bnext = sqrt(dot(n, w, w));
        betas[j] = bnext;
        if (bnext == 0.0) { j++; break; }
        for (i = 0; i < n; i++) Q[(long)(j + 1) * n + i] = w[i] / bnext;
    }
    return j;
}

int orc_lanczos(const orc_op *A, int m, const double *v0, double *alphas, double *betas, double *work) {
    const long n = A->n;
    double *q = work, *q_prev = work + n, *w = work + 2 * n;
    double nv = sqrt(dot(n, v0, v0));
    if (!(nv > 0.0)) return -1;
    long i;
    for (i = 0; i < n; i++) { q[i] = v0[i] / nv; q_prev[i] = 0.0; }
    double beta_prev = 0.0;
    int j;
    for (j = 0; j < m; j++) {
        orc_op_apply(A, q, w);
        for (i = 0; i < n; i++) w[i] -= beta_prev * q_prev[i];
        double a = dot(n, q, w);
        for (i = 0; i < n; i++) w[i] -= a * q[i];
        double bnext = sqrt(dot(n, w, w));
        alphas[j] = a;
        betas[j] = bnext;
        if (bnext == 0.0) { j++; break; }
        for (i = 0; i < n; i++) { q_prev[i] = q[i]; q[i] = w[i] / bnext; }
        beta_prev = bnext;
    }
    return j;
}

/* ------------------------------------------------------------------------------------ */
/* Textbook PCG (O5; Saad Alg. 9.1), stopping rule (reading A5):        */
/* ||r_i||_2 / ||b||_2 <= tol on the recursively updated residual, iterations counted as  */
/* x-updates.  When it fires, the true residual b - A x is formed; if it is above tol the */
/* true residual replaces r and PCG restarts from the current x (p = z, beta = 0; reading */
/* A23 in DESIGN.md), at most 50 times: the 51st true check still above tol ends the      */
/* solve, not converged (a true residual stuck above tol is the attainable-accuracy floor).*/
/* Preconditioner: m < 0 -> none (CG); m >= 0 -> Chebyshev p_m (Alg. 2) on [alpha, beta]. */
/* ------------------------------------------------------------------------------------ */
typedef struct {
    int iters, converged, breakdown;
    long long mvp, ddot;
    double relres_recursive, relres_true;
    int true_checks;            /* true residuals formed by the stopping test (A23) */
} orc_pcg_stats;

int orc_pcg(const orc_op *A, int m, double alpha, double beta, double xi,
            const double *b, double *x, double tol, int maxit, double *history, orc_pcg_stats *st,
            int lr_p, const double *lr_V, const double *lr_L) {
    const long n = A->n;
    long i;
    double *r = (double *)malloc(sizeof(double) * n), *z = (double *)malloc(sizeof(double) * n);
    double *p = (double *)malloc(sizeof(double) * n), *q = (double *)malloc(sizeof(double) * n);
    double *work = (double *)malloc(sizeof(double) * 3 * n);
    double *lr_c = (double *)malloc(sizeof(double) * (lr_p > 0 ? lr_p : 1));
    memset(st, 0, sizeof(*st));
    int true_done = 0;          /* true residual computed for the final x */
    int restart = 0;            /* set by a residual replacement (A23)     */
    double rr = 0.0, rz = 0.0;
    int x0_nonzero = 0;
    for (i = 0; i < n; i++) if (x[i] != 0.0) { x0_nonzero = 1; break; }
    double bnorm = sqrt(dot(n, b, b));
    st->ddot++;
    if (bnorm == 0.0) {                               /* zero right-hand side -> x = 0 */
        for (i = 0; i < n; i++) x[i] = 0.0;
        st->converged = 1;
        true_done = 1;
        goto done;
    }
    if (x0_nonzero) {
        orc_op_apply(A, x, q); st->mvp++;
        for (i = 0; i < n; i++) r[i] = b[i] - q[i];
    } else {
        for (i = 0; i < n; i++) r[i] = b[i];
    }
    rr = dot(n, r, r); st->ddot++;
    st->relres_recursive = sqrt(rr) / bnorm;
    if (history) history[0] = st->relres_recursive;
    if (st->relres_recursive <= tol) { st->converged = 1; goto done; }
#define APPLY_M(src, dst)                                                              \
    do {                                                                               \
        if (m < 0) memcpy(dst, src, sizeof(double) * n);                               \
        else { orc_cheb_apply(A, m, alpha, beta, xi, src, dst, work); st->mvp += m; }   \
        if (lr_p > 0) { lowrank_add(n, lr_p, lr_V, lr_L, src, dst, lr_c); st->ddot += lr_p; } \
    } while (0)
    APPLY_M(r, z);
    for (i = 0; i < n; i++) p[i] = z[i];
    rz = dot(n, r, z); st->ddot++;
    if (!(rz > 0.0)) { st->breakdown = 1; goto done; }
    for (int it = 1; it <= maxit; it++) {
        orc_op_apply(A, p, q); st->mvp++;
        double pq = dot(n, p, q); st->ddot++;
        if (!(pq > 0.0)) { st->breakdown = 1; break; }
        double a = rz / pq;
#pragma omp parallel for schedule(static)
        for (i = 0; i < n; i++) x[i] += a * p[i];
#pragma omp parallel for schedule(static)
        for (i = 0; i < n; i++) r[i] -= a * q[i];
        rr = dot(n, r, r); st->ddot++;
        st->iters = it;
        st->relres_recursive = sqrt(rr) / bnorm;
        if (history) history[it] = st->relres_recursive;
        if (st->relres_recursive <= tol) {
            orc_op_apply(A, x, q); st->mvp++;
            for (i = 0; i < n; i++) q[i] = b[i] - q[i];
            double tr = sqrt(dot(n, q, q)) / bnorm; st->ddot++;
            st->relres_true = tr;
            st->true_checks++;
            if (tr <= tol) { st->converged = 1; true_done = 1; break; }
            if (st->true_checks > 50) { true_done = 1; break; }   /* A23 cap: not converged */
            for (i = 0; i < n; i++) r[i] = q[i];      /* residual replacement ...        */
            restart = 1;                              /* ... and restart: p = z below    */
        }
        if (it == maxit) break;
        APPLY_M(r, z);
        double rz_new = dot(n, r, z); st->ddot++;
        if (!(rz_new > 0.0)) { st->breakdown = 1; break; }
        double bet = restart ? 0.0 : rz_new / rz;
        restart = 0;
        rz = rz_new;
#pragma omp parallel for schedule(static)
        for (i = 0; i < n; i++) p[i] = z[i] + bet * p[i];
    }
#undef APPLY_M
done:
    if (!true_done) {
        /* report the true residual of the final iterate */
        orc_op_apply(A, x, q); st->mvp++;
        for (i = 0; i < n; i++) q[i] = b[i] - q[i];
        st->relres_true = sqrt(dot(n, q, q)) / bnorm; st->ddot++;
    }
    free(r); free(z); free(p); free(q); free(work); free(lr_c);
    return 0;
}
