"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This module holds NO arithmetic of the method (no operator application, no polynomial,
no Krylov step): it only draws random numbers and lays out the operators the method is
applied to.  Every recipe below is the one written down in DESIGN.md §"Input recipe"
(SURVEY.md §8(d) table "Inputs"; ambiguity readings A13-A18).  The paper's own matrices
(Cube_5317k, DFN #1-#4, Frac16/32 -- PAPER.md:513-514, 919-944) are not available; these
configs stand in for them (configs 1-3: PDE stencils like the fracture blocks of A,
PAPER.md:686-689; config 4: an unstructured SPD matrix like Cube_5317k; config 5: the
"global product - local inverse - transposed product" shape of S_u).

All generators use numpy.random.default_rng(seed) (PCG64), one stream per config, in the
draw order stated in each docstring.  Index types are int32 (max nnz 156.7M < 2^31).
"""
from __future__ import annotations

import numpy as np

__all__ = [
    "config1", "config2", "config3", "config4", "config5", "dfn", "dfn_owner_order",
    "tab_epsil_diag", "laplacian_1d_csr", "random_spd_dense", "dense_to_csr", "lanczos_start",
    "CONFIG_DEFAULTS",
]

# Per-config solver parameters (BASELINE.json "configs").
CONFIG_DEFAULTS = {
    1: dict(k=10, tol=1e-8, lanczos_steps=20),
    2: dict(k=30, tol=1e-10, lanczos_steps=20),
    3: dict(k=50, ks=(20, 50, 100), tol=1e-8, lanczos_steps=20),
    4: dict(k=60, tol=1e-8, lanczos_steps=20),
    5: dict(k=50, ks=(10, 50, 100, 200), tol=1e-8, lanczos_steps=20),
}


def _csr_from_padded(cols: np.ndarray, vals: np.ndarray, mask: np.ndarray):
    """Compress a (n, w) padded row layout (columns already ascending per row) into CSR."""
    counts = mask.sum(axis=1, dtype=np.int64)
    rowptr = np.zeros(cols.shape[0] + 1, dtype=np.int64)
    np.cumsum(counts, out=rowptr[1:])
    assert rowptr[-1] < 2**31
    m = mask.ravel()
    return rowptr.astype(np.int32), cols.ravel()[m].astype(np.int32), vals.ravel()[m].astype(np.float64)


def grid_laplacian_csr(dims, diag, offdiag):
    """Constant-coefficient 2D 5-point / 3D 7-point Dirichlet operator as CSR.

    Grid ordering i = x + nx*y + nx*ny*z (x fastest, reading A16); columns ascending.
    """
    dims = tuple(int(d) for d in dims)
    n = int(np.prod(dims))
    idx = np.arange(n, dtype=np.int64)
    coords = []
    stride = 1
    strides = []
    rem = idx
    for d in dims:
        coords.append(rem % d)
        rem = rem // d
        strides.append(stride)
        stride *= d
    # neighbour offsets in ascending column order: -s_last ... -s_0, 0, +s_0 ... +s_last
    offs, conds, vals_list = [], [], []
    for a in reversed(range(len(dims))):
        offs.append(-strides[a]); conds.append(coords[a] > 0)
    offs.append(0); conds.append(np.ones(n, dtype=bool))
    for a in range(len(dims)):
        offs.append(strides[a]); conds.append(coords[a] < dims[a] - 1)
    w = len(offs)
    cols = np.empty((n, w), dtype=np.int64)
    vals = np.empty((n, w), dtype=np.float64)
    mask = np.empty((n, w), dtype=bool)
    for j, (o, c) in enumerate(zip(offs, conds)):
        cols[:, j] = idx + o
        vals[:, j] = diag if o == 0 else offdiag
        mask[:, j] = c
    cols[~mask] = 0
    return _csr_from_padded(cols, vals, mask)


def config1(side: int = 64, seed: int = 0):
    """Config 1: 2D 5-point Laplacian, side x side (64x64 -> n=4096, nnz=20224), Dirichlet,
    diagonal 4, off-diagonal -1, CSR.  seed 0: b = uniform(-1, 1, n).  x0 = 0."""
    rowptr, colidx, vals = grid_laplacian_csr((side, side), 4.0, -1.0)
    rng = np.random.default_rng(seed)
    b = rng.uniform(-1.0, 1.0, side * side)
    return dict(kind="csr", name=f"config1_{side}x{side}", n=side * side, rowptr=rowptr,
                colidx=colidx, vals=vals, b=b, grid=(side, side), **CONFIG_DEFAULTS[1])


def config2(side: int = 128, seed: int = 1):
    """Config 2: 3D 7-point constant-coefficient Laplacian (diag 6, off -1, Dirichlet, A13),
    side^3 grid, applied matrix-free.  seed 1: b = uniform(-1, 1, n)."""
    n = side ** 3
    rng = np.random.default_rng(seed)
    b = rng.uniform(-1.0, 1.0, n)
    return dict(kind="stencil", name=f"config2_{side}^3", n=n, dim=3, nx=side, ny=side, nz=side,
                diag=6.0, offdiag=-1.0, b=b, **CONFIG_DEFAULTS[2])


def config3(side: int = 256, seed: int = 2, want_b: bool = True):
    """Config 3: 3D 7-point variable-coefficient diffusion on side^3, CSR (reading A13).

    Face coefficients c = exp(2 z), z ~ N(0,1), i.i.d. per face INCLUDING boundary faces.
    Draw order (seed 2): x-faces as C-order (z, y, x_face=side+1), then y-faces
    (z, y_face=side+1, x), then z-faces (z_face=side+1, y, x).
    A_ii = sum of the 6 face coefficients, A_ij = -c_face for interior faces.
    b = A*ones, which equals the sum of the cell's boundary-face coefficients (exact
    solution x* = 1, pin P11); it is formed from the faces, not by a product with A.
    """
    N = int(side)
    rng = np.random.default_rng(seed)
    cx = np.exp(2.0 * rng.standard_normal((N, N, N + 1)))
    cy = np.exp(2.0 * rng.standard_normal((N, N + 1, N)))
    cz = np.exp(2.0 * rng.standard_normal((N + 1, N, N)))
    n = N ** 3
    w_, e_ = cx[:, :, :N], cx[:, :, 1:]
    s_, n_ = cy[:, :N, :], cy[:, 1:, :]
    d_, u_ = cz[:N, :, :], cz[1:, :, :]
    diag = (w_ + e_) + (s_ + n_) + (d_ + u_)
    z, y, x = np.meshgrid(np.arange(N), np.arange(N), np.arange(N), indexing="ij")
    idx = np.arange(n, dtype=np.int64)
    cols = np.empty((n, 7), dtype=np.int64)
    vals = np.empty((n, 7), dtype=np.float64)
    mask = np.empty((n, 7), dtype=bool)
    spec = [(-N * N, d_, z > 0), (-N, s_, y > 0), (-1, w_, x > 0), (0, None, None),
            (1, e_, x < N - 1), (N, n_, y < N - 1), (N * N, u_, z < N - 1)]
    for j, (o, c, cond) in enumerate(spec):
        cols[:, j] = idx + o
        if o == 0:
            vals[:, j] = diag.ravel()
            mask[:, j] = True
        else:
            vals[:, j] = -c.ravel()
            mask[:, j] = cond.ravel()
    del z, y, x
    cols[~mask] = 0
    rowptr, colidx, v = _csr_from_padded(cols, vals, mask)
    del cols, vals, mask
    out = dict(kind="csr", name=f"config3_{N}^3", n=n, rowptr=rowptr, colidx=colidx, vals=v,
               grid=(N, N, N), **CONFIG_DEFAULTS[3])
    if want_b:
        b = np.zeros((N, N, N))
        b[:, :, 0] += cx[:, :, 0]
        b[:, :, N - 1] += cx[:, :, N]
        b[:, 0, :] += cy[:, 0, :]
        b[:, N - 1, :] += cy[:, N, :]
        b[0, :, :] += cz[0, :, :]
        b[N - 1, :, :] += cz[N, :, :]
        out["b"] = b.ravel()
        out["x_exact"] = 1.0
    return out


def config4(n: int = 8_000_000, seed: int = 3, knn: int = 16, shift: float = 1e-3):
    """Config 4: graph Laplacian of a symmetric kNN graph + shift*I, RCM-ordered CSR.

    Draw order (seed 3): points uniform[0,1)^3 (n x 3); edge weights uniform[0.1, 10] for the
    undirected edges in (i<j) lexicographic order; b = uniform(-1, 1, n) in original vertex
    order.  Edges: Euclidean knn excluding self, symmetrised by union (A18).  The matrix and b
    are then permuted by scipy's reverse_cuthill_mckee (symmetric_mode=True), computed here
    and shipped as `perm` (A17).  The library applies its own SELL sigma-sort on top.
    """
    from scipy.spatial import cKDTree
    import scipy.sparse as sp
    from scipy.sparse.csgraph import reverse_cuthill_mckee

    rng = np.random.default_rng(seed)
    pts = rng.random((n, 3))
    tree = cKDTree(pts)
    _, nbr = tree.query(pts, k=knn + 1, workers=-1)
    nbr = nbr.astype(np.int64)
    src = np.repeat(np.arange(n, dtype=np.int64), knn + 1)
    dst = nbr.ravel()
    keep = src != dst
    src, dst = src[keep], dst[keep]
    lo, hi = np.minimum(src, dst), np.maximum(src, dst)
    key = np.unique(lo * n + hi)
    ei, ej = key // n, key % n
    w = rng.uniform(0.1, 10.0, key.size)
    b = rng.uniform(-1.0, 1.0, n)
    W = sp.coo_matrix((np.concatenate([w, w]), (np.concatenate([ei, ej]), np.concatenate([ej, ei]))),
                      shape=(n, n)).tocsr()
    deg = np.asarray(W.sum(axis=1)).ravel()
    A = (sp.diags(deg + shift) - W).tocsr()
    perm = reverse_cuthill_mckee(A, symmetric_mode=True).astype(np.int64)
    A = A[perm][:, perm].tocsr()
    A.sort_indices()
    assert A.nnz < 2**31
    return dict(kind="csr", name=f"config4_knn{knn}_{n}", n=n, rowptr=A.indptr.astype(np.int32),
                colidx=A.indices.astype(np.int32), vals=A.data.astype(np.float64), b=b[perm],
                perm=perm, sell_C=32, sell_sigma=256, **CONFIG_DEFAULTS[4])


def config5(n: int = 4_000_000, seed: int = 4, rows_per_trace: int = 3):
    """Config 5: DFN-like Schur complement S = C + B^T D^{-1} B, never assembled.

    C = tridiag(-1, 2 + c, -1) (1D Laplacian plus diagonal c ~ U[1,2]); B is (3n) x n with
    row lengths uniform in {2,3,4} at distinct sorted random columns, values N(0,1);
    D ~ U[1,100].  Draw order (seed 4): c (n), row lengths (nb), columns (all rows at once,
    then rows with a duplicate are redrawn one by one in row order until distinct), values
    (nnz), D (nb), b = uniform(-1,1,n) (A14).
    """
    rng = np.random.default_rng(seed)
    nb = rows_per_trace * n
    c = rng.uniform(1.0, 2.0, n)
    lens = rng.integers(2, 5, nb)
    browptr = np.zeros(nb + 1, dtype=np.int64)
    np.cumsum(lens, out=browptr[1:])
    nnz = int(browptr[-1])
    cols = rng.integers(0, n, nnz)
    pad = np.full((nb, 4), np.iinfo(np.int64).max, dtype=np.int64)
    slot = np.arange(nnz) - np.repeat(browptr[:-1], lens)
    rowid = np.repeat(np.arange(nb), lens)
    pad[rowid, slot] = cols
    pad.sort(axis=1)
    dup = np.any((pad[:, 1:] == pad[:, :-1]) & (pad[:, 1:] != np.iinfo(np.int64).max), axis=1)
    for r in np.nonzero(dup)[0]:
        L = int(lens[r])
        while True:
            cand = rng.integers(0, n, L)
            if np.unique(cand).size == L:
                break
        pad[r, :] = np.iinfo(np.int64).max
        pad[r, :L] = np.sort(cand)
    bcol = pad[rowid, slot]
    bval = rng.standard_normal(nnz)
    D = rng.uniform(1.0, 100.0, nb)
    b = rng.uniform(-1.0, 1.0, n)
    return dict(kind="schur", name=f"config5_{n}", n=n, nb=nb, c=c, browptr=browptr.astype(np.int32),
                bcolidx=bcol.astype(np.int32), bvals=bval, d=D, b=b, **CONFIG_DEFAULTS[5])


def dfn(nf: int = 2000, seed: int = 5, traces_per_fracture: int = 8, grid=(4, 8), trace_len=(8, 16),
        alpha: float | None = None):
    """Synthetic DFN block system (SPEC.md generate_synthetic), the
    stand-in for the paper's DFN test cases (Table size; Frac32 has ~34
    head unknowns per fracture and n^u / n^h ~ 2.8).  Structure follows the bullets of
    Eq. algebraic_model:

    * nf fractures, fracture f a grid nx_f x ny_f (uniform in [grid[0], grid[1]]), head
      unknowns h numbered fracture by fracture, x fastest (block-diagonal structure);
    * A = block-diag(K_f L_f): L_f the 2D 5-point Dirichlet Laplacian of the fracture grid,
      transmissivity K_f = exp(0.5 N(0,1)) -- SPD, "a 2-D discrete Laplacian" per block;
    * traces: traces_per_fracture * nf pairs (f, g), f != g uniform; trace t carries L_t flux
      unknowns u (L_t uniform in trace_len); the trace lies on a horizontal or vertical grid
      line of each of its two fractures; u-dof k sits at s_k = (k + 1/2)/L_t along the line and
      couples to its two nearest line nodes with hat weights (1 - th, th) / L_t;
    * C: the owner fracture's (min(f, g)) couplings -- fracture-local rectangular blocks;
      E: the other fracture's couplings (support disjoint from C's blocks); B = C + E;
    * G^h = block-diag: for every trace on fracture f, the path-graph Laplacian of the nodes
      of its line (SPSD, rank-deficient), summed;
    * G^u = block-diag over traces of tridiag(-1, 2, -1) (1D Dirichlet, SPD; trace dofs tie
      the two fractures of a trace: "global nature");
    * alpha ("usually on the order of 1"; SPD "by wisely selecting alpha",
      PAPER.md:774-777): unless given, half the value that makes S_u(alpha) SPD by the norm
      bound alpha ||B^T A^-1 C + C^T A^-1 B|| <= 2 alpha ||B|| ||C|| / lambda_min(A) <
      lambda_min(G^u), with ||M||_2 <= sqrt(||M||_1 ||M||_inf) and the closed-form Laplacian
      eigenvalues 4 sin^2(pi / (2(m+1))) -- input construction, no method arithmetic;
    * b (the Schur right-hand side, u-space) = uniform(-1, 1, n^u).

    Draw order (seed): grid dims (nf x 2), K_f (nf), trace pairs f (T), g (T), lengths (T),
    line orientation + index for the owner then the other fracture (4 x T), b (n^u).
    """
    import scipy.sparse as sp
    rng = np.random.default_rng(seed)
    dims = rng.integers(grid[0], grid[1] + 1, size=(nf, 2))
    nx, ny = dims[:, 0].astype(np.int64), dims[:, 1].astype(np.int64)
    nblk = nx * ny
    hoff = np.zeros(nf + 1, dtype=np.int64)
    np.cumsum(nblk, out=hoff[1:])
    nh = int(hoff[-1])
    K = np.exp(0.5 * rng.standard_normal(nf))
    T = traces_per_fracture * nf
    f = rng.integers(0, nf, T)
    g = rng.integers(0, nf - 1, T)
    g = g + (g >= f)
    L = rng.integers(trace_len[0], trace_len[1] + 1, T)
    orient = rng.integers(0, 2, size=(2, T))          # 0: horizontal line (fixed y), 1: vertical
    linepick = rng.random(size=(2, T))                # line index = floor(pick * lines)
    owner, other = np.minimum(f, g), np.maximum(f, g)
    uoff = np.zeros(T + 1, dtype=np.int64)
    np.cumsum(L, out=uoff[1:])
    nu = int(uoff[-1])
    b = rng.uniform(-1.0, 1.0, nu)

    # ---- A: block-diag K_f * 5-point Dirichlet Laplacian
    rows, cols, vals = [], [], []
    for (mx, my) in {(int(a), int(c)) for a, c in dims}:
        sel = np.nonzero((nx == mx) & (ny == my))[0]
        loc = np.arange(mx * my)
        x, y = loc % mx, loc // mx
        lr, lc, lv = [loc], [loc], [np.full(loc.size, 4.0)]
        for dx, dy in ((-1, 0), (1, 0), (0, -1), (0, 1)):
            ok = (x + dx >= 0) & (x + dx < mx) & (y + dy >= 0) & (y + dy < my)
            lr.append(loc[ok]); lc.append(loc[ok] + dx + mx * dy); lv.append(np.full(ok.sum(), -1.0))
        lr, lc, lv = np.concatenate(lr), np.concatenate(lc), np.concatenate(lv)
        rows.append((hoff[sel][:, None] + lr[None, :]).ravel())
        cols.append((hoff[sel][:, None] + lc[None, :]).ravel())
        vals.append((K[sel][:, None] * lv[None, :]).ravel())
    A = sp.csr_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))), shape=(nh, nh))

    # ---- trace lines on both fractures: node ids of each line
    def line_nodes(fr, o, pick):
        mx, my = nx[fr], ny[fr]
        m = np.where(o == 0, mx, my)                      # nodes along the line
        nlines = np.where(o == 0, my, mx)
        li = np.minimum((pick * nlines).astype(np.int64), nlines - 1)
        return m, li
    cr, cc, cv, er, ec, ev = [], [], [], [], [], []
    ghr, ghc, ghv = [], [], []
    for side, fr in ((0, owner), (1, other)):
        o, pick = orient[side], linepick[side]
        m, li = line_nodes(fr, o, pick)
        # u-dof k of trace t -> nodes j0 = floor(s), j0 + 1 along the line, s = (k+1/2)/L (m-1)
        tt = np.repeat(np.arange(T), L)
        kk = np.arange(nu) - uoff[tt]
        s = (kk + 0.5) / L[tt] * (m[tt] - 1)
        j0 = np.minimum(np.floor(s).astype(np.int64), m[tt] - 2)
        th = s - j0
        def node(j):
            return np.where(o[tt] == 0, hoff[fr[tt]] + li[tt] * nx[fr[tt]] + j, hoff[fr[tt]] + j * nx[fr[tt]] + li[tt])
        w0, w1 = (1.0 - th) / L[tt], th / L[tt]
        tr, tc, tv = (cr, cc, cv) if side == 0 else (er, ec, ev)
        tr += [node(j0), node(j0 + 1)]
        tc += [np.arange(nu), np.arange(nu)]
        tv += [w0, w1]
        # G^h: path Laplacian along the line (edges j, j+1 for j < m-1)
        te = np.repeat(np.arange(T), m - 1)
        je = np.arange(int((m - 1).sum())) - np.repeat(np.cumsum(m - 1) - (m - 1), m - 1)
        def node_t(j):
            return np.where(o[te] == 0, hoff[fr[te]] + li[te] * nx[fr[te]] + j, hoff[fr[te]] + j * nx[fr[te]] + li[te])
        a_, c_ = node_t(je), node_t(je + 1)
        ghr += [a_, c_, a_, c_]; ghc += [a_, c_, c_, a_]
        one = np.ones(a_.size)
        ghv += [one, one, -one, -one]
    C = sp.csr_matrix((np.concatenate(cv), (np.concatenate(cr), np.concatenate(cc))), shape=(nh, nu))
    E = sp.csr_matrix((np.concatenate(ev), (np.concatenate(er), np.concatenate(ec))), shape=(nh, nu))
    B = (C + E).tocsr()
    Gh = sp.csr_matrix((np.concatenate(ghv), (np.concatenate(ghr), np.concatenate(ghc))), shape=(nh, nh))
    # ---- G^u: per-trace tridiag(-1, 2, -1)
    ku = np.arange(nu) - uoff[np.repeat(np.arange(T), L)]
    Lr = np.repeat(L, L)
    gr, gc, gv = [np.arange(nu)], [np.arange(nu)], [np.full(nu, 2.0)]
    nxt = np.nonzero(ku < Lr - 1)[0]
    gr += [nxt, nxt + 1]; gc += [nxt + 1, nxt]; gv += [-np.ones(nxt.size), -np.ones(nxt.size)]
    Gu = sp.csr_matrix((np.concatenate(gv), (np.concatenate(gr), np.concatenate(gc))), shape=(nu, nu))
    for M in (A, B, C, Gh, Gu):
        M.sum_duplicates()
        M.sort_indices()
    if alpha is None:
        def n2(M):
            a = abs(M)
            return float(np.sqrt(a.sum(axis=0).max() * a.sum(axis=1).max()))
        lam_a = float(np.min(K * (4 * np.sin(np.pi / (2 * (nx + 1))) ** 2 + 4 * np.sin(np.pi / (2 * (ny + 1))) ** 2)))
        lam_gu = float(4 * np.sin(np.pi / (2 * (L.max() + 1))) ** 2)
        alpha = 0.5 * lam_gu * lam_a / (2.0 * n2(B) * n2(C))

    def csr(M):
        return (M.indptr.astype(np.int32), M.indices.astype(np.int32), M.data.astype(np.float64))
    return dict(kind="dfn", name=f"dfn_{nf}", n=nu, nh=nh, nf=nf, hblk=hoff.astype(np.int32), alpha=float(alpha),
                A=csr(A), Gh=csr(Gh), C=csr(C), B=csr(B), Gu=csr(Gu), b=b, k=30, tol=1e-8, lanczos_steps=20)


def dfn_owner_order(w: dict):
    """Renumber the u unknowns of a dfn() system so that the flux unknowns owned by each
    fracture (the columns of C with rows in it; C is fracture-local) are contiguous and in
    fracture order -- the DSMat layout of PAPER.md:879-899, where a rank stores consecutive
    whole fracture blocks and that subdivision "guides the partitioning of the other matrices
    B and G^u".  A symmetric permutation of S_u (data layout only).  Returns a new dict with
    'uoff' (nf + 1): the first u unknown owned by each fracture."""
    import scipy.sparse as sp
    nh, nu, nf = w["nh"], w["n"], w["nf"]
    hb = np.asarray(w["hblk"], dtype=np.int64)
    blk = np.searchsorted(hb, np.arange(nh), side="right") - 1
    crp, cci, _ = w["C"]
    rows = np.repeat(np.arange(nh), np.diff(crp))
    own = np.full(nu, nf, dtype=np.int64)
    np.minimum.at(own, cci, blk[rows])
    perm = np.argsort(own, kind="stable")          # new -> old
    inv = np.empty(nu, dtype=np.int64)
    inv[perm] = np.arange(nu)
    uoff = np.searchsorted(own[perm], np.arange(nf + 1), side="left").astype(np.int64)

    def recol(t, ncols):
        rp, ci, v = t
        M = sp.csr_matrix((v, inv[ci], rp), shape=(len(rp) - 1, ncols))
        M.sort_indices()
        return (M.indptr.astype(np.int32), M.indices.astype(np.int32), M.data.astype(np.float64))
    grp, gci, gv = w["Gu"]
    Gu = sp.csr_matrix((gv, gci, grp), shape=(nu, nu))[perm][:, perm].tocsr()
    Gu.sort_indices()
    out = dict(w, C=recol(w["C"], nu), B=recol(w["B"], nu),
               Gu=(Gu.indptr.astype(np.int32), Gu.indices.astype(np.int32), Gu.data.astype(np.float64)),
               b=np.asarray(w["b"])[perm], uoff=uoff, name=w["name"] + "_owner")
    return out


def tab_epsil_diag(n: int = 100_000, seed: int = 42):
    """The diagonal test of Table tab:epsil: A_ii = i, i = 1..1e5.

    Right-hand side "random": uniform[0,1) from default_rng(42) (Appendix A.2
    of SURVEY.md reproduces the paper's iteration column exactly with this draw)."""
    rowptr = np.arange(n + 1, dtype=np.int32)
    colidx = np.arange(n, dtype=np.int32)
    vals = np.arange(1, n + 1, dtype=np.float64)
    b = np.random.default_rng(seed).random(n)
    return dict(kind="csr", name="tab_epsil_diag", n=n, rowptr=rowptr, colidx=colidx, vals=vals, b=b)


LANCZOS_SEED = 0x5EED


def lanczos_start(n: int, offset: int = 0, seed: int = LANCZOS_SEED) -> np.ndarray:
    """Start vector of the spectrum estimate (reading A11): uniform[-1, 1) from a counter-based
    splitmix64 hash of (seed, global row index + 1), so any row partition draws the same
    vector.  libnpc implements the same generator on the device (npc_estimate_spectrum with
    v0 = NULL); both sides consume it as an input."""
    M = np.uint64(0xFFFFFFFFFFFFFFFF)
    i = np.arange(offset + 1, offset + n + 1, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = (np.uint64(seed) + np.uint64(0x9E3779B97F4A7C15) * i) & M
        z = ((z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)) & M
        z = ((z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)) & M
        z = z ^ (z >> np.uint64(31))
    return 2.0 * ((z >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)) - 1.0


def laplacian_1d_csr(n: int):
    """tridiag(-1, 2, -1) of size n (Dirichlet), CSR."""
    return grid_laplacian_csr((n,), 2.0, -1.0)


def random_spd_dense(n: int, seed: int, cond: float = 1e3):
    """Dense SPD matrix Q diag(l) Q^T with log-uniform spectrum in [1, cond]."""
    rng = np.random.default_rng(seed)
    Q, _ = np.linalg.qr(rng.standard_normal((n, n)))
    lam = np.exp(rng.uniform(0.0, np.log(cond), n))
    lam[0], lam[-1] = 1.0, cond
    A = (Q * lam) @ Q.T
    return 0.5 * (A + A.T), lam


def dense_to_csr(A: np.ndarray):
    """Dense -> CSR with every entry stored (ascending columns)."""
    n = A.shape[0]
    rowptr = (np.arange(n + 1, dtype=np.int64) * n).astype(np.int32)
    colidx = np.tile(np.arange(n, dtype=np.int32), n)
    return rowptr, colidx, np.ascontiguousarray(A, dtype=np.float64).ravel()


def pcg_replacement_case(scale: float, seed: int = 11):
    """Crafted PCG input for the residual-replacement branch (reading A23): a 30 x 30 dense
    SPD matrix with spectrum in [1, 10] (as CSR), b ~ U[-1,1], and x0 = x* + scale * N(0,1):
    with ||A x0|| >> ||b||, b - A x carries an absolute rounding error ~eps ||A|| ||x0|| that
    the recursive residual does not see.  Returns (workload dict, x0)."""
    n = 30
    A, _ = random_spd_dense(n, seed, cond=10.0)
    rowptr, colidx, vals = dense_to_csr(A)
    rng = np.random.default_rng(seed + 1)
    b = rng.uniform(-1.0, 1.0, n)
    xs = np.linalg.solve(A, b)
    x0 = xs + scale * rng.standard_normal(n)
    return dict(kind="csr", name=f"replacement_{scale:g}", n=n, rowptr=rowptr, colidx=colidx, vals=vals,
                b=b, dense=A), x0


def pcg_floor_case(seed: int = 21):
    """Crafted PCG input whose true relative residual has a floor ~2e-7 (reading A23's cap):
    a 30 x 30 dense SPD matrix with one eigenvalue 1e-8 and the rest in [1, 10], b mostly
    along the 1e-8 eigenvector (so x* ~ 1e8 b).  Returns a workload dict (x0 = 0)."""
    n = 30
    rng = np.random.default_rng(seed)
    Q, _ = np.linalg.qr(rng.standard_normal((n, n)))
    lam = np.concatenate([[1e-8], np.linspace(1.0, 10.0, n - 1)])
    A = (Q * lam) @ Q.T
    A = 0.5 * (A + A.T)
    rowptr, colidx, vals = dense_to_csr(A)
    return dict(kind="csr", name="floor", n=n, rowptr=rowptr, colidx=colidx, vals=vals,
                b=Q[:, 0] + 1e-3 * rng.standard_normal(n), dense=A)
