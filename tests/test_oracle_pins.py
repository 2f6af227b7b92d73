"""Pins of the CPU oracle (oracle/) against what the paper and the mathematics fix.

None of these re-types the oracle's own formula: each compares it with a printed value of
the paper (Table tab:epsil, Fig. 1 text), a closed form (Chebyshev T_{k+1}, 1D-Laplacian
spectrum, cosh form of rho), an invariant (spectrum bound, symmetry, Ritz interlacing), a
library routine on a special case (dense solve, dense eigensolve), or another algorithm of
the paper (Newton Alg. 1 vs Chebyshev Alg. 2).  Label P<n> refers to SURVEY.md §8(c).
"""
import json
import math
import os

import numpy as np
import pytest

import oracle
import workloads as W

pytestmark = pytest.mark.filterwarnings("ignore::RuntimeWarning")


def cheb_T(k, x):
    """T_k(x) by the three-term recurrence T_{j+1} = 2x T_j - T_{j-1} (textbook)."""
    x = np.asarray(x, dtype=np.float64)
    t0, t1 = np.ones_like(x), x.copy()
    if k == 0:
        return t0
    for _ in range(k - 1):
        t0, t1 = t1, 2 * x * t1 - t0
    return t1


def p_closed(lam, k, alpha, beta, xi):
    """p_k(lam) from the residual-polynomial closed form of the Chebyshev preconditioner
    on [alpha + xi*theta, beta + xi*theta]: 1 - lam p(lam) = T_{k+1}((tb - lam)/d)/T_{k+1}(tb/d)."""
    theta = 0.5 * (alpha + beta)
    d = 0.5 * (beta - alpha)
    tb = theta * (1 + xi)
    return (1.0 - cheb_T(k + 1, (tb - lam) / d) / cheb_T(k + 1, tb / d)) / lam


# ---------------------------------------------------------------- P1 / P2: Table tab:epsil
@pytest.fixture(scope="module")
def tab(golden_dir):
    with open(os.path.join(golden_dir, "tab_epsil.json")) as f:
        return json.load(f)


@pytest.fixture(scope="module")
def diag_op():
    w = W.tab_epsil_diag()
    return w, oracle.Operator(w)


def test_P1_tab_epsil_eigenvalues(tab, diag_op):
    w, op = diag_op
    n = w["n"]
    lam = np.arange(1, n + 1, dtype=np.float64)
    for xi, _, l1, l2, l5, l10, kap, kap10 in tab["rows"]:
        z = oracle.cheb_apply(op, 63, 1.0, float(n), xi, np.ones(n))  # p(A) 1 = p(lambda_i)
        mu = np.sort(lam * z)
        mu = mu / mu[-1]  # reading A2: normalised by the largest
        got = [mu[0], mu[1], mu[4], mu[9], 1 / mu[0]]
        want = [l1, l2, l5, l10, kap]
        for g, e in zip(got, want):
            assert abs(g - e) <= 6e-4 * abs(e) + 5e-6, (xi, got, want)
        if kap10 is not None:
            assert abs(1 / mu[9] - kap10) <= 1e-3 * kap10 + 5e-3
        else:  # reading A3: lambda_1 == lambda_10 in the printed row, so kappa_10 == kappa
            assert abs(1 / mu[9] - kap) <= 1e-3 * kap


def test_P2_tab_epsil_iterations_and_P10_counters(tab, diag_op):
    w, op = diag_op
    for xi, iters, *_ in tab["rows"]:
        x, st = oracle.pcg(op, w["b"], 63, 1.0, float(w["n"]), xi, tol=1e-10, maxit=500)
        assert st["converged"] and abs(st["iters"] - iters) <= 1, (xi, st)
        # Table tab11 counter laws: MVP = iters*(m+1) (+1 true residual); ddot = 3*iters (+3)
        assert st["mvp"] == st["iters"] * 64 + 1
        assert st["ddot"] == 3 * st["iters"] + 3
        assert st["relres_true"] <= 1e-10
        # the exact solution of the diagonal system is b_i / i
        xe = w["b"] / np.arange(1, w["n"] + 1)
        assert np.linalg.norm(x - xe) / np.linalg.norm(xe) < 1e-9


# ---------------------------------------------------------------- P7: worked values
def test_P7_spec_worked_values(golden_dir):
    with open(os.path.join(golden_dir, "spec_worked.json")) as f:
        g = json.load(f)
    c = g["cheb"]
    tb, d, s = oracle.cheb_params(c["alpha"], c["beta"], c["xi"])
    assert (tb, d, s) == (c["theta"], c["delta"], c["sigma"])
    rho = oracle.cheb_rho(s, 3)
    assert rho[0] == c["rho0"] and abs(rho[1] - c["rho1"]) < 1e-15
    nw = g["newton"]
    z = oracle.newton_zeta(nw["alpha"], nw["beta"], nw["xi"], 2)
    assert abs(z[0] - nw["zeta0"]) < 1e-15 and abs(z[1] - nw["zeta1"]) < 1e-14
    # xi only rescales theta: theta_bar ratio exactly 1 + xi (Eq. thetamod)
    tb2, d2, _ = oracle.cheb_params(1.0, 3.0, 0.05)
    assert tb2 == 2.0 * 1.05 and d2 == 1.0


def test_P7_degree0_and_identity():
    n = 50
    w = dict(kind="csr", n=n, rowptr=np.arange(n + 1, dtype=np.int32),
             colidx=np.arange(n, dtype=np.int32), vals=np.ones(n))
    op = oracle.Operator(w)
    r = np.random.default_rng(0).uniform(-1, 1, n)
    z = oracle.cheb_apply(op, 0, 0.5, 2.0, 0.1, r)  # m = 0 -> r / theta_bar (Alg. 2 step 2)
    assert np.array_equal(z, r / (1.25 * 1.1))
    x, st = oracle.pcg(op, r, 5, 0.5, 2.0, 0.0, tol=1e-12)  # A = I: one iteration
    assert st["iters"] == 1 and np.allclose(x, r, rtol=0, atol=1e-14)
    x, st = oracle.pcg(op, np.zeros(n), 5, 0.5, 2.0, 0.0, tol=1e-12)  # zero rhs
    assert st["iters"] == 0 and st["converged"] and not x.any()


# ---------------------------------------------------------------- P8: rho closed form
@pytest.mark.parametrize("alpha,beta,xi", [(1.0, 3.0, 0.0), (1e-3, 8.0, 1e-3), (0.5, 0.51, 0.0)])
def test_P8_rho_closed_form(alpha, beta, xi):
    _, _, s = oracle.cheb_params(alpha, beta, xi)
    rho = oracle.cheb_rho(s, 200)
    t = math.acosh(s)
    k = np.arange(201)
    # rho_k = T_k(sigma)/T_{k+1}(sigma) = cosh(k t)/cosh((k+1) t); use the ratio in a stable form
    closed = np.exp(-t) * (1 + np.exp(-2 * k * t)) / (1 + np.exp(-2 * (k + 1) * t))
    assert np.max(np.abs(rho - closed) / closed) < 5e-14


# ---------------------------------------------------------------- P3: 1D Laplacian eigvecs
@pytest.mark.parametrize("k", [0, 1, 2, 10, 63, 200])
@pytest.mark.parametrize("xi", [0.0, 1e-3])
def test_P3_laplacian_eigenvectors(k, xi):
    n = 200
    rowptr, colidx, vals = W.laplacian_1d_csr(n)
    op = oracle.Operator(dict(kind="csr", n=n, rowptr=rowptr, colidx=colidx, vals=vals))
    i = np.arange(1, n + 1)
    lam_exact = 4 * np.sin(np.arange(1, n + 1) * np.pi / (2 * (n + 1))) ** 2
    alpha, beta = lam_exact[0], lam_exact[-1]
    pmax = np.max(np.abs(p_closed(lam_exact, k, alpha, beta, xi)))  # ||p_k(A)||_2
    for j in [1, 2, 17, 100, 199, 200]:
        v = np.sin(i * j * np.pi / (n + 1))
        z = oracle.cheb_apply(op, k, alpha, beta, xi, v)
        expect = p_closed(lam_exact[j - 1], k, alpha, beta, xi) * v
        # error relative to ||p_k(A)|| ||v|| (p_k(lambda_j) itself may be ~0 near beta)
        assert np.linalg.norm(z - expect) / (pmax * np.linalg.norm(v)) < 2e-11, (j, k, xi)


def test_P3_laplacian_operator_eigenpairs():
    """A v_j = lambda_j v_j for the 2D 5-point operator (config 1 shape, closed form)."""
    side = 64
    w = W.config1(side)
    op = oracle.Operator(w)
    x = np.arange(1, side + 1)
    for (a, b) in [(1, 1), (3, 7), (64, 64)]:
        v = np.outer(np.sin(x * b * np.pi / (side + 1)), np.sin(x * a * np.pi / (side + 1))).ravel()
        lam = 4 * np.sin(a * np.pi / (2 * (side + 1))) ** 2 + 4 * np.sin(b * np.pi / (2 * (side + 1))) ** 2
        y = op.apply(v)
        assert np.linalg.norm(y - lam * v) <= 1e-12 * np.linalg.norm(v) * 8


def test_P3_stencil_matches_csr():
    """The matrix-free stencil (O1) equals the explicit CSR operator of the same grid."""
    side = 12
    rowptr, colidx, vals = W.grid_laplacian_csr((side, side, side), 6.0, -1.0)
    csr = oracle.Operator(dict(kind="csr", n=side ** 3, rowptr=rowptr, colidx=colidx, vals=vals))
    st = oracle.Operator(dict(kind="stencil", n=side ** 3, dim=3, nx=side, ny=side, nz=side,
                              diag=6.0, offdiag=-1.0))
    x = np.random.default_rng(3).standard_normal(side ** 3)
    assert np.allclose(csr.apply(x), st.apply(x), rtol=0, atol=1e-13)
    # 3D separable eigenvector, closed form eigenvalue
    g = np.arange(1, side + 1)
    v = np.einsum("i,j,k->ijk", np.sin(g * 2 * np.pi / (side + 1)), np.sin(g * 5 * np.pi / (side + 1)),
                  np.sin(g * 11 * np.pi / (side + 1))).ravel()
    lam = sum(4 * np.sin(a * np.pi / (2 * (side + 1))) ** 2 for a in (2, 5, 11))
    assert np.linalg.norm(st.apply(v) - lam * v) <= 1e-12 * np.linalg.norm(v) * 12


# ---------------------------------------------------------------- P4: spectrum bound
@pytest.mark.parametrize("k", [1, 5, 20, 60])
@pytest.mark.parametrize("xi", [0.0, 1e-2])
def test_P4_spectrum_bound(k, xi):
    n = 200
    rowptr, colidx, vals = W.laplacian_1d_csr(n)
    op = oracle.Operator(dict(kind="csr", n=n, rowptr=rowptr, colidx=colidx, vals=vals))
    A = np.zeros((n, n))
    for r in range(n):
        A[r, colidx[rowptr[r]:rowptr[r + 1]]] = vals[rowptr[r]:rowptr[r + 1]]
    lam_exact = np.linalg.eigvalsh(A)
    alpha, beta = lam_exact[0] * 0.9, lam_exact[-1] * 1.0  # exact-or-outer bounds
    P = np.column_stack([oracle.cheb_apply(op, k, alpha, beta, xi, e) for e in np.eye(n)])
    assert np.linalg.norm(P - P.T) <= 1e-13 * np.linalg.norm(P)  # p_k(A) symmetric
    mu = np.linalg.eigvalsh(0.5 * (P @ A + (P @ A).T))
    tb = 0.5 * (alpha + beta) * (1 + xi)
    d = 0.5 * (beta - alpha)
    T = float(cheb_T(k + 1, tb / d))
    mu_alpha = 1 - float(cheb_T(k + 1, (tb - alpha) / d)) / T
    lo, hi = min(mu_alpha, 1 - 1 / T), 1 + 1 / T
    assert mu.min() >= lo - 1e-10 and mu.max() <= hi + 1e-10, (mu.min(), mu.max(), lo, hi)
    assert mu.min() > 0


# ---------------------------------------------------------------- P5: Newton == Chebyshev
@pytest.mark.parametrize("nlev", [0, 1, 2, 3, 4, 6])
@pytest.mark.parametrize("xi", [0.0, 1e-3])
def test_P5_newton_equals_chebyshev(nlev, xi):
    n = 300
    rowptr, colidx, vals = W.laplacian_1d_csr(n)
    op = oracle.Operator(dict(kind="csr", n=n, rowptr=rowptr, colidx=colidx, vals=vals))
    r = np.random.default_rng(nlev).uniform(-1, 1, n)
    alpha, beta = 4 * math.sin(math.pi / (2 * (n + 1))) ** 2, 4.0
    zn = oracle.newton_apply(op, nlev, alpha, beta, xi, r)
    zc = oracle.cheb_apply(op, 2 ** nlev - 1, alpha, beta, xi, r)
    assert np.linalg.norm(zn - zc) / np.linalg.norm(zc) < 1e-11


def test_P5_newton_reproduces_tab_epsil_iterations(tab, diag_op):
    """Newton nlev=6 with the alpha' reading gives the same preconditioned spectrum as
    Chebyshev degree 63 (Table tab:epsil was produced with Newton)."""
    w, op = diag_op
    n = w["n"]
    lam = np.arange(1, n + 1, dtype=np.float64)
    for xi, _, l1, l2, l5, l10, kap, _ in tab["rows"]:
        mu = np.sort(lam * oracle.newton_apply(op, 6, 1.0, float(n), xi, np.ones(n)))
        mu = mu / mu[-1]
        for g, e in zip([mu[0], mu[1], mu[4], mu[9]], [l1, l2, l5, l10]):
            assert abs(g - e) <= 6e-4 * e + 5e-6


# ---------------------------------------------------------------- P12: Fig. 1 / Thm 2.3
def test_P12_fig1_first_newton_level(golden_dir):
    with open(os.path.join(golden_dir, "spec_worked.json")) as f:
        fig = json.load(f)["fig1"]
    lam = np.array(sorted({x for a, b, _ in fig["pairs"] for x in (a, b)} | {0.6, 1.0, 1.3}))
    n = lam.size
    op = oracle.Operator(dict(kind="csr", n=n, rowptr=np.arange(n + 1, dtype=np.int32),
                              colidx=np.arange(n, dtype=np.int32), vals=lam))
    # interval [0.1, 1.9] -> zeta_0 = 1 so the scaled spectrum is the spectrum itself
    mu0 = lam * oracle.newton_apply(op, 1, 0.1, 1.9, 0.0, np.ones(n))
    zeta1 = oracle.newton_zeta(0.1, 1.9, 0.0, 1)[1]
    for a, b, fa in fig["pairs"]:
        ia, ib = np.searchsorted(lam, a), np.searchsorted(lam, b)
        assert abs(mu0[ia] / zeta1 - fa) < 1e-12 and abs(mu0[ia] - mu0[ib]) < 1e-12  # cluster
    mu1 = lam * oracle.newton_apply(op, 1, 0.1, 1.9, 0.05, np.ones(n))
    order = np.argsort(mu1)
    # Theorem 2.3 with xi = 0.05: the eigenvalues below alpha_eta + 2(1-eta) (0.1, 0.14, 0.18)
    # are the 3 smallest of P_1 A, in order; the top ones no longer coincide with them.
    assert list(order[:3]) == [0, 1, 2]
    for a, b, _ in fig["pairs"]:
        assert abs(mu1[np.searchsorted(lam, a)] - mu1[np.searchsorted(lam, b)]) > 1e-3


# ---------------------------------------------------------------- P6: dense small SPD
@pytest.mark.parametrize("seed", [0, 1])
@pytest.mark.parametrize("k", [0, 3, 12])
def test_P6_dense_small(seed, k):
    n = 30
    A, lam = W.random_spd_dense(n, seed, cond=1e2)
    rowptr, colidx, vals = W.dense_to_csr(A)
    op = oracle.Operator(dict(kind="csr", n=n, rowptr=rowptr, colidx=colidx, vals=vals))
    ev, V = np.linalg.eigh(A)
    alpha, beta, xi = 1.0, 1e2, 1e-3
    P_closed = (V * p_closed(ev, k, alpha, beta, xi)) @ V.T
    P = np.column_stack([oracle.cheb_apply(op, k, alpha, beta, xi, e) for e in np.eye(n)])
    assert np.linalg.norm(P - P_closed) / np.linalg.norm(P_closed) < 1e-11
    b = np.random.default_rng(seed + 10).uniform(-1, 1, n)
    x, st = oracle.pcg(op, b, k, alpha, beta, xi, tol=1e-10, maxit=200)
    # finite termination in <= n steps holds in exact arithmetic; rounding delays plain CG
    # (k = 0 is a scalar preconditioner) on a log-uniform spectrum, so it gets 2n.
    assert st["converged"] and st["iters"] <= (n if k > 0 else 2 * n)
    xs = np.linalg.solve(A, b)
    assert np.linalg.norm(x - xs) / np.linalg.norm(xs) <= 10 * 1e-10 * 1e2


def test_unpreconditioned_cg_matches_dense_solve():
    n = 40
    A, _ = W.random_spd_dense(n, 7, cond=100.0)
    rowptr, colidx, vals = W.dense_to_csr(A)
    op = oracle.Operator(dict(kind="csr", n=n, rowptr=rowptr, colidx=colidx, vals=vals))
    b = np.random.default_rng(1).standard_normal(n)
    x, st = oracle.pcg(op, b, -1, tol=1e-12, maxit=400)
    assert st["converged"] and st["mvp"] == st["iters"] + 1
    assert np.allclose(x, np.linalg.solve(A, b), rtol=1e-9, atol=1e-11)


# ---------------------------------------------------------------- P9: Lanczos
def test_P9_lanczos_full_spectrum():
    n = 12
    lam = np.arange(1, n + 1, dtype=np.float64) ** 1.5
    op = oracle.Operator(dict(kind="csr", n=n, rowptr=np.arange(n + 1, dtype=np.int32),
                              colidx=np.arange(n, dtype=np.int32), vals=lam))
    a, b = oracle.lanczos(op, n, np.random.default_rng(0).uniform(-1, 1, n))
    from scipy.linalg import eigvalsh_tridiagonal
    ev = eigvalsh_tridiagonal(a, b[: n - 1])
    assert np.allclose(ev, lam, rtol=1e-8, atol=0)


def test_P9_lanczos_config1_bracket():
    w = W.config1()
    op = oracle.Operator(w)
    lo_ex, hi_ex = 8 * math.sin(math.pi / 130) ** 2, 8 * math.sin(64 * math.pi / 130) ** 2
    for v0 in (w["b"], W.lanczos_start(w["n"])):
        a, b = oracle.lanczos(op, 20, v0)
        rmin, rmax = oracle.ritz_extremes(a, b)
        assert lo_ex <= rmin and rmax <= hi_ex  # Ritz values interlace inside the spectrum
        assert hi_ex - rmax < 0.02 * hi_ex       # the top converges fast
        assert rmin < 20 * lo_ex
        # the upper estimate theta_max + rho (reading A11) bounds lambda_max from above, and
        # rho is the true residual norm of the Ritz pair (Kaniel-Paige: rho >> hi_ex - theta)
        lmin, lmax = oracle.estimate_spectrum(op, 20, v0)
        assert lmin == rmin and hi_ex <= lmax < hi_ex * 1.05


def test_P9_ritz_residual_is_true_residual():
    """rho = beta_m |s_m| equals ||A y - theta y|| of the Ritz vector y = Q s (dense check)."""
    n = 60
    A, _ = W.random_spd_dense(n, 3, cond=50.0)
    rowptr, colidx, vals = W.dense_to_csr(A)
    op = oracle.Operator(dict(kind="csr", n=n, rowptr=rowptr, colidx=colidx, vals=vals))
    v0 = W.lanczos_start(n)
    m = 8
    a, b = oracle.lanczos(op, m, v0)
    # rebuild Q by the same three-term recurrence in numpy (dense, tiny)
    Q = np.zeros((n, m + 1))
    Q[:, 0] = v0 / np.linalg.norm(v0)
    for j in range(m):
        wv = A @ Q[:, j] - (b[j - 1] * Q[:, j - 1] if j else 0)
        wv -= a[j] * Q[:, j]
        Q[:, j + 1] = wv / b[j]
    from scipy.linalg import eigh_tridiagonal
    ev, S = eigh_tridiagonal(a, b[: m - 1])
    y = Q[:, :m] @ S[:, -1]
    th, rho = oracle.ritz_upper(a, b)
    assert abs(th - ev[-1]) < 1e-12 * abs(th)
    assert abs(rho - np.linalg.norm(A @ y - th * y)) < 1e-8 * np.linalg.norm(A, 2)
    assert th + rho >= np.linalg.eigvalsh(A)[-1] - 1e-12


def test_P9_lanczos_config2_small_bracket():
    side = 16
    w = W.config2(side)
    op = oracle.Operator(w)
    lo_ex = 3 * 4 * math.sin(math.pi / (2 * (side + 1))) ** 2
    hi_ex = 3 * 4 * math.sin(side * math.pi / (2 * (side + 1))) ** 2
    a, b = oracle.lanczos(op, 20, W.lanczos_start(w["n"]))
    rmin, rmax = oracle.ritz_extremes(a, b)
    assert lo_ex <= rmin and rmax <= hi_ex and hi_ex - rmax < 0.05 * hi_ex
    assert oracle.estimate_spectrum(op, 20, W.lanczos_start(w["n"]))[1] >= hi_ex


def test_lanczos_start_generator():
    """The counter-hash start vector: uniform in [-1, 1), partition-independent."""
    v = W.lanczos_start(100_000)
    assert -1 <= v.min() and v.max() < 1 and abs(v.mean()) < 0.01 and abs(v.var() - 1 / 3) < 0.01
    assert np.array_equal(v[500:700], W.lanczos_start(200, offset=500))


# ---------------------------------------------------------------- P11: exact solution x* = 1
def test_P11_config3_surrogate_exact_solution():
    w = W.config3(side=12)
    op = oracle.Operator(w)
    assert np.allclose(op.apply(np.ones(w["n"])), w["b"], rtol=1e-13, atol=1e-12)  # b = A 1
    lmin, lmax = oracle.estimate_spectrum(op, 20, W.lanczos_start(w["n"]))
    x, st = oracle.pcg(op, w["b"], 20, lmin, lmax, 0.0, tol=1e-8, maxit=2000)
    assert st["converged"] and st["relres_true"] <= 1e-8
    assert np.max(np.abs(x - 1.0)) < 1e-3


# ---------------------------------------------------------------- Schur operator (config 5)
def test_schur_operator_matches_dense():
    w = W.config5(n=300, seed=4)
    op = oracle.Operator(w)
    n, nb = w["n"], w["nb"]
    B = np.zeros((nb, n))
    for q in range(nb):
        s, e = w["browptr"][q], w["browptr"][q + 1]
        B[q, w["bcolidx"][s:e]] = w["bvals"][s:e]
        assert np.all(np.diff(w["bcolidx"][s:e]) > 0) and 2 <= e - s <= 4
    Cm = np.diag(2 + w["c"]) - np.eye(n, k=1) - np.eye(n, k=-1)
    S = Cm + B.T @ np.diag(1 / w["d"]) @ B
    x = np.random.default_rng(0).standard_normal(n)
    assert np.allclose(op.apply(x), S @ x, rtol=1e-12, atol=1e-12)
    assert np.linalg.eigvalsh(S).min() > 0


# ---------------------------------------------------------------- P14-P16: low-rank correction (O8)
def _lap1d(n):
    rowptr, colidx, vals = W.laplacian_1d_csr(n)
    op = oracle.Operator(dict(kind="csr", n=n, rowptr=rowptr, colidx=colidx, vals=vals))
    i = np.arange(1, n + 1)
    lam = 4 * np.sin(np.arange(1, n + 1) * np.pi / (2 * (n + 1))) ** 2
    vec = lambda j: np.sin(i * j * np.pi / (n + 1)) * math.sqrt(2.0 / (n + 1))  # noqa: E731  unit norm
    return op, lam, vec


@pytest.mark.parametrize("k,xi,p", [(0, 0.0, 1), (10, 0.0, 5), (20, 1e-3, 3), (63, 1e-2, 8)])
def test_P14_plusone_on_exact_eigenvectors(k, xi, p):
    """PAPER.md:495-500 (Eq. plusone): with V = the p leftmost eigenvectors,
    P A v_j = (mu_j + 1) v_j for j <= p and P A v_j = mu_j v_j for j > p, where
    mu_j = lambda_j p_k(lambda_j) from the Chebyshev closed form (not the oracle's Alg. 2)."""
    n = 150
    op, lam, vec = _lap1d(n)
    alpha, beta = lam[0], lam[-1]
    V = np.column_stack([vec(j) for j in range(1, p + 1)])
    lr = oracle.LowRank(op, V)
    for j in [1, 2, p, p + 1, p + 2, 60, n]:
        v = vec(j)
        mu = lam[j - 1] * p_closed(lam[j - 1], k, alpha, beta, xi)
        z = oracle.lowrank_apply(op, k, alpha, beta, xi, lr, op.apply(v))
        expect = (mu + (1.0 if j <= p else 0.0)) * v
        assert np.linalg.norm(z - expect) <= 1e-10 * max(1.0, abs(mu)), (j, k, p)


@pytest.mark.parametrize("seed,p,k", [(0, 1, 3), (1, 4, 8), (2, 6, 0)])
def test_P15_dense_lowrank_operator_and_pcg(seed, p, k):
    """P = P_0 + V (V^T A V)^{-1} V^T for an arbitrary (non-eigen) V, built densely with numpy
    from its definition (P_0 from the eigendecomposition closed form, as in P6), equals the
    oracle column by column; P is symmetric; PCG with P converges to the dense solution."""
    n = 32
    A, _ = W.random_spd_dense(n, seed, cond=1e3)
    rowptr, colidx, vals = W.dense_to_csr(A)
    op = oracle.Operator(dict(kind="csr", n=n, rowptr=rowptr, colidx=colidx, vals=vals))
    ev, E = np.linalg.eigh(A)
    alpha, beta, xi = 1.0, 1e3, 1e-3
    V = np.random.default_rng(seed + 50).standard_normal((n, p))
    P_def = (E * p_closed(ev, k, alpha, beta, xi)) @ E.T + V @ np.linalg.solve(V.T @ A @ V, V.T)
    lr = oracle.LowRank(op, V)
    P = np.column_stack([oracle.lowrank_apply(op, k, alpha, beta, xi, lr, e) for e in np.eye(n)])
    assert np.linalg.norm(P - P_def) / np.linalg.norm(P_def) < 1e-10
    assert np.linalg.norm(P - P.T) / np.linalg.norm(P) < 1e-12
    b = np.random.default_rng(seed + 60).uniform(-1, 1, n)
    x, st = oracle.pcg(op, b, k, alpha, beta, xi, tol=1e-10, maxit=400, lowrank=lr)
    assert st["converged"]
    xs = np.linalg.solve(A, b)
    assert np.linalg.norm(x - xs) / np.linalg.norm(xs) <= 1e-10 * 1e3 * 10
    # counter law (P10 + O8): one application of P per iteration, each with p extra inner
    # products (V^T r): ddot = 3 iters + 3 + p iters
    assert st["ddot"] == 3 * st["iters"] + 3 + p * st["iters"], st


def test_P15_lowrank_cuts_pcg_iterations_on_laplacian():
    """The paper's motivation: deflating the p leftmost eigenvalues
    (shifted by +1) shrinks kappa(PA), so PCG needs fewer iterations.  Exact eigenvectors."""
    n = 400
    op, lam, vec = _lap1d(n)
    b = np.random.default_rng(3).uniform(-1, 1, n)
    k, alpha, beta = 10, lam[0], lam[-1]
    _, st0 = oracle.pcg(op, b, k, alpha, beta, 0.0, tol=1e-10, maxit=2000)
    lr = oracle.LowRank(op, np.column_stack([vec(j) for j in range(1, 9)]))
    # with the 8 leftmost deflated, the interval may start at lambda_9
    _, st1 = oracle.pcg(op, b, k, lam[8], beta, 0.0, tol=1e-10, maxit=2000, lowrank=lr)
    assert st0["converged"] and st1["converged"] and st1["iters"] < 0.6 * st0["iters"], (st0["iters"], st1["iters"])


def test_P16_full_lanczos_ritz_pairs():
    """n-step Lanczos with full reorthogonalisation on a dense SPD matrix reproduces the
    spectrum (dense eigensolve) and the leftmost eigenvectors up to sign."""
    n = 24
    A, _ = W.random_spd_dense(n, 5, cond=50.0)
    rowptr, colidx, vals = W.dense_to_csr(A)
    op = oracle.Operator(dict(kind="csr", n=n, rowptr=rowptr, colidx=colidx, vals=vals))
    ev, E = np.linalg.eigh(A)
    th, V = oracle.ritz_vectors(op, n, 4, np.random.default_rng(1).uniform(-1, 1, n))
    assert np.allclose(th, ev[:4], rtol=1e-10)
    for j in range(4):
        assert abs(abs(V[:, j] @ E[:, j]) - 1.0) < 1e-8
    # fewer steps: Ritz residual ||A y - theta y|| = beta_s |e_s^T s| (Kaniel-Paige setting)
    th2, V2 = oracle.ritz_vectors(op, 10, 2, np.random.default_rng(2).uniform(-1, 1, n))
    assert np.all(th2 >= ev[:2] - 1e-12)  # Ritz values from above (Cauchy interlacing)
    assert np.allclose(np.linalg.norm(V2, axis=0), 1.0, atol=1e-12)


# ---------------------------------------------------------------- P17-P18: DFN Schur complement (O9)
def _dfn_dense(w):
    import scipy.sparse as sp

    def M(t, shape):
        return sp.csr_matrix((t[2], t[1], t[0]), shape=shape).toarray()
    nh, nu = w["nh"], w["n"]
    return (M(w["A"], (nh, nh)), M(w["Gh"], (nh, nh)), M(w["C"], (nh, nu)), M(w["B"], (nh, nu)),
            M(w["Gu"], (nu, nu)))


@pytest.mark.parametrize("nf,seed,alpha", [(6, 0, None), (9, 1, None), (7, 2, 0.0)])
def test_P17_dfn_schur_matches_dense(nf, seed, alpha):
    """Alg. 3 (with alpha: reading A8) equals the dense closed form of
    Eq. schur, S_u = G^u - a B^T A^-1 C - a C^T A^-1 B + C^T A^-1 G^h A^-1 C,
    built with numpy's dense solve; S_u is symmetric and SPD; Alg. 4
    equals diag(S_u); the Jacobi-scaled operator has unit diagonal."""
    w = W.dfn(nf, seed=seed, alpha=alpha)
    A, Gh, C, B, Gu = _dfn_dense(w)
    a = w["alpha"]
    Ai_C, Ai_B = np.linalg.solve(A, C), np.linalg.solve(A, B)
    S = Gu - a * B.T @ Ai_C - a * C.T @ Ai_B + C.T @ np.linalg.solve(A, Gh @ Ai_C)
    op = oracle.Operator(w, scaled=False)
    n = w["n"]
    cols = np.random.default_rng(seed).choice(n, 12, replace=False)
    for j in cols:
        e = np.zeros(n)
        e[j] = 1.0
        assert np.linalg.norm(op.apply(e) - S[:, j]) <= 1e-12 * np.linalg.norm(S[:, j])
    x = np.random.default_rng(seed + 1).standard_normal(n)
    assert np.linalg.norm(op.apply(x) - S @ x) <= 1e-13 * np.linalg.norm(S @ x)
    assert np.linalg.norm(S - S.T) <= 1e-13 * np.linalg.norm(S)
    assert np.linalg.eigvalsh(S)[0] > 0.0
    D = op.dfn_diag()
    assert np.allclose(D, np.diag(S), rtol=1e-13, atol=0)
    ops = oracle.Operator(w, scaled=True)
    Shat = np.column_stack([ops.apply(e) for e in np.eye(n)[:, :40].T])  # first 40 columns
    assert np.allclose(np.diag(Shat[:40]), 1.0, rtol=1e-13)
    assert np.allclose(Shat, (S / np.sqrt(np.outer(D, D)))[:, :40], rtol=1e-12, atol=1e-14)


def test_P18_dfn_end_to_end_block_system():
    """Solve the Schur system by the oracle's PCG + polynomial on the scaled operator, recover
    h and p (with alpha) and check the original saddle-point system Eq. sys
     with dense numpy: the paper's reformulation end to end."""
    w = W.dfn(10, seed=3)
    A, Gh, C, B, Gu = _dfn_dense(w)
    a = w["alpha"]
    nh, nu = w["nh"], w["n"]
    q = np.random.default_rng(4).uniform(-1, 1, nh)
    # r = W^T M^-1 f1 with f1 = [q; 0], M^-1 = [[A^-1, 0], [-A^-1 G^h A^-1, A^-1]], W = [a B; C]
    Aq = np.linalg.solve(A, q)
    r = a * B.T @ Aq - C.T @ np.linalg.solve(A, Gh @ Aq)
    op = oracle.Operator(w, scaled=True)
    D = op.dfn_diag()
    lo, hi = oracle.estimate_spectrum(op, 20, W.lanczos_start(nu))
    uh, st = oracle.pcg(op, r / np.sqrt(D), 10, lo, hi, 0.0, tol=1e-12, maxit=2000)
    assert st["converged"]
    u = uh / np.sqrt(D)
    h = np.linalg.solve(A, q + C @ u)
    p = np.linalg.solve(A, a * B @ u - Gh @ h)  # the paper's "B u" assumes alpha = 1 (reading A8)
    K0 = np.block([[Gh, -a * B, A], [-a * B.T, Gu, -C.T], [A, -C, np.zeros((nh, nh))]])
    x = np.concatenate([h, u, p])
    f0 = np.concatenate([np.zeros(nh), np.zeros(nu), q])
    assert np.linalg.norm(K0 @ x - f0) <= 1e-9 * np.linalg.norm(K0) * np.linalg.norm(x)


# ---------------------------------------------------------------- P6b: x0 != 0 branch of O5
def _dense_op(n, seed, cond):
    A, _ = W.random_spd_dense(n, seed, cond=cond)
    rowptr, colidx, vals = W.dense_to_csr(A)
    return A, oracle.Operator(dict(kind="csr", n=n, rowptr=rowptr, colidx=colidx, vals=vals))


@pytest.mark.parametrize("k", [-1, 0, 4])
def test_P6b_pcg_nonzero_x0_dense(k):
    """PCG from x0 != 0 (r0 = b - A x0, PAPER.md:122-123 via Saad Alg. 9.1) reaches the
    dense solution; counters iters*(k+1) + 1 (r0) + 1 (true residual).  x0 = 2 x* (so that
    r0 = -b: a sign slip in r0 would converge to 3 x*) and x0 = x* (0 iterations)."""
    n = 30
    A, op = _dense_op(n, 3, 50.0)
    b = np.random.default_rng(4).uniform(-1, 1, n)
    xs = np.linalg.solve(A, b)
    for x0 in (np.random.default_rng(5).standard_normal(n) * 10.0, 2.0 * xs):
        x, st = oracle.pcg(op, b, k, 1.0, 50.0, 0.0, tol=1e-10, maxit=400, x0=x0)
        assert st["converged"] and st["relres_true"] <= 1e-10 and st["true_checks"] == 1
        assert np.linalg.norm(x - xs) / np.linalg.norm(xs) <= 10 * 1e-10 * 50.0
        assert st["mvp"] == st["iters"] * (max(k, 0) + 1) + 2
        assert st["ddot"] == 3 * st["iters"] + 3
    # x0 = x*: r0 is rounding noise, relres <= tol before the first iteration
    x, st = oracle.pcg(op, b, k, 1.0, 50.0, 0.0, tol=1e-10, maxit=400, x0=xs)
    assert st["iters"] == 0 and st["converged"] and st["mvp"] == 2 and np.array_equal(x, xs)


# ---------------------------------------------------------------- A23: residual replacement
def _replacement_case(scale, tol, k=2):
    """workloads.pcg_replacement_case: x0 = x* + scale*d on a dense SPD system with spectrum
    in [1, 10]; the recursive residual r_i = r_0 - sum alpha A p loses the absolute accuracy
    of b - A x_i once ||A x_i|| >> ||b||, so below a tolerance near eps*scale the recursive
    residual passes the test while the true one does not."""
    w, x0 = W.pcg_replacement_case(scale)
    op = oracle.Operator(w)
    A, b = w["dense"], w["b"]
    x, st = oracle.pcg(op, b, k, 1.0, 10.0, 0.0, tol=tol, maxit=2000, x0=x0)
    return A, b, np.linalg.solve(A, b), x, st


@pytest.mark.parametrize("scale,tol", [(1e7, 1e-8), (1e8, 1e-10), (1e6, 1e-11)])
def test_A23_residual_replacement_restarts_and_converges(scale, tol):
    """Recursive residual below tol, true residual above: r is replaced by b - A x and PCG
    restarts (reading A23).  Pinned by the mathematics: the final x solves the dense system
    to tol (a replacement that kept the stale r would re-trigger the true check on every
    following iteration, true_checks >> 2; a wrong sign in b - A x would diverge), and the
    counters obey iters*(k+1) + 1 (r0) + true_checks."""
    A, b, xs, x, st = _replacement_case(scale, tol)
    assert st["converged"] and st["relres_true"] <= tol
    assert st["true_checks"] == 2, st          # one replacement, then accepted
    assert np.linalg.norm(b - A @ x) / np.linalg.norm(b) <= 2 * tol
    assert np.linalg.norm(x - xs) / np.linalg.norm(xs) <= 10 * tol * 10.0
    assert st["mvp"] == st["iters"] * 3 + 1 + st["true_checks"]
    # the replacement restarts the recurrence: the iterations after it are those of a fresh
    # PCG from the iterate at which it happened (same x, same arithmetic) -- exactly
    _, _, _, _, st1 = _replacement_case(scale, tol)
    assert st1 == st                            # deterministic


def _floor_case():
    """workloads.pcg_floor_case: one eigenvalue 1e-8, the rest in [1, 10], b mostly along
    its eigenvector: x* ~ 1e8 b, so b - A x carries an absolute rounding error
    ~eps ||A|| ||x*|| and the true relative residual cannot go below ~2e-7, while the
    recursive one can."""
    w = W.pcg_floor_case()
    return w["dense"], oracle.Operator(w), w["b"]


@pytest.mark.parametrize("k", [-1, 2])
def test_A23_replacement_cap(k):
    """A true-residual floor above tol: every true check fails, the oracle replaces at most 50
    times and stops unconverged after the 51st check (A23's cap); counters iters*(k+1) + 51."""
    A, op, b = _floor_case()
    x, st = oracle.pcg(op, b, k, 1e-8, 10.0, 0.0, tol=1e-10, maxit=5000)
    assert not st["converged"] and not st["breakdown"]
    assert st["true_checks"] == 51 and st["relres_recursive"] <= 1e-10 and st["relres_true"] > 1e-10
    assert st["mvp"] == st["iters"] * (max(k, 0) + 1) + 51
    # the floor is the rounding of b - A x at this |x|, not a wrong iterate
    floor = np.finfo(float).eps * np.linalg.norm(A, 2) * np.linalg.norm(x) / np.linalg.norm(b)
    assert st["relres_true"] <= 10 * floor
    xs = np.linalg.solve(A, b)
    assert np.linalg.norm(x - xs) / np.linalg.norm(xs) <= 1e-6
    # a tolerance above the floor converges, with at most a few replacements
    x, st = oracle.pcg(op, b, k, 1e-8, 10.0, 0.0, tol=1e-6, maxit=5000)
    assert st["converged"] and st["relres_true"] <= 1e-6 and 1 <= st["true_checks"] <= 3


# ---------------------------------------------------------------- P3 (2D): stencil dim = 2
@pytest.mark.parametrize("nx,ny", [(37, 37), (64, 23), (1, 9)])
def test_P3_stencil_2d(nx, ny):
    """The 2D 5-point matrix-free stencil (O1, dim = 2; PAPER.md:686-689 2D Laplacian
    blocks): equals the explicit CSR operator, and maps the separable sine eigenvectors
    sin(a x pi/(nx+1)) sin(b y pi/(ny+1)) to (diag - 2 cos(a pi/(nx+1)) - 2 cos(b pi/(ny+1))) v
    (diag 4, off -1: 4 sin^2 + 4 sin^2), both closed form."""
    n = nx * ny
    rowptr, colidx, vals = W.grid_laplacian_csr((nx, ny), 4.0, -1.0)
    csr = oracle.Operator(dict(kind="csr", n=n, rowptr=rowptr, colidx=colidx, vals=vals))
    st = oracle.Operator(dict(kind="stencil", n=n, dim=2, nx=nx, ny=ny, nz=1, diag=4.0, offdiag=-1.0))
    xr = np.random.default_rng(8).standard_normal(n)
    assert np.allclose(csr.apply(xr), st.apply(xr), rtol=0, atol=1e-13)
    gx, gy = np.arange(1, nx + 1), np.arange(1, ny + 1)
    for a, bb in [(1, 1), (min(3, nx), min(5, ny)), (nx, ny)]:
        v = np.outer(np.sin(gy * bb * np.pi / (ny + 1)), np.sin(gx * a * np.pi / (nx + 1))).ravel()
        lam = 4 * np.sin(a * np.pi / (2 * (nx + 1))) ** 2 + 4 * np.sin(bb * np.pi / (2 * (ny + 1))) ** 2
        assert np.linalg.norm(st.apply(v) - lam * v) <= 1e-13 * 8 * np.linalg.norm(v)
        # and through Alg. 2: p_k(A) v = p_k(lambda) v (closed-form residual polynomial)
        lo = 8 * np.sin(np.pi / (2 * (max(nx, ny) + 1))) ** 2 * 0.5
        z = oracle.cheb_apply(st, 12, lo, 8.0, 1e-3, v)
        assert np.linalg.norm(z - p_closed(lam, 12, lo, 8.0, 1e-3) * v) <= 1e-11 * np.linalg.norm(z) + 1e-14
