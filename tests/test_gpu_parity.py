"""GPU parity: libnpc (CUDA, sm_100a) vs the CPU fp64 oracle on the same seeded inputs.

Bars (BASELINE.json north star): p_k(A) v relative 2-norm error <= 1e-10 for k <= 200; PCG
iteration count within +-2 of the oracle's textbook PCG and true relative residual <= tol.
Operator applications: relative error <= 1e-13 (only the summation order may differ).
All calls go through the C ABI (paper_2208_01339_b200 = ctypes marshalling of libnpc.so).
"""
import numpy as np
import pytest

import oracle
import workloads as W

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2208_01339_b200 as npc  # noqa: E402

POLY_TOL = 1e-10


@pytest.fixture(scope="module")
def ctx():
    c = npc.npc_context_create(0)
    yield c
    torch.cuda.synchronize()


def dev(a):
    return torch.tensor(np.asarray(a, dtype=np.float64), device="cuda")


def host(t):
    torch.cuda.synchronize()
    return t.cpu().numpy()


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


# ------------------------------------------------------------------ workloads (small sizes)
SMALL = {
    "c1": lambda: W.config1(),
    "c1_ragged": lambda: W.config1(side=37),  # 1369 rows: ragged tiles / chunks
    "c2": lambda: W.config2(side=24),
    "c2_ragged": lambda: W.config2(side=19),
    "c3": lambda: W.config3(side=20),
    "c4": lambda: W.config4(n=30_000),
    "c5": lambda: W.config5(n=20_000),
}
KINDS = {"c1": ["csr", "sell"], "c1_ragged": ["csr", "sell"], "c2": ["stencil"], "c2_ragged": ["stencil"],
         "c3": ["csr", "sell"], "c4": ["sell", "csr"], "c5": ["schur"]}
CASES = [(w, k) for w in SMALL for k in KINDS[w]]


@pytest.fixture(scope="module")
def wl():
    cache = {}

    def get(name):
        if name not in cache:
            cache[name] = SMALL[name]()
        return cache[name]
    return get


@pytest.mark.parametrize("name,kind", CASES)
def test_operator_apply(ctx, wl, name, kind):
    w = wl(name)
    op = npc.create_from_workload(ctx, w, kind)
    orc = oracle.Operator(w)
    x = np.random.default_rng(5).standard_normal(w["n"])
    y = torch.empty(w["n"], dtype=torch.float64, device="cuda")
    npc.npc_apply_operator(op, dev(x), y)
    assert rel(host(y), orc.apply(x)) <= 1e-13


@pytest.mark.parametrize("name,kind", CASES)
@pytest.mark.parametrize("k", [0, 1, 2, 3, 10, 30, 60, 100, 200])
@pytest.mark.parametrize("xi", [0.0, 1e-3])
def test_apply_poly_parity(ctx, wl, name, kind, k, xi):
    w = wl(name)
    orc = oracle.Operator(w)
    lmin, lmax = oracle.estimate_spectrum(orc, 20, W.lanczos_start(w["n"]))  # oracle's interval, both sides (A11)
    op = npc.create_from_workload(ctx, w, kind)
    poly = npc.npc_set_poly(op, k, lmin, lmax, xi)
    r = np.random.default_rng(11).uniform(-1, 1, w["n"])
    z = torch.full((w["n"],), np.nan, dtype=torch.float64, device="cuda")
    npc.npc_apply_poly(poly, dev(r), z)
    ref = oracle.cheb_apply(orc, k, lmin, lmax, xi, r)
    assert rel(host(z), ref) <= POLY_TOL, (name, kind, k, xi)


@pytest.mark.parametrize("name,kind", [("c1", "csr"), ("c2", "stencil"), ("c3", "csr"), ("c4", "sell"),
                                       ("c5", "schur"), ("c3", "sell")])
def test_lanczos_parity(ctx, wl, name, kind):
    w = wl(name)
    orc = oracle.Operator(w)
    v0 = W.lanczos_start(w["n"])
    a, b = oracle.lanczos(orc, 20, v0)
    lo_o, _ = oracle.ritz_extremes(a, b)
    th_o, rho_o = oracle.ritz_upper(a, b)
    op = npc.create_from_workload(ctx, w, kind)
    ex = npc.npc_estimate_spectrum_ex(op, 20, dev(v0))
    ex0 = npc.npc_estimate_spectrum_ex(op, 20, None)  # default start = the same counter hash
    if kind != "schur":  # Schur's B^T pass uses fp64 atomics: run-to-run rounding differs
        assert ex0 == ex
    for key in ("theta_min", "theta_max", "rho"):
        assert abs(ex0[key] - ex[key]) <= 1e-9 * abs(ex["theta_max"])
    lo, hi = npc.npc_estimate_spectrum(op, 20, None)
    if kind != "schur":
        assert lo == ex["theta_min"] and hi == ex["theta_max"] + ex["rho"]
    else:  # a third run: same bar as ex0 vs ex above
        assert abs(lo - ex["theta_min"]) <= 1e-9 * abs(ex["theta_max"])
        assert abs(hi - (ex["theta_max"] + ex["rho"])) <= 2e-9 * abs(ex["theta_max"])
    # theta_max has converged after 20 steps: unique to rounding.  theta_min and rho have not,
    # and Lanczos without reorthogonalisation amplifies rounding once orthogonality is lost,
    # so their bar is the oracle's own sensitivity to a 1e-15 relative perturbation of v0 (x20).
    assert abs(ex["theta_max"] - th_o) <= 1e-9 * abs(th_o)
    s_lo = s_rho = 0.0
    for s in range(3):
        vp = v0 * (1 + 1e-15 * np.random.default_rng(100 + s).standard_normal(w["n"]))
        ap, bp = oracle.lanczos(orc, 20, vp)
        s_lo = max(s_lo, abs(oracle.ritz_extremes(ap, bp)[0] - lo_o))
        s_rho = max(s_rho, abs(oracle.ritz_upper(ap, bp)[1] - rho_o))
    assert abs(ex["theta_min"] - lo_o) <= max(1e-8 * abs(lo_o), 20 * s_lo), (ex, lo_o, s_lo)
    assert abs(ex["rho"] - rho_o) <= max(1e-6 * abs(rho_o) + 1e-12 * th_o, 20 * s_rho), (ex, rho_o, s_rho)
    assert 0 < lo < hi


PCG_CASES = [("c1", "csr", 10, 0.0), ("c1", "csr", 10, 1e-3), ("c1", "sell", 0, 0.0), ("c2", "stencil", 30, 0.0),
             ("c3", "csr", 20, 0.0), ("c3", "csr", 50, 1e-3), ("c3", "sell", 20, 0.0), ("c4", "sell", 60, 0.0),
             ("c4", "csr", 60, 1e-3), ("c5", "schur", 10, 0.0), ("c5", "schur", 50, 0.0)]


@pytest.mark.parametrize("name,kind,k,xi", PCG_CASES)
def test_pcg_parity(ctx, wl, name, kind, k, xi):
    w = wl(name)
    tol = w["tol"]
    orc = oracle.Operator(w)
    lo_o, hi_o = oracle.estimate_spectrum(orc, 20, W.lanczos_start(w["n"]))
    x_o, st_o = oracle.pcg(orc, w["b"], k, lo_o, hi_o, xi, tol=tol, maxit=20000)
    assert st_o["converged"]
    op = npc.create_from_workload(ctx, w, kind)
    lo, hi = npc.npc_estimate_spectrum(op, 20, None)
    poly = npc.npc_set_poly(op, k, lo, hi, xi)
    x = torch.zeros(w["n"], dtype=torch.float64, device="cuda")
    st = npc.npc_pcg_solve(poly, op, dev(w["b"]), x, tol, 20000, history=True)
    assert st["converged"] and abs(st["iters"] - st_o["iters"]) <= 2, (st, st_o)
    assert st["relres_true"] <= tol
    xg = host(x)
    r = w["b"] - orc.apply(xg)
    assert np.linalg.norm(r) / np.linalg.norm(w["b"]) <= tol  # oracle-side residual check
    assert st["op_applications"] >= st["iters"] * (k + 1) + 1  # Table tab11 MVP law (+ true residual)
    assert len(st["history"]) == st["iters"] + 1 and st["history"][-1] <= tol
    if "x_exact" in w:
        assert np.max(np.abs(xg - 1.0)) < 1e-2


@pytest.mark.parametrize("name,kind", [("c1", "csr"), ("c3", "sell"), ("c2", "stencil"), ("c5", "schur")])
@pytest.mark.parametrize("nlev", [0, 1, 2, 3, 5])
@pytest.mark.parametrize("xi", [0.0, 1e-3])
def test_newton_variant(ctx, wl, name, kind, nlev, xi):
    """Alg. 1 on the GPU == the oracle's Alg. 1 == GPU Chebyshev of degree 2^nlev - 1."""
    w = wl(name)
    orc = oracle.Operator(w)
    lmin, lmax = oracle.estimate_spectrum(orc, 20, W.lanczos_start(w["n"]))
    op = npc.create_from_workload(ctx, w, kind)
    r = np.random.default_rng(nlev).uniform(-1, 1, w["n"])
    zn = torch.empty(w["n"], dtype=torch.float64, device="cuda")
    zc = torch.empty_like(zn)
    npc.npc_apply_poly(npc.npc_set_poly_newton(op, nlev, lmin, lmax, xi), dev(r), zn)
    npc.npc_apply_poly(npc.npc_set_poly(op, 2 ** nlev - 1, lmin, lmax, xi), dev(r), zc)
    ref = oracle.newton_apply(orc, nlev, lmin, lmax, xi, r)
    assert rel(host(zn), ref) <= POLY_TOL
    assert rel(host(zn), host(zc)) <= 1e-10


def test_tab_epsil_newton_on_gpu(ctx):
    """Table tab:epsil was produced with Newton, nlev = 6: the GPU Newton
    variant inside PCG reproduces its iteration column (58, 57, 50, 34, 39, 62) +-1."""
    w = W.tab_epsil_diag()
    op = npc.create_from_workload(ctx, w)
    for xi, it in [(0.0, 58), (1e-6, 57), (1e-5, 50), (1e-4, 34), (1e-3, 39), (1e-2, 62)]:
        poly = npc.npc_set_poly_newton(op, 6, 1.0, 1e5, xi)
        x = torch.zeros(w["n"], dtype=torch.float64, device="cuda")
        st = npc.npc_pcg_solve(poly, op, dev(w["b"]), x, 1e-10, 500)
        assert abs(st["iters"] - it) <= 1 and st["relres_true"] <= 1e-10
        assert st["op_applications"] == st["iters"] * 64 + 1


def test_schur_deterministic_mode(ctx, wl, monkeypatch):
    """The default single-rank Schur form is the split two-pass (no atomics) form: parity, and
    bit-identical results run to run and for any number of t ranges (the per-row summation
    sequence does not depend on the split)."""
    w = wl("c5")
    orc = oracle.Operator(w)
    lmin, lmax = oracle.estimate_spectrum(orc, 20, W.lanczos_start(w["n"]))
    r = np.random.default_rng(4).uniform(-1, 1, w["n"])
    outs = []
    for split in ("1", "2", "3", "2"):
        monkeypatch.setenv("NPC_SCHUR_SPLIT", split)
        op = npc.create_from_workload(ctx, w, "schur")
        monkeypatch.delenv("NPC_SCHUR_SPLIT")
        poly = npc.npc_set_poly(op, 30, lmin, lmax, 0.0)
        z = torch.empty(w["n"], dtype=torch.float64, device="cuda")
        npc.npc_apply_poly(poly, dev(r), z)
        outs.append(host(z))
    for o in outs[1:]:
        assert np.array_equal(outs[0], o)
    assert rel(outs[0], oracle.cheb_apply(orc, 30, lmin, lmax, 0.0, r)) <= POLY_TOL
    x = torch.zeros(w["n"], dtype=torch.float64, device="cuda")
    st = npc.npc_pcg_solve(npc.npc_set_poly(op, 10, lmin, lmax, 0.0), op, dev(w["b"]), x, 1e-8, 100)
    _, st_o = oracle.pcg(orc, w["b"], 10, lmin, lmax, 0.0, tol=1e-8)
    assert abs(st["iters"] - st_o["iters"]) <= 2


def test_schur_atomic_mode(ctx, wl, monkeypatch):
    """NPC_SCHUR_ATOMIC=1 selects the fp64-RED form (the one used across ranks): parity."""
    w = wl("c5")
    monkeypatch.setenv("NPC_SCHUR_ATOMIC", "1")
    op = npc.create_from_workload(ctx, w, "schur")
    monkeypatch.delenv("NPC_SCHUR_ATOMIC")
    orc = oracle.Operator(w)
    lmin, lmax = oracle.estimate_spectrum(orc, 20, W.lanczos_start(w["n"]))
    r = np.random.default_rng(5).uniform(-1, 1, w["n"])
    z = torch.empty(w["n"], dtype=torch.float64, device="cuda")
    npc.npc_apply_poly(npc.npc_set_poly(op, 40, lmin, lmax, 1e-3), dev(r), z)
    assert rel(host(z), oracle.cheb_apply(orc, 40, lmin, lmax, 1e-3, r)) <= POLY_TOL
    x = torch.zeros(w["n"], dtype=torch.float64, device="cuda")
    st = npc.npc_pcg_solve(npc.npc_set_poly(op, 10, lmin, lmax, 0.0), op, dev(w["b"]), x, 1e-8, 100)
    _, st_o = oracle.pcg(orc, w["b"], 10, lmin, lmax, 0.0, tol=1e-8)
    assert st["converged"] and abs(st["iters"] - st_o["iters"]) <= 2


def test_unpreconditioned_cg(ctx, wl):
    w = wl("c1")
    orc = oracle.Operator(w)
    _, st_o = oracle.pcg(orc, w["b"], -1, tol=1e-8, maxit=5000)
    op = npc.create_from_workload(ctx, w)
    x = torch.zeros(w["n"], dtype=torch.float64, device="cuda")
    st = npc.npc_pcg_solve(None, op, dev(w["b"]), x, 1e-8, 5000)
    assert abs(st["iters"] - st_o["iters"]) <= 2 and st["relres_true"] <= 1e-8


def test_callback_operator(ctx, wl):
    """CALLBACK kind: the user's y = A x is another npc operator; recurrence in k_axpby."""
    w = wl("c3")
    inner = npc.create_from_workload(ctx, w)
    lib = npc.lib()

    def apply(x, y, stream):
        return lib.npc_apply_operator(inner.h, x, y)

    op = npc.npc_create_operator(ctx, "callback", n_local=w["n"], apply=apply)
    orc = oracle.Operator(w)
    lmin, lmax = oracle.estimate_spectrum(orc, 20, W.lanczos_start(w["n"]))
    for k in (0, 1, 7, 40):
        poly = npc.npc_set_poly(op, k, lmin, lmax, 1e-3)
        r = np.random.default_rng(k).uniform(-1, 1, w["n"])
        z = torch.empty(w["n"], dtype=torch.float64, device="cuda")
        npc.npc_apply_poly(poly, dev(r), z)
        assert rel(host(z), oracle.cheb_apply(orc, k, lmin, lmax, 1e-3, r)) <= POLY_TOL
    x = torch.zeros(w["n"], dtype=torch.float64, device="cuda")
    poly = npc.npc_set_poly(op, 20, lmin, lmax, 0.0)
    st = npc.npc_pcg_solve(poly, op, dev(w["b"]), x, 1e-8, 5000)
    _, st_o = oracle.pcg(orc, w["b"], 20, lmin, lmax, 0.0, tol=1e-8, maxit=5000)
    assert abs(st["iters"] - st_o["iters"]) <= 2


# ------------------------------------------------------------------ edge cases
def test_tab_epsil_on_gpu(ctx):
    """Table tab:epsil reproduced through the GPU path: iterations
    (58, 57, 50, 34, 39, 62) +-1 with the exact interval [1, 1e5], degree 63."""
    w = W.tab_epsil_diag()
    op = npc.create_from_workload(ctx, w)
    for xi, it in [(0.0, 58), (1e-6, 57), (1e-5, 50), (1e-4, 34), (1e-3, 39), (1e-2, 62)]:
        poly = npc.npc_set_poly(op, 63, 1.0, 1e5, xi)
        x = torch.zeros(w["n"], dtype=torch.float64, device="cuda")
        st = npc.npc_pcg_solve(poly, op, dev(w["b"]), x, 1e-10, 500)
        assert abs(st["iters"] - it) <= 1 and st["relres_true"] <= 1e-10


def test_zero_rhs_identity_and_x0(ctx):
    n = 1000
    eye = dict(kind="csr", n=n, rowptr=np.arange(n + 1, dtype=np.int32), colidx=np.arange(n, dtype=np.int32),
               vals=np.ones(n))
    op = npc.create_from_workload(ctx, eye)
    poly = npc.npc_set_poly(op, 4, 0.5, 2.0, 0.0)
    x = torch.ones(n, dtype=torch.float64, device="cuda")
    st = npc.npc_pcg_solve(poly, op, torch.zeros(n, dtype=torch.float64, device="cuda"), x, 1e-8, 10)
    assert st["iters"] == 0 and st["converged"] and not host(x).any()
    b = np.random.default_rng(0).uniform(-1, 1, n)
    x = torch.zeros(n, dtype=torch.float64, device="cuda")
    st = npc.npc_pcg_solve(poly, op, dev(b), x, 1e-12, 10)
    assert st["iters"] == 1 and np.allclose(host(x), b, atol=1e-14)
    # nonzero x0 on config 1: same iterate count as the oracle started from the same x0
    w = W.config1()
    orc = oracle.Operator(w)
    op = npc.create_from_workload(ctx, w)
    lo, hi = oracle.estimate_spectrum(orc, 20, W.lanczos_start(w["n"]))
    poly = npc.npc_set_poly(op, 10, lo, hi, 0.0)
    x0 = np.random.default_rng(3).uniform(-1, 1, w["n"])
    _, st_o = oracle.pcg(orc, w["b"], 10, lo, hi, 0.0, tol=1e-8, x0=x0)
    x = dev(x0)
    st = npc.npc_pcg_solve(poly, op, dev(w["b"]), x, 1e-8, 1000)
    assert abs(st["iters"] - st_o["iters"]) <= 2 and st["op_applications"] == st["iters"] * 11 + 2


def test_errors(ctx):
    w = W.config1(side=8)
    op = npc.create_from_workload(ctx, w)
    with pytest.raises(npc.NpcError) as e:
        npc.npc_set_poly(op, 5, 1.0, 1.0, 0.0)
    assert e.value.name == "NPC_ERR_DEGENERATE_INTERVAL"
    for bad in [(5, 0.0, 1.0, 0.0), (5, 2.0, 1.0, 0.0), (-1, 1.0, 2.0, 0.0), (5, 1.0, 2.0, -1e-3)]:
        with pytest.raises(npc.NpcError) as e:
            npc.npc_set_poly(op, *bad)
        assert e.value.name == "NPC_ERR_INVALID_ARGUMENT"
    bad_cols = w["colidx"].copy()
    bad_cols[3] = w["n"] + 5
    with pytest.raises(npc.NpcError) as e:
        npc.npc_create_operator(ctx, "csr", n_local=w["n"], rowptr=w["rowptr"], colidx=bad_cols, vals=w["vals"])
    assert e.value.name == "NPC_ERR_DIMENSION"
    unsorted = w["colidx"].copy()
    unsorted[0], unsorted[1] = unsorted[1], unsorted[0]
    with pytest.raises(npc.NpcError):
        npc.npc_create_operator(ctx, "csr", n_local=w["n"], rowptr=w["rowptr"], colidx=unsorted, vals=w["vals"])
    poly = npc.npc_set_poly(op, 3, 0.1, 8.0, 0.0)
    b = dev(w["b"])
    with pytest.raises(npc.NpcError) as e:
        npc.npc_pcg_solve(poly, op, b, b, 1e-8, 10)
    with pytest.raises(npc.NpcError) as e:
        npc.npc_pcg_solve(poly, op, b, torch.zeros_like(b), 1.5, 10)
    assert e.value.name == "NPC_ERR_INVALID_ARGUMENT"
    st = npc.npc_pcg_solve(poly, op, b, torch.zeros_like(b), 1e-14, 2, raise_on_error=False)
    assert st["status"] == "NPC_ERR_NOT_CONVERGED" and st["iters"] == 2
    # indefinite operator -> breakdown
    n = 64
    neg = dict(kind="csr", n=n, rowptr=np.arange(n + 1, dtype=np.int32), colidx=np.arange(n, dtype=np.int32),
               vals=np.where(np.arange(n) % 2 == 0, 1.0, -1.0))
    opn = npc.create_from_workload(ctx, neg)
    st = npc.npc_pcg_solve(None, opn, dev(np.ones(n)), torch.zeros(n, dtype=torch.float64, device="cuda"), 1e-8,
                           100, raise_on_error=False)
    assert st["status"] == "NPC_ERR_BREAKDOWN"


def test_empty_rows_and_single_row(ctx):
    # CSR with empty rows (a zero row block) still applies correctly
    n = 700
    rng = np.random.default_rng(1)
    rows = []
    for i in range(n):
        if i % 97 == 5:
            rows.append([])
        else:
            rows.append(sorted(set(rng.integers(0, n, 5).tolist()) | {i}))
    rowptr = np.zeros(n + 1, dtype=np.int32)
    rowptr[1:] = np.cumsum([len(r) for r in rows])
    colidx = np.array([c for r in rows for c in r], dtype=np.int32)
    vals = rng.standard_normal(len(colidx))
    w = dict(kind="csr", n=n, rowptr=rowptr, colidx=colidx, vals=vals)
    orc = oracle.Operator(w)
    for kind in ("csr", "sell"):
        op = npc.create_from_workload(ctx, w, kind)
        x = rng.standard_normal(n)
        y = torch.empty(n, dtype=torch.float64, device="cuda")
        npc.npc_apply_operator(op, dev(x), y)
        assert rel(host(y), orc.apply(x)) <= 1e-13
    one = dict(kind="csr", n=1, rowptr=np.array([0, 1], dtype=np.int32), colidx=np.array([0], dtype=np.int32),
               vals=np.array([3.0]))
    op = npc.create_from_workload(ctx, one)
    poly = npc.npc_set_poly(op, 5, 1.0, 4.0, 0.0)
    z = torch.empty(1, dtype=torch.float64, device="cuda")
    npc.npc_apply_poly(poly, dev([2.0]), z)
    assert abs(host(z)[0] - oracle.cheb_apply(oracle.Operator(one), 5, 1.0, 4.0, 0.0, np.array([2.0]))[0]) < 1e-14


def test_closed_form_eigenvector_stencil(ctx):
    """P3 on the GPU stencil directly: p_k(A) v = p_k(lambda) v for a separable sine mode."""
    side = 32
    w = W.config2(side=side)
    op = npc.create_from_workload(ctx, w)
    g = np.arange(1, side + 1)
    modes = (1, 4, 9)
    v = np.einsum("i,j,k->ijk", *[np.sin(g * m * np.pi / (side + 1)) for m in modes[::-1]]).ravel()
    lam = sum(4 * np.sin(m * np.pi / (2 * (side + 1))) ** 2 for m in modes)
    lmin = 3 * 4 * np.sin(np.pi / (2 * (side + 1))) ** 2
    lmax = 3 * 4 * np.sin(side * np.pi / (2 * (side + 1))) ** 2
    k = 30
    th, dl = 0.5 * (lmin + lmax), 0.5 * (lmax - lmin)

    def T(m, x):
        a, b = 1.0, x
        for _ in range(m - 1):
            a, b = b, 2 * x * b - a
        return b
    p = (1 - T(k + 1, (th - lam) / dl) / T(k + 1, th / dl)) / lam
    poly = npc.npc_set_poly(op, k, lmin, lmax, 0.0)
    z = torch.empty(w["n"], dtype=torch.float64, device="cuda")
    npc.npc_apply_poly(poly, dev(v), z)
    assert rel(host(z), p * v) < 1e-10


def test_in_library_timing_with_graphs(ctx, wl):
    """npc_context_set_timing: the PCG iteration graph carries event-record nodes, is replayed
    one graph per sync, and the per-class device times are collected; the solve is the same
    (iterations, solution) as without timing."""
    w = W.config3(side=32)  # 32,768 rows: above the cluster-resident size, so graphs are used
    op = npc.create_from_workload(ctx, w, "csr")
    lo, hi = npc.npc_estimate_spectrum(op, 20, None)
    k = 12
    res = {}
    for timing in (False, True):
        poly = npc.npc_set_poly(op, k, lo, hi, 0.0)
        npc.npc_context_set_timing(ctx, timing)
        npc.npc_context_get_timing(ctx)  # reset
        x = torch.zeros(w["n"], dtype=torch.float64, device="cuda")
        st = npc.npc_pcg_solve(poly, op, dev(w["b"]), x, 1e-8, 2000)
        tm = npc.npc_context_get_timing(ctx)
        npc.npc_context_set_timing(ctx, False)
        res[timing] = (st, host(x), tm)
    (s0, x0, _), (s1, x1, tm) = res[False], res[True]
    assert s0["iters"] == s1["iters"] and np.array_equal(x0, x1)
    ms, n = tm["degree"]
    # every degree launch of every replayed iteration is timed (the last graph replay may run
    # up to 3 no-op iterations after convergence)
    assert s1["iters"] * k <= n <= (s1["iters"] + 3) * k and ms > 0.0
    assert tm["operator"][1] >= s1["iters"] and tm["update"][1] >= s1["iters"]


def test_boundary_seed_setup_seconds_last_error(ctx):
    """SURVEY §8(b) boundary details: npc_estimate_spectrum's seed selects the counter-hash
    start vector (the same generator as workloads.lanczos_start), the PCG stats carry the
    preconditioner setup (estimate + set_poly) apart from the solve, and npc_last_error(ctx)
    holds the last failing call made through that context only."""
    w = W.config3(side=20)
    n = w["n"]
    op = npc.create_from_workload(ctx, w, "csr")
    for seed in (npc.NPC_DEFAULT_SEED, 12345):
        a = npc.npc_estimate_spectrum(op, 20, None, seed=seed)
        b = npc.npc_estimate_spectrum(op, 20, dev(W.lanczos_start(n, seed=seed)))
        assert a == b, (seed, a, b)
    assert npc.npc_estimate_spectrum(op, 20, None, seed=12345) != npc.npc_estimate_spectrum(op, 20, None)
    lo, hi = npc.npc_estimate_spectrum(op, 20, None)
    poly = npc.npc_set_poly(op, 20, lo, hi, 0.0)
    x = torch.zeros(n, dtype=torch.float64, device="cuda")
    st = npc.npc_pcg_solve(poly, op, dev(w["b"]), x, w["tol"], 5000)
    assert 0.0 < st["setup_seconds"] < 10.0 and st["solve_seconds"] > 0.0
    st0 = npc.npc_pcg_solve(None, op, dev(w["b"]), torch.zeros_like(x), w["tol"], 5000, raise_on_error=False)
    assert st0["setup_seconds"] == 0.0
    # context-scoped error messages
    other = npc.npc_context_create(0)
    assert npc.npc_last_error(other) == ""
    st = npc.npc_pcg_solve(poly, op, dev(w["b"]), torch.zeros_like(x), 1e-12, 2, raise_on_error=False)
    assert st["status"] == "NPC_ERR_NOT_CONVERGED"
    assert "did not converge" in npc.npc_last_error(ctx)
    assert npc.npc_last_error(other) == ""
