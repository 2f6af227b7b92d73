"""GPU parity of the low-rank spectral correction P = p_k(A) + V (V^T A V)^{-1} V^T
 and of the fully reorthogonalised Ritz vectors,
against the CPU oracle (O8) on the same seeded inputs, through the C ABI.

Bars: applications of P relative 2-norm error <= 1e-10 (the north-star bar for p_k(A) v);
PCG iterations within +-2 and true relative residual <= tol; Ritz values 1e-8 relative and
Ritz vectors |<v_gpu, v_oracle>| >= 1 - 1e-6 on well-separated leftmost eigenvalues.
"""
import threading

import numpy as np
import pytest

import oracle
import workloads as W

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

import bench  # noqa: E402
import paper_2208_01339_b200 as npc  # noqa: E402


@pytest.fixture(scope="module")
def ctx():
    c = npc.npc_context_create(0)
    yield c
    torch.cuda.synchronize()


def dev(a):
    return torch.tensor(np.ascontiguousarray(a, dtype=np.float64), device="cuda")


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


WL = {
    "c1": (lambda: W.config1(side=37), "csr"),
    "c1_sell": (lambda: W.config1(side=37), "sell"),  # permuted internal order
    "c2": (lambda: W.config2(side=19), "stencil"),
    "c3": (lambda: W.config3(side=14), "csr"),
    "c4": (lambda: W.config4(n=12_000), "sell"),
    "c5": (lambda: W.config5(n=9_001), "schur"),
}
_cache = {}


def wl(name):
    if name not in _cache:
        _cache[name] = WL[name][0]()
    return _cache[name]


@pytest.mark.parametrize("name", list(WL))
@pytest.mark.parametrize("p,k,newton", [(1, 10, False), (4, 30, False), (16, 5, False), (3, 15, True)])
def test_lowrank_apply_parity(ctx, name, p, k, newton):
    w = wl(name)
    kind = WL[name][1]
    orc = oracle.Operator(w)
    n = w["n"]
    lo, hi = oracle.estimate_spectrum(orc, 20, W.lanczos_start(n))
    V = np.random.default_rng(p + 100).standard_normal((n, p))  # any full-rank V
    lr = oracle.LowRank(orc, V)
    r = np.random.default_rng(7).uniform(-1, 1, n)
    op = npc.create_from_workload(ctx, w, kind)
    if newton:
        nlev = int(np.log2(k + 1))
        poly = npc.npc_set_poly_newton(op, nlev, lo, hi, 1e-3)
        ref0 = oracle.newton_apply(orc, nlev, lo, hi, 1e-3, r)
        ref = ref0 + (oracle.lowrank_apply(orc, 0, lo, hi, 1e-3, lr, r) - oracle.cheb_apply(orc, 0, lo, hi, 1e-3, r))
    else:
        poly = npc.npc_set_poly(op, k, lo, hi, 1e-3)
        ref = oracle.lowrank_apply(orc, k, lo, hi, 1e-3, lr, r)
    npc.npc_poly_set_lowrank(poly, dev(V.T))
    z = torch.empty(n, dtype=torch.float64, device="cuda")
    npc.npc_apply_poly(poly, dev(r), z)
    assert rel(z.cpu().numpy(), ref) <= 1e-10, (name, p, k)
    # removing the correction restores p_k(A) r
    npc.npc_poly_set_lowrank(poly, None)
    npc.npc_apply_poly(poly, dev(r), z)
    ref0 = oracle.newton_apply(orc, int(np.log2(k + 1)), lo, hi, 1e-3, r) if newton else \
        oracle.cheb_apply(orc, k, lo, hi, 1e-3, r)
    assert rel(z.cpu().numpy(), ref0) <= 1e-10


@pytest.mark.parametrize("name,p", [("c1", 4), ("c3", 6), ("c4", 3), ("c1_sell", 2)])
def test_lowrank_pcg_parity(ctx, name, p):
    """PCG with P = p_k(A) + V (V^T A V)^{-1} V^T, V = the oracle's Ritz vectors (both sides
    get the same V and interval); iterations within +-2, true residual <= tol."""
    w = wl(name)
    kind = WL[name][1]
    orc = oracle.Operator(w)
    n = w["n"]
    lo, hi = oracle.estimate_spectrum(orc, 20, W.lanczos_start(n))
    _, V = oracle.ritz_vectors(orc, 40, p, W.lanczos_start(n))
    lr = oracle.LowRank(orc, V)
    k = 10
    _, st_o = oracle.pcg(orc, w["b"], k, lo, hi, 0.0, tol=w["tol"], maxit=5000, lowrank=lr)
    op = npc.create_from_workload(ctx, w, kind)
    poly = npc.npc_set_poly(op, k, lo, hi, 0.0)
    npc.npc_poly_set_lowrank(poly, dev(V.T))
    x = torch.zeros(n, dtype=torch.float64, device="cuda")
    st = npc.npc_pcg_solve(poly, op, dev(w["b"]), x, w["tol"], 5000)
    assert st["converged"] and abs(st["iters"] - st_o["iters"]) <= 2, (st, st_o)
    assert st["relres_true"] <= w["tol"]
    assert np.linalg.norm(w["b"] - orc.apply(x.cpu().numpy())) / np.linalg.norm(w["b"]) <= w["tol"]
    # one extra reduction point per iteration (V^T r) besides the single CG reduction
    assert st["reductions"] == 2 * st["iters"] + 3


def test_ritz_vectors_parity(ctx):
    w = W.config3(side=12)  # variable coefficients: no symmetric degeneracy in the spectrum
    orc = oracle.Operator(w)
    n = w["n"]
    v0 = W.lanczos_start(n)
    th_o, V_o = oracle.ritz_vectors(orc, 120, 4, v0)
    op = npc.create_from_workload(ctx, w, "csr")
    th, V = npc.npc_ritz_vectors(op, 120, 4, None)  # default start = the same counter hash
    V = V.cpu().numpy().T
    assert np.allclose(th, th_o, rtol=1e-8), (th, th_o)
    for j in range(4):
        assert abs(np.linalg.norm(V[:, j]) - 1.0) < 1e-10
        gap = min(abs(th_o[j] - th_o[i]) for i in range(4) if i != j) / th_o[-1]
        if gap > 1e-3:
            assert abs(V[:, j] @ V_o[:, j]) >= 1 - 1e-6, j
        res = np.linalg.norm(orc.apply(V[:, j]) - th[j] * V[:, j])
        res_o = np.linalg.norm(orc.apply(V_o[:, j]) - th_o[j] * V_o[:, j])
        assert res <= 1.5 * res_o + 1e-8 * th_o[-1]


def test_lowrank_argument_errors(ctx):
    w = wl("c1")
    op = npc.create_from_workload(ctx, w, "csr")
    poly = npc.npc_set_poly(op, 5, 0.1, 8.0, 0.0)
    with pytest.raises(npc.NpcError) as e:
        npc.npc_poly_set_lowrank(poly, torch.zeros((17, w["n"]), dtype=torch.float64, device="cuda"))
    assert e.value.name == "NPC_ERR_INVALID_ARGUMENT"
    with pytest.raises(npc.NpcError) as e:  # V rank-deficient -> V^T A V singular
        npc.npc_poly_set_lowrank(poly, torch.zeros((2, w["n"]), dtype=torch.float64, device="cuda"))
    assert e.value.name == "NPC_ERR_BREAKDOWN"


def test_lowrank_multirank_local(ctx):
    """2 ranks (host threads, local transport): V^T r is allreduced; same result as the oracle."""
    w = wl("c3")
    orc = oracle.Operator(w)
    n = w["n"]
    lo, hi = oracle.estimate_spectrum(orc, 20, W.lanczos_start(n))
    V = np.random.default_rng(3).standard_normal((n, 3))
    lr = oracle.LowRank(orc, V)
    r = np.random.default_rng(8).uniform(-1, 1, n)
    ref = oracle.lowrank_apply(orc, 12, lo, hi, 0.0, lr, r)
    ws, out, err = 2, [None, None], [None, None]

    def body(rank):
        c = None
        try:
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                c = npc.npc_context_create_local(0, ws, rank, "lowrank-mr", s)
                op, r0, r1 = bench.create_operator(npc, c, w, "csr", ws, rank, 3)
                poly = npc.npc_set_poly(op, 12, lo, hi, 0.0)
                npc.npc_poly_set_lowrank(poly, dev(V[r0:r1].T))
                z = torch.empty(r1 - r0, dtype=torch.float64, device="cuda")
                npc.npc_apply_poly(poly, dev(r[r0:r1]), z)
                s.synchronize()
                out[rank] = (r0, z.cpu().numpy())
        except BaseException as e:  # noqa: BLE001
            err[rank] = e
            if c is not None:
                c.close()

    th = [threading.Thread(target=body, args=(q,), daemon=True) for q in range(ws)]
    for t in th:
        t.start()
    for t in th:
        t.join(240)
    for e in err:
        if e is not None:
            raise e
    z = np.concatenate([o[1] for o in sorted(out, key=lambda o: o[0])])
    assert rel(z, ref) <= 1e-10
