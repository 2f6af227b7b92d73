"""GPU parity of the DFN Schur-complement operator (NPC_OP_DFN; SURVEY §8(f) NEXT row 2;
PAPER.md §4.2-4.3, Eq. schur, Alg. 3, Alg. 4) against oracle O9 on the same seeded synthetic
DFN systems, through the C ABI.

Bars: operator application relative error <= 1e-12 (banded vs dense per-block Cholesky and a
different summation order; both are backward stable on these SPD blocks), p_k(S^) v <= 1e-10
(north-star bar), PCG iterations within +-2 and true relative residual <= tol.
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


@pytest.fixture(scope="module")
def ctx():
    c = npc.npc_context_create(0)
    yield c
    torch.cuda.synchronize()


def dev(a):
    return torch.tensor(np.ascontiguousarray(a, dtype=np.float64), device="cuda")


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


SYS = {
    "small": lambda: W.dfn(12, seed=1),
    "ragged": lambda: W.dfn(157, seed=2, grid=(3, 11)),  # 9..121 rows: explicit inverses, 128-thread CTAs
    "alpha0": lambda: W.dfn(40, seed=3, alpha=0.0),
    "wide": lambda: W.dfn(20, seed=4, grid=(16, 36)),    # blocks > 128 rows: banded solves, 32-lane groups
    "mixed": lambda: W.dfn(60, seed=6, grid=(6, 14)),     # 36..196 rows: dense inverses and banded solves
}
_cache = {}


def sysw(name):
    if name not in _cache:
        _cache[name] = SYS[name]()
    return _cache[name]


@pytest.mark.parametrize("name", list(SYS))
@pytest.mark.parametrize("scaled", [True, False])
def test_dfn_apply(ctx, name, scaled):
    w = dict(sysw(name), scaled=int(scaled))
    orc = oracle.Operator(w, scaled=scaled)
    op = npc.create_from_workload(ctx, w, "dfn")
    x = np.random.default_rng(5).standard_normal(w["n"])
    y = torch.empty(w["n"], dtype=torch.float64, device="cuda")
    npc.npc_apply_operator(op, dev(x), y)
    assert rel(y.cpu().numpy(), orc.apply(x)) <= 1e-12, name


@pytest.mark.parametrize("name", ["small", "ragged", "mixed"])
@pytest.mark.parametrize("k,xi", [(1, 0.0), (10, 1e-3), (40, 0.0)])
def test_dfn_apply_poly(ctx, name, k, xi):
    w = sysw(name)
    orc = oracle.Operator(w)
    lo, hi = oracle.estimate_spectrum(orc, 20, W.lanczos_start(w["n"]))
    op = npc.create_from_workload(ctx, w, "dfn")
    poly = npc.npc_set_poly(op, k, lo, hi, xi)
    r = np.random.default_rng(6).uniform(-1, 1, w["n"])
    z = torch.empty(w["n"], dtype=torch.float64, device="cuda")
    npc.npc_apply_poly(poly, dev(r), z)
    assert rel(z.cpu().numpy(), oracle.cheb_apply(orc, k, lo, hi, xi, r)) <= 1e-10


@pytest.mark.parametrize("name,k", [("small", 10), ("ragged", 30), ("alpha0", 5), ("mixed", 20)])
def test_dfn_pcg(ctx, name, k):
    w = sysw(name)
    orc = oracle.Operator(w)
    lo_o, hi_o = oracle.estimate_spectrum(orc, 20, W.lanczos_start(w["n"]))
    _, st_o = oracle.pcg(orc, w["b"], k, lo_o, hi_o, 0.0, tol=w["tol"], maxit=5000)
    op = npc.create_from_workload(ctx, w, "dfn")
    lo, hi = npc.npc_estimate_spectrum(op, 20, None)
    assert abs(hi - hi_o) <= 1e-6 * hi_o
    poly = npc.npc_set_poly(op, k, lo, hi, 0.0)
    x = torch.zeros(w["n"], dtype=torch.float64, device="cuda")
    st = npc.npc_pcg_solve(poly, op, dev(w["b"]), x, w["tol"], 5000)
    assert st["converged"] and abs(st["iters"] - st_o["iters"]) <= 2, (st, st_o)
    assert np.linalg.norm(w["b"] - orc.apply(x.cpu().numpy())) / np.linalg.norm(w["b"]) <= w["tol"]


def test_dfn_rejects_bad_input(ctx):
    w = sysw("small")
    rp, ci, v = w["A"]
    ci2 = ci.copy()
    ci2[0] = w["nh"] - 1  # row 0 (block 0) -> a column in the last block: not block-diagonal
    bad = dict(w, A=(rp, ci2, v))
    with pytest.raises(npc.NpcError) as e:
        npc.create_from_workload(ctx, bad, "dfn")
    assert e.value.name == "NPC_ERR_DIMENSION"
    neg = dict(w, A=(rp, ci, -v))  # not SPD
    with pytest.raises(npc.NpcError) as e:
        npc.create_from_workload(ctx, neg, "dfn")
    assert e.value.name == "NPC_ERR_DIMENSION"
