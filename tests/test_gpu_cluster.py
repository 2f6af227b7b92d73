"""Cluster-resident polynomial for small CSR operators (csr_cluster.cu): all k degrees of
Alg. 2 in one thread-block-cluster launch with DSMEM gathers.  The launch-per-degree path's
result to a few ulps (same per-row operation order) and the oracle's within the north-star bar;
PCG through it keeps iteration parity."""
import os

import numpy as np
import pytest

import oracle
import workloads as W

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2208_01339_b200 as npc  # noqa: E402


@pytest.fixture(scope="module")
def ctx():
    c = npc.npc_context_create(0)
    yield c
    torch.cuda.synchronize()


def run(ctx, w, k, lo, hi, xi, r, cluster):
    if cluster:
        os.environ.pop("NPC_NO_CLUSTER", None)
    else:
        os.environ["NPC_NO_CLUSTER"] = "1"
    try:
        op = npc.create_from_workload(ctx, w, "csr")
        poly = npc.npc_set_poly(op, k, lo, hi, xi)
        z = torch.empty(w["n"], dtype=torch.float64, device="cuda")
        npc.npc_apply_poly(poly, torch.tensor(r, device="cuda"), z)
        return z.cpu().numpy()
    finally:
        os.environ.pop("NPC_NO_CLUSTER", None)


CASES = {"c1": lambda: W.config1(), "c1_ragged": lambda: W.config1(side=37), "c3_20": lambda: W.config3(side=20),
         "c4_16k": lambda: W.config4(n=16_384), "tiny": lambda: W.config1(side=5)}


@pytest.mark.parametrize("name", list(CASES))
@pytest.mark.parametrize("k,xi", [(1, 0.0), (2, 1e-3), (3, 0.0), (10, 1e-3), (63, 0.0)])
def test_cluster_poly_bitwise_and_oracle(ctx, name, k, xi):
    w = CASES[name]()
    orc = oracle.Operator(w)
    lo, hi = oracle.estimate_spectrum(orc, 20, W.lanczos_start(w["n"]))
    r = np.random.default_rng(k).uniform(-1, 1, w["n"])
    zc = run(ctx, w, k, lo, hi, xi, r, True)
    zl = run(ctx, w, k, lo, hi, xi, r, False)
    # same per-row operation order; the compiler may contract the epilogue differently (ulps)
    assert np.max(np.abs(zc - zl)) <= 1e-12 * np.max(np.abs(zl)), np.max(np.abs(zc - zl))
    ref = oracle.cheb_apply(orc, k, lo, hi, xi, r)
    assert np.linalg.norm(zc - ref) <= 1e-10 * np.linalg.norm(ref)


def test_cluster_pcg_config1(ctx):
    w = W.config1()
    orc = oracle.Operator(w)
    lo_o, hi_o = oracle.estimate_spectrum(orc, 20, W.lanczos_start(w["n"]))
    _, st_o = oracle.pcg(orc, w["b"], 10, lo_o, hi_o, 0.0, tol=w["tol"])
    op = npc.create_from_workload(ctx, w, "csr")
    lo, hi = npc.npc_estimate_spectrum(op, 20, None)
    poly = npc.npc_set_poly(op, 10, lo, hi, 0.0)
    x = torch.zeros(w["n"], dtype=torch.float64, device="cuda")
    st = npc.npc_pcg_solve(poly, op, torch.tensor(w["b"], device="cuda"), x, w["tol"], 1000)
    assert st["converged"] and abs(st["iters"] - st_o["iters"]) <= 2 and st["relres_true"] <= w["tol"]
    assert st["op_applications"] == st["iters"] * 11 + 1


@pytest.mark.parametrize("name,k,x0", [("c1", 10, False), ("c1_ragged", 5, True), ("c3_20", 20, False),
                                       ("tiny", 3, False), ("c1", 0, True)])
def test_cluster_whole_pcg_matches_graph_path(ctx, name, k, x0, monkeypatch):
    """The one-launch cluster PCG and the graph-replayed multi-kernel PCG run the same
    recurrences: same iteration count (+-1: reduction order), same counter laws, both within
    tol of the true residual, history consistent."""
    w = CASES[name]()
    b = torch.tensor(w["b"] if "b" in w else np.random.default_rng(1).uniform(-1, 1, w["n"]), device="cuda")
    xinit = np.random.default_rng(3).standard_normal(w["n"]) * 0.01 if x0 else np.zeros(w["n"])
    out = {}
    for mode in ("cluster", "graph"):
        if mode == "graph":
            monkeypatch.setenv("NPC_NO_CLUSTER", "1")
        op = npc.create_from_workload(ctx, w, "csr")
        lo, hi = npc.npc_estimate_spectrum(op, 20, None)
        poly = npc.npc_set_poly(op, k, lo, hi, 0.0)
        x = torch.tensor(xinit, device="cuda")
        st = npc.npc_pcg_solve(poly, op, b, x, 1e-8, 2000, history=True)
        out[mode] = (st, x.cpu().numpy())
    (sc, xc), (sg, xg) = out["cluster"], out["graph"]
    assert sc["converged"] and sg["converged"]
    assert abs(sc["iters"] - sg["iters"]) <= 1, (sc["iters"], sg["iters"])
    assert sc["relres_true"] <= 1e-8
    assert sc["op_applications"] == sc["iters"] * (k + 1) + (1 if x0 else 0) + 1
    assert sc["reductions"] == sc["iters"] + 3
    hc = np.asarray(sc["history"])
    assert len(hc) == sc["iters"] + 1 and hc[-1] <= 1e-8 and hc[0] > 1e-8
    orc = oracle.Operator(w)
    assert np.linalg.norm(b.cpu().numpy() - orc.apply(xc)) / np.linalg.norm(b.cpu().numpy()) <= 1e-8


def test_cluster_whole_pcg_edge_cases(ctx):
    w = CASES["c1"]()
    op = npc.create_from_workload(ctx, w, "csr")
    poly = npc.npc_set_poly(op, 4, 0.03, 8.1, 0.0)
    z = torch.zeros(w["n"], dtype=torch.float64, device="cuda")
    x = torch.ones_like(z)
    st = npc.npc_pcg_solve(poly, op, z, x, 1e-8, 100)  # b = 0 -> x = 0, 0 iterations
    assert st["iters"] == 0 and st["converged"] and float(torch.abs(x).max()) == 0.0
    b = torch.tensor(w["b"], device="cuda")
    x = torch.zeros_like(b)
    with pytest.raises(npc.NpcError) as e:  # maxit
        npc.npc_pcg_solve(poly, op, b, x, 1e-12, 3)
    assert e.value.name == "NPC_ERR_NOT_CONVERGED"
    st = npc.npc_pcg_solve(poly, op, b, x, 1e-12, 3, raise_on_error=False)
    assert st["iters"] == 3 and not st["converged"] and st["relres_true"] > 1e-12
    # not SPD: -A -> breakdown
    wn = dict(w, vals=-w["vals"])
    opn = npc.create_from_workload(ctx, wn, "csr")
    pn = npc.npc_set_poly(opn, 4, 0.03, 8.1, 0.0)
    with pytest.raises(npc.NpcError) as e:
        npc.npc_pcg_solve(pn, opn, b, torch.zeros_like(b), 1e-8, 100)
    assert e.value.name == "NPC_ERR_BREAKDOWN"
