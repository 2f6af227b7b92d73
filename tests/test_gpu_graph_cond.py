"""GPU: PCG with conditional (IF-node) iteration bodies in the replayed CUDA graph
(NPC_GRAPH_COND=1, opt-in): iterations after convergence are skipped instead of launched as
no-ops.  The same kernels run in the same order, so the solve must be bitwise identical to
the default graph and match the oracle's iteration count (SURVEY §8(a) a5/a6 bars)."""
import os

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


CASES = {"csr": (lambda: W.config3(side=22), "csr", 40), "stencil": (lambda: W.config2(side=24), "stencil", 10),
         "dfn": (lambda: W.dfn(30, seed=8), "dfn", 30), "schur": (lambda: W.config5(n=20_000), "schur", 50)}


@pytest.mark.parametrize("name", list(CASES))
def test_conditional_iterations_match(ctx, name):
    make, kind, k = CASES[name]
    w = make()
    n = w["n"]
    op = npc.create_from_workload(ctx, w, kind)
    lo, hi = npc.npc_estimate_spectrum(op, 20, None)
    b = torch.tensor(w["b"], device="cuda")
    out = []
    for cond in (False, True):
        if cond:
            os.environ["NPC_GRAPH_COND"] = "1"
        try:
            poly = npc.npc_set_poly(op, k, lo, hi, 0.0)  # fresh polynomial: a new graph each time
            x = torch.zeros(n, dtype=torch.float64, device="cuda")
            st = npc.npc_pcg_solve(poly, op, b, x, w["tol"], 5000)
        finally:
            os.environ.pop("NPC_GRAPH_COND", None)
        out.append((st, x))
    (s0, x0), (s1, x1) = out
    assert s0["iters"] == s1["iters"] and s0["op_applications"] == s1["op_applications"]
    assert torch.equal(x0, x1)
    orc = oracle.Operator(w)
    lo_o, hi_o = oracle.estimate_spectrum(orc, 20, W.lanczos_start(n))
    _, st_o = oracle.pcg(orc, w["b"], k, lo_o, hi_o, 0.0, tol=w["tol"], maxit=5000)
    assert abs(s1["iters"] - st_o["iters"]) <= 2 and s1["relres_true"] <= w["tol"]
    assert np.linalg.norm(w["b"] - orc.apply(x1.cpu().numpy())) / np.linalg.norm(w["b"]) <= w["tol"]
