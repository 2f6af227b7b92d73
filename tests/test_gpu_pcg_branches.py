"""GPU parity of the PCG branches the headline solves rarely take (reading A23, x0 != 0):
residual replacement with restart, the 50-replacement cap, and a nonzero initial guess, on
the cluster-resident single-launch PCG (small CSR), the multi-kernel PCG (NPC_NO_CLUSTER=1)
and the SELL operator.  Inputs: workloads.pcg_replacement_case / pcg_floor_case (crafted,
seeded); expected behaviour from oracle O5, itself pinned in tests/test_oracle_pins.py
(test_A23_*, test_P6b_*).
"""
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

PATHS = ["cluster", "multikernel", "sell"]


@pytest.fixture(scope="module")
def ctx():
    c = npc.npc_context_create(0)
    yield c
    torch.cuda.synchronize()


@pytest.fixture
def path(request, ctx, monkeypatch):
    if request.param == "multikernel":
        monkeypatch.setenv("NPC_NO_CLUSTER", "1")
    return request.param


def _op(ctx, w, path):
    return npc.create_from_workload(ctx, w, "sell" if path == "sell" else "csr")


def _dev(a):
    return torch.tensor(np.asarray(a, dtype=np.float64), device="cuda")


@pytest.mark.parametrize("path", PATHS, indirect=True)
@pytest.mark.parametrize("scale,tol", [(1e7, 1e-8), (1e8, 1e-10), (1e6, 1e-11)])
def test_replacement_restart_parity(ctx, path, scale, tol):
    w, x0 = W.pcg_replacement_case(scale)
    orc = oracle.Operator(w)
    _, st_o = oracle.pcg(orc, w["b"], 2, 1.0, 10.0, 0.0, tol=tol, maxit=2000, x0=x0)
    assert st_o["converged"] and st_o["true_checks"] == 2
    op = _op(ctx, w, path)
    poly = npc.npc_set_poly(op, 2, 1.0, 10.0, 0.0)
    x = _dev(x0)
    st = npc.npc_pcg_solve(poly, op, _dev(w["b"]), x, tol, 2000)
    torch.cuda.synchronize()
    assert st["converged"] and st["relres_true"] <= tol
    assert abs(st["iters"] - st_o["iters"]) <= 2, (st, st_o)
    A, b = w["dense"], w["b"]
    xg = x.cpu().numpy()
    assert np.linalg.norm(b - A @ xg) / np.linalg.norm(b) <= 2 * tol


@pytest.mark.parametrize("path", PATHS, indirect=True)
@pytest.mark.parametrize("k", [-1, 2])
def test_replacement_cap_parity(ctx, path, k):
    w = W.pcg_floor_case()
    orc = oracle.Operator(w)
    _, st_o = oracle.pcg(orc, w["b"], k, 1e-8, 10.0, 0.0, tol=1e-10, maxit=5000)
    assert not st_o["converged"] and st_o["true_checks"] == 51
    op = _op(ctx, w, path)
    poly = npc.npc_set_poly(op, k, 1e-8, 10.0, 0.0) if k >= 0 else None
    x = torch.zeros(w["n"], dtype=torch.float64, device="cuda")
    st = npc.npc_pcg_solve(poly, op, _dev(w["b"]), x, 1e-10, 5000, raise_on_error=False)
    assert st["status"] == "NPC_ERR_NOT_CONVERGED" and not st["converged"], st
    assert st["relres_true"] > 1e-10 and st["relres_recursive"] <= 1e-10
    # both stop after the 51st true check; the iteration counts between checks depend on
    # rounding, so compare the total loosely (51 restarts of a few iterations each)
    assert abs(st["iters"] - st_o["iters"]) <= max(2, 0.25 * st_o["iters"]), (st, st_o)


@pytest.mark.parametrize("path", PATHS, indirect=True)
def test_nonzero_x0_parity(ctx, path):
    n = 30
    A, _ = W.random_spd_dense(n, 3, cond=50.0)
    rowptr, colidx, vals = W.dense_to_csr(A)
    w = dict(kind="csr", n=n, rowptr=rowptr, colidx=colidx, vals=vals)
    b = np.random.default_rng(4).uniform(-1, 1, n)
    xs = np.linalg.solve(A, b)
    orc = oracle.Operator(w)
    op = _op(ctx, w, path)
    poly = npc.npc_set_poly(op, 4, 1.0, 50.0, 0.0)
    for x0 in (np.random.default_rng(5).standard_normal(n) * 10.0, 2.0 * xs):
        _, st_o = oracle.pcg(orc, b, 4, 1.0, 50.0, 0.0, tol=1e-10, maxit=400, x0=x0)
        x = _dev(x0)
        st = npc.npc_pcg_solve(poly, op, _dev(b), x, 1e-10, 400)
        torch.cuda.synchronize()
        assert st["converged"] and abs(st["iters"] - st_o["iters"]) <= 2
        assert st["op_applications"] == st["iters"] * 5 + 2
        assert np.linalg.norm(x.cpu().numpy() - xs) / np.linalg.norm(xs) <= 10 * 1e-10 * 50.0
