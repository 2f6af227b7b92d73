"""Temporal blocking of the stencil operator (two degrees per pass):
the fused pass must give exactly the single-degree path's bits (same operation order, zeros
for Dirichlet ghosts) and match the oracle within the north-star bar, on cubes and on ragged
non-cubic grids whose tiles and z-chunks do not divide the grid."""
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


def stencil_w(nx, ny, nz):
    return dict(kind="stencil", name=f"st{nx}x{ny}x{nz}", n=nx * ny * nz, dim=3, nx=nx, ny=ny, nz=nz, diag=6.0,
                offdiag=-1.0)


@pytest.fixture(scope="module")
def ctx():
    c = npc.npc_context_create(0)
    yield c
    torch.cuda.synchronize()


ENGINE_ENV = ("NPC_STEP2", "NPC_NO_STEP2", "NPC_ST_TMA", "NPC_ST_NOTMA", "NPC_ST_TMA2")


def apply(ctx, w, k, lo, hi, xi, r, step2, engine="reg"):
    """step2: force the fused two-degree pass on (small grids are L2-resident) or off;
    engine: 'reg' = register-marching kernels (k_stencil_step / k_stencil_step2), 'tma' = the
    TMA-staged kernels (k_stencil_tma / k_stencil_tma2, even nx only)."""
    for v in ENGINE_ENV:
        os.environ.pop(v, None)
    os.environ["NPC_STEP2" if step2 else "NPC_NO_STEP2"] = "1"
    os.environ["NPC_ST_TMA" if engine == "tma" else "NPC_ST_NOTMA"] = "1"
    if engine == "tma":
        os.environ["NPC_ST_TMA2"] = "1"  # the two-degree TMA pass is opt-in
    try:
        op = npc.create_from_workload(ctx, w, "stencil")
        poly = npc.npc_set_poly(op, k, lo, hi, xi)
        z = torch.empty(w["n"], dtype=torch.float64, device="cuda")
        npc.npc_apply_poly(poly, torch.tensor(r, device="cuda"), z)
        return z.cpu().numpy()
    finally:
        for v in ENGINE_ENV:
            os.environ.pop(v, None)


@pytest.mark.parametrize("dims,engine", [((24, 24, 24), "reg"), ((37, 13, 29), "reg"), ((33, 9, 17), "reg"),
                                         ((8, 8, 40), "reg"), ((24, 24, 24), "tma"), ((8, 8, 40), "tma"),
                                         ((40, 18, 21), "tma"), ((66, 34, 12), "tma"), ((96, 40, 3), "tma")])
@pytest.mark.parametrize("k", [4, 5, 10, 31])
def test_step2_bitwise_and_oracle(ctx, dims, engine, k):
    w = stencil_w(*dims)
    orc = oracle.Operator(w)
    lo, hi = oracle.estimate_spectrum(orc, 20, W.lanczos_start(w["n"]))
    r = np.random.default_rng(k).uniform(-1, 1, w["n"])
    z2 = apply(ctx, w, k, lo, hi, 1e-3, r, True, engine)
    z1 = apply(ctx, w, k, lo, hi, 1e-3, r, False)
    assert np.array_equal(z1, z2), np.max(np.abs(z1 - z2))
    ref = oracle.cheb_apply(orc, k, lo, hi, 1e-3, r)
    assert np.linalg.norm(z2 - ref) <= 1e-10 * np.linalg.norm(ref)


@pytest.mark.parametrize("engine", ["reg", "tma"])
def test_step2_pcg(ctx, monkeypatch, engine):
    monkeypatch.setenv("NPC_STEP2", "1")
    monkeypatch.setenv("NPC_ST_TMA" if engine == "tma" else "NPC_ST_NOTMA", "1")
    if engine == "tma":
        monkeypatch.setenv("NPC_ST_TMA2", "1")
    w = W.config2(side=30)
    orc = oracle.Operator(w)
    lo_o, hi_o = oracle.estimate_spectrum(orc, 20, W.lanczos_start(w["n"]))
    _, st_o = oracle.pcg(orc, w["b"], 30, lo_o, hi_o, 0.0, tol=w["tol"], maxit=2000)
    op = npc.create_from_workload(ctx, w, "stencil")
    lo, hi = npc.npc_estimate_spectrum(op, 20, None)
    poly = npc.npc_set_poly(op, 30, lo, hi, 0.0)
    x = torch.zeros(w["n"], dtype=torch.float64, device="cuda")
    st = npc.npc_pcg_solve(poly, op, torch.tensor(w["b"], device="cuda"), x, w["tol"], 2000)
    assert st["converged"] and abs(st["iters"] - st_o["iters"]) <= 2 and st["relres_true"] <= w["tol"]
