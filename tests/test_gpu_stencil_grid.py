"""GPU: all k degrees of p_k(A) r in one cooperative launch for L2-resident stencils
(op_stencil.cu k_stencil_poly_grid: the default for single-rank odd-nx stencils whose four vectors
fit L2, NPC_GRID_POLY=1 for even nx, where the 128-bit per-degree kernels are faster) against k launches of the per-degree kernel (NPC_NO_GRID_POLY=1,
k_stencil_step) and the oracle (Alg. 2 verbatim), through the C ABI.

Same decomposition and the same explicit FMAs per element, so s_k must be BITWISE equal to
the per-degree path; against the oracle the usual bars hold (p_k(A) v 1e-10, PCG +-2).
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


@pytest.fixture(scope="module")
def ctx():
    c = npc.npc_context_create(0)
    yield c
    torch.cuda.synchronize()


def dev(a):
    return torch.tensor(np.ascontiguousarray(a, dtype=np.float64), device="cuda")


class per_degree:
    """NPC_NO_GRID_POLY=1 while active: the library takes k launches of the per-degree kernel."""

    def __enter__(self):
        os.environ["NPC_NO_GRID_POLY"] = "1"

    def __exit__(self, *a):
        os.environ.pop("NPC_NO_GRID_POLY", None)


def stencil2d(nx, ny, seed=0):
    b = np.random.default_rng(seed).uniform(-1, 1, nx * ny)
    return dict(kind="stencil", name=f"st2d_{nx}x{ny}", n=nx * ny, dim=2, nx=nx, ny=ny, nz=1, diag=4.0, offdiag=-1.0,
                b=b, tol=1e-8)


def stencil3d(nx, ny, nz, seed=1):
    b = np.random.default_rng(seed).uniform(-1, 1, nx * ny * nz)
    return dict(kind="stencil", name=f"st3d_{nx}x{ny}x{nz}", n=nx * ny * nz, dim=3, nx=nx, ny=ny, nz=nz, diag=6.0,
                offdiag=-1.0, b=b, tol=1e-10)


CASES = {
    "c2_24": lambda: W.config2(side=24),
    "c2_64": lambda: W.config2(side=64),
    "box_40x24x9": lambda: stencil3d(40, 24, 9),       # ragged tiles in x and y, short z
    "box_67x33x17": lambda: stencil3d(67, 33, 17),     # odd nx, ragged z chunk
    "tall_8x8x300": lambda: stencil3d(8, 8, 300),      # fewer items than CTAs per z column
    "2d_64x23": lambda: stencil2d(64, 23),
    "2d_131x66": lambda: stencil2d(131, 66),
    "c2_128": lambda: W.config2(side=128),             # BASELINE config 2 at full size
}


@pytest.mark.parametrize("name", list(CASES))
def test_grid_poly_bitwise_equals_per_degree_and_oracle(ctx, name):
    w = CASES[name]()
    n = w["n"]
    op = npc.create_from_workload(ctx, w, "stencil")
    orc = oracle.Operator(w)
    lo, hi = oracle.estimate_spectrum(orc, 20, W.lanczos_start(n))
    r = np.random.default_rng(4).uniform(-1, 1, n)
    zg, zd = (torch.empty(n, dtype=torch.float64, device="cuda") for _ in range(2))
    ks = (1, 2, 3, 30) if n > 1_000_000 else (1, 2, 3, 8, 30, 200)
    for k in ks:
        for xi in (0.0, 1e-3):
            os.environ["NPC_GRID_POLY"] = "1"  # even nx: the per-degree 128-bit kernels are the default
            try:
                npc.npc_apply_poly(npc.npc_set_poly(op, k, lo, hi, xi), dev(r), zg)
            finally:
                os.environ.pop("NPC_GRID_POLY", None)
            with per_degree():
                npc.npc_apply_poly(npc.npc_set_poly(op, k, lo, hi, xi), dev(r), zd)
            assert torch.equal(zg, zd), (k, xi)
            if xi == 0.0 or k <= 30:
                refz = oracle.cheb_apply(orc, k, lo, hi, xi, r)
                assert np.linalg.norm(zg.cpu().numpy() - refz) <= 1e-10 * np.linalg.norm(refz), (k, xi)


@pytest.mark.parametrize("name,k", [("c2_24", 10), ("c2_64", 30), ("2d_64x23", 10), ("box_67x33x17", 7),
                                    ("c2_64", 40)])  # k >= 32: first iteration eager (grid kernel), then the graph
def test_grid_poly_pcg_parity(ctx, name, k):
    """PCG with the fused-poly kernel (gamma partial from its last degree) against the oracle's
    textbook PCG (+-2 iterations, true residual <= tol) and the per-degree path.  By default
    the PCG's captured graph takes the per-degree kernels (faster there); NPC_GRID_IN_GRAPH=1
    puts the cooperative kernel into the graph, which must work and agree."""
    w = CASES[name]()
    n = w["n"]
    orc = oracle.Operator(w)
    lo_o, hi_o = oracle.estimate_spectrum(orc, 20, W.lanczos_start(n))
    _, st_o = oracle.pcg(orc, w["b"], k, lo_o, hi_o, 0.0, tol=w["tol"], maxit=5000)
    res = []
    for grid in (True, False):
        op = npc.create_from_workload(ctx, w, "stencil")
        lo, hi = npc.npc_estimate_spectrum(op, 20, None)
        x = torch.zeros(n, dtype=torch.float64, device="cuda")
        if grid:
            os.environ["NPC_GRID_IN_GRAPH"] = "1"
            try:
                st = npc.npc_pcg_solve(npc.npc_set_poly(op, k, lo, hi, 0.0), op, dev(w["b"]), x, w["tol"], 5000)
            finally:
                os.environ.pop("NPC_GRID_IN_GRAPH", None)
        else:
            with per_degree():
                st = npc.npc_pcg_solve(npc.npc_set_poly(op, k, lo, hi, 0.0), op, dev(w["b"]), x, w["tol"], 5000)
        assert st["converged"] and abs(st["iters"] - st_o["iters"]) <= 2, (grid, st, st_o)
        assert st["relres_true"] <= w["tol"]
        res.append((st["iters"], x))
    # the gamma partials are summed per CTA of a different grid: same iterates up to rounding
    assert abs(res[0][0] - res[1][0]) <= 1
    assert torch.allclose(res[0][1], res[1][1], rtol=1e-9, atol=1e-12)


def test_grid_poly_done_flag_noop(ctx):
    """A converged PCG's later graph-replayed applications must not touch z (the done flag
    is read once, uniformly, before any degree)."""
    w = CASES["c2_24"]()
    n = w["n"]
    op = npc.create_from_workload(ctx, w, "stencil")
    lo, hi = npc.npc_estimate_spectrum(op, 20, None)
    poly = npc.npc_set_poly(op, 10, lo, hi, 0.0)
    x = torch.zeros(n, dtype=torch.float64, device="cuda")
    st = npc.npc_pcg_solve(poly, op, dev(w["b"]), x, w["tol"], 5000)
    assert st["converged"]
    x2 = torch.zeros(n, dtype=torch.float64, device="cuda")
    st2 = npc.npc_pcg_solve(poly, op, dev(w["b"]), x2, w["tol"], 5000)
    assert st2["iters"] == st["iters"] and torch.equal(x, x2)
