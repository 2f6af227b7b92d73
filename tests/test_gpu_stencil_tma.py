"""GPU: the TMA-staged stencil kernel (op_stencil.cu k_stencil_tma: each z-plane of the input
arrives as one cp.async.bulk.tensor box with its in-plane halo, out-of-grid elements
zero-filled by the hardware = the Dirichlet boundary) against the register-marching kernel
(NPC_ST_NOTMA=1, k_stencil_step) and the oracle, through the C ABI.

Same neighbour-sum order (a zero-filled neighbour adds +0.0), so the two kernels must agree
BITWISE; against the oracle the usual bars hold (operator 1e-13, p_k(A) v 1e-10, PCG +-2).
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


def make(ctx, w, tma):
    """tma: force the TMA kernel on (NPC_ST_TMA=1; by default it serves only grids whose vectors
    exceed L2) or off (NPC_ST_NOTMA=1)."""
    var = "NPC_ST_TMA" if tma else "NPC_ST_NOTMA"
    os.environ[var] = "1"
    try:
        return npc.create_from_workload(ctx, w, "stencil")
    finally:
        os.environ.pop(var, None)


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
    "box_66x34x33": lambda: stencil3d(66, 34, 33),     # one column past a tile boundary
    "flat_96x80x2": lambda: stencil3d(96, 80, 2),
    "2d_64x23": lambda: stencil2d(64, 23),
    "2d_130x66": lambda: stencil2d(130, 66),
    "c2_200": lambda: W.config2(side=200),           # above 3/4 of L2: the default path
}


@pytest.mark.parametrize("name", list(CASES))
def test_tma_bitwise_equals_register_kernel_and_oracle(ctx, name):
    w = CASES[name]()
    n = w["n"]
    opt, opr = make(ctx, w, True), make(ctx, w, False)
    x = np.random.default_rng(3).standard_normal(n)
    yt, yr = (torch.empty(n, dtype=torch.float64, device="cuda") for _ in range(2))
    npc.npc_apply_operator(opt, dev(x), yt)
    npc.npc_apply_operator(opr, dev(x), yr)
    assert torch.equal(yt, yr)
    orc = oracle.Operator(w)
    ref = orc.apply(x)
    assert np.linalg.norm(yt.cpu().numpy() - ref) <= 1e-13 * np.linalg.norm(ref)
    lo, hi = oracle.estimate_spectrum(orc, 20, W.lanczos_start(n))
    r = np.random.default_rng(4).uniform(-1, 1, n)
    zt, zr = torch.empty_like(yt), torch.empty_like(yt)
    for k in (1, 2, 7, 30):
        npc.npc_apply_poly(npc.npc_set_poly(opt, k, lo, hi, 1e-3), dev(r), zt)
        npc.npc_apply_poly(npc.npc_set_poly(opr, k, lo, hi, 1e-3), dev(r), zr)
        assert torch.equal(zt, zr), k
        refz = oracle.cheb_apply(orc, k, lo, hi, 1e-3, r)
        assert np.linalg.norm(zt.cpu().numpy() - refz) <= 1e-10 * np.linalg.norm(refz), k


@pytest.mark.parametrize("name", ["c2_24", "2d_64x23", "box_66x34x33"])
def test_tma_pcg_parity(ctx, name):
    w = CASES[name]()
    n = w["n"]
    orc = oracle.Operator(w)
    lo_o, hi_o = oracle.estimate_spectrum(orc, 20, W.lanczos_start(n))
    _, st_o = oracle.pcg(orc, w["b"], 10, lo_o, hi_o, 0.0, tol=w["tol"], maxit=5000)
    res = []
    for tma in (True, False):
        op = make(ctx, w, tma)
        lo, hi = npc.npc_estimate_spectrum(op, 20, None)
        poly = npc.npc_set_poly(op, 10, lo, hi, 0.0)
        x = torch.zeros(n, dtype=torch.float64, device="cuda")
        st = npc.npc_pcg_solve(poly, op, dev(w["b"]), x, w["tol"], 5000)
        assert st["converged"] and abs(st["iters"] - st_o["iters"]) <= 2, (st, st_o)
        res.append((st["iters"], x))
    # same iterates up to the order of the per-CTA dot partials (the two kernels group rows
    # into different CTAs): identical iteration count, solutions within rounding
    assert res[0][0] == res[1][0]
    assert torch.allclose(res[0][1], res[1][1], rtol=1e-11, atol=1e-14)


def test_tma_misaligned_vector_falls_back(ctx):
    w = CASES["c2_24"]()
    n = w["n"]
    op = make(ctx, w, True)
    x = np.random.default_rng(5).standard_normal(n)
    buf = torch.zeros(n + 1, dtype=torch.float64, device="cuda")
    buf[1:] = dev(x)
    y1, y2 = (torch.empty(n, dtype=torch.float64, device="cuda") for _ in range(2))
    npc.npc_apply_operator(op, buf[1:], y1)
    npc.npc_apply_operator(op, dev(x), y2)
    assert torch.equal(y1, y2)
