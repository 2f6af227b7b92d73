"""GPU: the 128-bit register stencil kernel (op_stencil.cu k_stencil_step_v2: two x-points per
thread, every stream moved as double2) against the scalar per-degree kernel k_stencil_step and
the oracle (Alg. 2 verbatim), through the C ABI.

Same neighbour order and explicit FMAs per element, so p_k(A) r must be BITWISE equal to the
scalar kernel; the fused dot partial is summed in another order (thread = two points), so PCG is
held to the usual bars (iterations +-2 of the oracle, true residual <= tol).  Odd nx cannot
take the kernel (pairs would straddle rows): the library must fall back silently.
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
from test_gpu_stencil_grid import stencil2d, stencil3d  # noqa: E402  (seeded generators only)


@pytest.fixture(scope="module")
def ctx():
    c = npc.npc_context_create(0)
    yield c
    torch.cuda.synchronize()


class env:
    def __init__(self, **kv):
        self.kv = kv

    def __enter__(self):
        for k, v in self.kv.items():
            os.environ[k] = v

    def __exit__(self, *a):
        for k in self.kv:
            os.environ.pop(k, None)


CASES = {
    "c2_24": lambda: W.config2(side=24),
    "c2_64": lambda: W.config2(side=64),
    "box_40x24x9": lambda: stencil3d(40, 24, 9),       # ragged tiles in x and y, short z
    "box_66x33x17": lambda: stencil3d(66, 33, 17),     # nx = 2 past a tile, odd ny, ragged z chunk
    "box_67x33x17": lambda: stencil3d(67, 33, 17),     # odd nx: falls back to the scalar kernel
    "thin_2x5x40": lambda: stencil3d(2, 5, 40),        # one pair per row: no x neighbour loads
    "2d_64x23": lambda: stencil2d(64, 23),
    "2d_130x66": lambda: stencil2d(130, 66),
    "c2_128": lambda: W.config2(side=128),             # BASELINE config 2 at full size
}


@pytest.mark.parametrize("name", list(CASES))
def test_vec2_bitwise_equals_scalar_kernel_and_oracle(ctx, name):
    w = CASES[name]()
    n = w["n"]
    orc = oracle.Operator(w)
    lo, hi = oracle.estimate_spectrum(orc, 20, W.lanczos_start(n))
    r = np.random.default_rng(4).uniform(-1, 1, n)
    # per-degree launches on both sides (the cooperative all-degree kernel has its own test)
    with env(NPC_NO_GRID_POLY="1", NPC_ST_NOTMA="1", NPC_ST_NOV2="1"):
        op_s = npc.create_from_workload(ctx, w, "stencil")
    with env(NPC_NO_GRID_POLY="1", NPC_ST_NOTMA="1", NPC_ST_V2="1"):
        op_v = npc.create_from_workload(ctx, w, "stencil")
    zs, zv, y_s, y_v = (torch.empty(n, dtype=torch.float64, device="cuda") for _ in range(4))
    rd = torch.tensor(r, device="cuda")
    npc.npc_apply_operator(op_s, rd, y_s)
    npc.npc_apply_operator(op_v, rd, y_v)
    assert torch.equal(y_s, y_v)
    assert np.linalg.norm(y_v.cpu().numpy() - orc.apply(r)) <= 1e-13 * np.linalg.norm(orc.apply(r))
    for k in ((1, 2, 3, 30) if n > 1_000_000 else (1, 2, 3, 8, 30, 200)):
        for xi in (0.0, 1e-3):
            with env(NPC_NO_GRID_POLY="1"):
                ps = npc.npc_set_poly(op_s, k, lo, hi, xi)
                pv = npc.npc_set_poly(op_v, k, lo, hi, xi)
                npc.npc_apply_poly(ps, rd, zs)
                npc.npc_apply_poly(pv, rd, zv)
            assert torch.equal(zs, zv), (name, k, xi)
        ref = oracle.cheb_apply(orc, k, lo, hi, 1e-3, r)
        assert np.linalg.norm(zv.cpu().numpy() - ref) <= 1e-10 * np.linalg.norm(ref)
    # PCG through the vectorised kernel (captured in the iteration graph)
    k = 8
    _, st_o = oracle.pcg(orc, w["b"], k, lo, hi, 0.0, tol=w["tol"], maxit=5000)
    pv = npc.npc_set_poly(op_v, k, lo, hi, 0.0)
    b = torch.tensor(w["b"], device="cuda")
    x = torch.zeros_like(b)
    st = npc.npc_pcg_solve(pv, op_v, b, x, w["tol"], 5000)
    assert st["converged"] and st["relres_true"] <= w["tol"]
    assert abs(st["iters"] - st_o["iters"]) <= 2
