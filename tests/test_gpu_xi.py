"""GPU vs oracle at every xi of the sweep (DESIGN reading A12: xi in {0, 1e-4, 1e-3, 1e-2},
Eq. thetamod) and at several spectrum-estimate lengths (Lanczos m in
{20, 50, 100}): p_k(A) v to 1e-10 and PCG iterations within +-2 of the oracle's textbook PCG,
each side with its own estimate, on configs 1 (64x64), 2 (24^3) and 3 (64^3).
"""
import numpy as np
import pytest

import oracle
import workloads as W

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2208_01339_b200 as npc  # noqa: E402

XIS = [0.0, 1e-4, 1e-3, 1e-2]
WL = {"c1": (lambda: W.config1(), "csr"), "c2": (lambda: W.config2(side=24), "stencil"),
      "c3_64": (lambda: W.config3(side=64), "csr")}
_cache = {}


@pytest.fixture(scope="module")
def ctx():
    return npc.npc_context_create(0)


def _get(ctx, name):
    if name not in _cache:
        make, kind = WL[name]
        w = make()
        _cache[name] = (w, oracle.Operator(w), npc.create_from_workload(ctx, w, kind))
    return _cache[name]


@pytest.mark.parametrize("name", list(WL))
@pytest.mark.parametrize("xi", XIS)
def test_xi_pcg_iterations(ctx, name, xi):
    w, orc, op = _get(ctx, name)
    k = w["k"]
    lo_o, hi_o = oracle.estimate_spectrum(orc, 20, W.lanczos_start(w["n"]))
    _, st_o = oracle.pcg(orc, w["b"], k, lo_o, hi_o, xi, tol=w["tol"], maxit=20000)
    lo, hi = npc.npc_estimate_spectrum(op, 20, None)
    x = torch.zeros(w["n"], dtype=torch.float64, device="cuda")
    st = npc.npc_pcg_solve(npc.npc_set_poly(op, k, lo, hi, xi), op, torch.tensor(w["b"], device="cuda"), x,
                           w["tol"], 20000)
    assert st_o["converged"] and st["converged"] and st["relres_true"] <= w["tol"]
    assert abs(st["iters"] - st_o["iters"]) <= 2, (name, xi, st["iters"], st_o["iters"])
    # p_k(A) v with the oracle's interval at this xi
    r = np.random.default_rng(9).uniform(-1, 1, w["n"])
    z = torch.empty(w["n"], dtype=torch.float64, device="cuda")
    npc.npc_apply_poly(npc.npc_set_poly(op, k, lo_o, hi_o, xi), torch.tensor(r, device="cuda"), z)
    ref = oracle.cheb_apply(orc, k, lo_o, hi_o, xi, r)
    assert np.linalg.norm(z.cpu().numpy() - ref) <= 1e-10 * np.linalg.norm(ref)


@pytest.mark.parametrize("name", ["c1", "c3_64"])
@pytest.mark.parametrize("m", [50, 100])
def test_lanczos_steps_pcg_iterations(ctx, name, m):
    """Longer spectrum estimates (the sweep's m = 50, 100): same +-2 iteration parity, and the
    top Ritz value agrees with the oracle's (it has converged; the bottom one has not, A24)."""
    w, orc, op = _get(ctx, name)
    k = w["k"]
    a, b = oracle.lanczos(orc, m, W.lanczos_start(w["n"]))
    th_o, rho_o = oracle.ritz_upper(a, b)
    lo_o, hi_o = oracle.estimate_spectrum(orc, m, W.lanczos_start(w["n"]))
    ex = npc.npc_estimate_spectrum_ex(op, m, None)
    assert abs(ex["theta_max"] - th_o) <= 1e-8 * th_o
    _, st_o = oracle.pcg(orc, w["b"], k, lo_o, hi_o, 0.0, tol=w["tol"], maxit=20000)
    lo, hi = npc.npc_estimate_spectrum(op, m, None)
    x = torch.zeros(w["n"], dtype=torch.float64, device="cuda")
    st = npc.npc_pcg_solve(npc.npc_set_poly(op, k, lo, hi, 0.0), op, torch.tensor(w["b"], device="cuda"), x,
                           w["tol"], 20000)
    assert st["converged"] and abs(st["iters"] - st_o["iters"]) <= 2, (name, m, st["iters"], st_o["iters"])
