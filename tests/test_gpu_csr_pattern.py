"""GPU: the CSR operator's pattern form (op_csr.cu k_csr_pat_step: one pattern id per row,
lower-triangle values mirrored from their bitwise-equal transposes) against the plain int32
form and the oracle, through the C ABI.

Like the coded form it changes only how the matrix is stored: the same values are summed in
the same (ascending column) order, so every result is BITWISE equal to the plain form.
npc_operator_matrix_bytes tells which form was stored: a symmetric matrix streams its upper
triangle + diagonal (own values, in tile-ELL blocks) at 8 B each plus 1 B per row.
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
from test_gpu_csr_coded import banded_spd, make  # noqa: E402


@pytest.fixture(scope="module")
def ctx():
    c = npc.npc_context_create(0)
    yield c
    torch.cuda.synchronize()


def dev(a):
    return torch.tensor(np.ascontiguousarray(a, dtype=np.float64), device="cuda")


def upper_count(w):
    rp, ci = w["rowptr"], w["colidx"]
    rows = np.repeat(np.arange(w["n"]), np.diff(rp))
    return int(np.sum(ci >= rows))


def perturb_lower(w, row_hi, seed):
    """Break the symmetry of every lower entry of rows [0, row_hi) (their values no longer
    equal the transposes'): those entries become own entries, the rest stay mirrored."""
    w = dict(w)
    v = w["vals"].copy()
    rows = np.repeat(np.arange(w["n"]), np.diff(w["rowptr"]))
    pick = np.flatnonzero((w["colidx"] < rows) & (rows < row_hi))
    v[pick] *= 1.0 + 1e-12
    w["vals"] = v
    return w, len(pick)


WL = {"c3": lambda: W.config3(side=30), "c3_ragged": lambda: W.config3(side=23), "c1": lambda: W.config1(side=64),
      "c2csr": lambda: dict(kind="csr", n=40 ** 3, name="c2csr",
                            **dict(zip(("rowptr", "colidx", "vals"),
                                       W.grid_laplacian_csr((40, 40, 40), 6.0, -1.0)))),
      "band": lambda: banded_spd(4000, 7, seed=2),
      "c3_odd": lambda: W.config3(side=21)}  # n = 9,261 odd: window tails


def _all_forms_bitwise(ctx, w, k=17, xi=1e-3):
    n = w["n"]
    ops = {f: make(ctx, w, f)
           for f in ("pattern", "nomirror", "nostage", "stage", "ring2", "rpt4", "wave", "lag1", "wavep", "wavep1", "nofill", "coded",
                     "plain")}
    x = np.random.default_rng(1).standard_normal(n)
    ys = {}
    os.environ["NPC_NO_CLUSTER"] = "1"
    try:
        for f, op in ops.items():
            y = torch.empty(n, dtype=torch.float64, device="cuda")
            npc.npc_apply_operator(op, dev(x), y)
            ys[f] = y
        for f in ys:
            assert torch.equal(ys[f], ys["plain"]), f
        orc = oracle.Operator(w)
        ref = orc.apply(x)
        assert np.linalg.norm(ys["pattern"].cpu().numpy() - ref) <= 1e-13 * np.linalg.norm(ref)
        lo, hi = oracle.estimate_spectrum(orc, 20, W.lanczos_start(n))
        r = np.random.default_rng(2).uniform(-1, 1, n)
        zs = {}
        for f, op in ops.items():
            z = torch.empty(n, dtype=torch.float64, device="cuda")
            npc.npc_apply_poly(npc.npc_set_poly(op, k, lo, hi, xi), dev(r), z)
            zs[f] = z
        for f in zs:
            assert torch.equal(zs[f], zs["plain"]), f
        refz = oracle.cheb_apply(orc, k, lo, hi, xi, r)
        assert np.linalg.norm(zs["pattern"].cpu().numpy() - refz) <= 1e-10 * np.linalg.norm(refz)
    finally:
        os.environ.pop("NPC_NO_CLUSTER", None)
    return ops


@pytest.mark.parametrize("name", list(WL))
def test_pattern_bitwise_equals_plain(ctx, name):
    w = WL[name]()
    n, nnz = w["n"], int(w["rowptr"][-1])
    ops = _all_forms_bitwise(ctx, w)
    mb = npc.npc_operator_matrix_bytes(ops["pattern"])
    # symmetric: own values = upper triangle + diagonal, 8 B each (+ tile-ELL padding of the
    # boundary rows), + 1 B per row + tables
    own = upper_count(w)
    assert 8 * own + n <= mb <= 8 * own * 1.125 + n + 0.02 * 8 * nnz + 64 * 1024, (mb, own, nnz)
    assert npc.npc_operator_matrix_bytes(ops["nomirror"]) >= 8 * nnz + n


def test_pattern_partially_symmetric(ctx):
    """Lower entries whose transpose differs by a 1e-12 relative factor (all of the first
    tile's) are stored as own entries, not mirrored: the operator stays in the pattern form
    (fewer bytes than coded), stores more values, and results stay bitwise equal."""
    w0 = W.config3(side=24)
    w, nbroken = perturb_lower(w0, 512, seed=7)
    assert nbroken > 500
    _all_forms_bitwise(ctx, w, k=5, xi=0.0)
    mb0 = npc.npc_operator_matrix_bytes(make(ctx, w0, "pattern"))
    mb = npc.npc_operator_matrix_bytes(make(ctx, w, "pattern"))
    mbc = npc.npc_operator_matrix_bytes(make(ctx, w, "coded"))
    assert mb0 + 8 * nbroken <= mb < mbc, (mb, mb0, mbc, nbroken)


def test_pattern_pcg_matches_plain(ctx):
    """Whole PCG (graph-captured degree kernels) on the pattern form: the same iterates."""
    w = W.config3(side=20)
    n = w["n"]
    res = []
    for form in ("pattern", "plain"):
        op = make(ctx, w, form)
        lo, hi = npc.npc_estimate_spectrum(op, 20, None)
        poly = npc.npc_set_poly(op, 20, lo, hi, 0.0)
        x = torch.zeros(n, dtype=torch.float64, device="cuda")
        st = npc.npc_pcg_solve(poly, op, dev(w["b"]), x, w["tol"], 5000)
        res.append((st["iters"], x))
    for it, xf in res[1:]:
        assert it == res[0][0] and torch.equal(xf, res[0][1])


def test_ring_pcg_forms(ctx):
    """PCG through the pattern kernels (64,000 rows: above the cluster-resident size).  The
    one-tile-per-CTA ring kernel, its two-degree wave form (at the default and the smallest
    lag) and k_csr_pat_stage write the same z and the same per-tile dot partials: bitwise the
    same solve.  The persistent ring kernel (2 stages) and the
    4-rows-per-thread form sum the dot partials in another order: same iterations +-1."""
    w = W.config3(side=40)
    n = w["n"]
    res = {}
    for form in ("pattern", "stage", "ring2", "rpt4", "wave", "lag1", "wavep", "wavep1"):
        op = make(ctx, w, form)
        lo, hi = npc.npc_estimate_spectrum(op, 20, None)
        poly = npc.npc_set_poly(op, 20, lo, hi, 0.0)
        x = torch.zeros(n, dtype=torch.float64, device="cuda")
        st = npc.npc_pcg_solve(poly, op, dev(w["b"]), x, w["tol"], 5000)
        assert st["converged"] and st["relres_true"] <= w["tol"], (form, st)
        res[form] = (st["iters"], x)
    for f in ("stage", "wave", "lag1", "wavep", "wavep1"):  # two-degree wave passes: the same sums and partials
        assert res["pattern"][0] == res[f][0] and torch.equal(res["pattern"][1], res[f][1]), f
    for f in ("ring2", "rpt4"):
        assert abs(res[f][0] - res["pattern"][0]) <= 1, (f, res[f][0], res["pattern"][0])


def test_pattern_too_many_patterns_falls_back(ctx):
    """kNN rows in natural order: every row its own pattern (> 256 per tile) -> plain."""
    w = W.config4(n=12_000)
    n, nnz = w["n"], int(w["rowptr"][-1])
    op = make(ctx, w, "pattern")
    assert npc.npc_operator_matrix_bytes(op) == 12 * nnz + 4 * (n + 1)


def test_pattern_large_band_falls_back_to_coded(ctx):
    """61 own values per row x 512 rows exceed the shared-memory budget -> coded form."""
    w = banded_spd(3000, 60, seed=4)
    nnz = int(w["rowptr"][-1])
    mb = npc.npc_operator_matrix_bytes(make(ctx, w, "pattern"))
    assert mb < 9.5 * nnz + 4 * (w["n"] + 1) and mb > 8 * nnz


def test_pattern_misaligned_x(ctx):
    """An input vector that is only 8-byte aligned cannot feed the TMA window copies: every
    tile then runs k_csr_pat_step, same result."""
    w = W.config3(side=26)
    n = w["n"]
    op, opp = make(ctx, w, "pattern"), make(ctx, w, "plain")
    x = np.random.default_rng(9).standard_normal(n)
    buf = torch.zeros(n + 1, dtype=torch.float64, device="cuda")
    buf[1:] = dev(x)
    xm = buf[1:]
    assert xm.data_ptr() % 16 == 8
    y, yp = torch.empty(n, dtype=torch.float64, device="cuda"), torch.empty(n, dtype=torch.float64, device="cuda")
    npc.npc_apply_operator(op, xm, y)
    npc.npc_apply_operator(opp, dev(x), yp)
    assert torch.equal(y, yp)
