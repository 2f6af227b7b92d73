"""GPU: the CSR operator's coded column ids (op_csr.cu: per-tile dictionary of column offsets,
one byte per nonzero) against the plain int32 form and the oracle, through the C ABI.

The coded form changes only how column ids are stored: same values, same per-row summation
order, so every result must be BITWISE equal to the plain form (NPC_CSR_PLAIN=1).  Matrices
whose tiles have more than 256 distinct offsets (unstructured kNN in natural order) fall back
to the plain form; npc_operator_matrix_bytes tells which form was stored.
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


FORM_ENV = {"plain": "NPC_CSR_PLAIN", "coded": "NPC_CSR_CODED", "nomirror": "NPC_CSR_NOMIRROR",
            "nostage": "NPC_CSR_NOSTAGE", "stage": "NPC_CSR_NORING", "nofill": "NPC_CSR_NOFILL",
            "ring2": "NPC_RING_NS=2", "rpt4": "NPC_RING_RPT=4",
            "wave": "NPC_CSR_WAVE", "lag1": "NPC_CSR_WAVE,NPC_WAVE_LAG=1",
            "wavep": "NPC_CSR_WAVE,NPC_WAVE_PERSIST", "wavep1": "NPC_CSR_WAVE,NPC_WAVE_PERSIST,NPC_WAVE_LAG=1"}


def make(ctx, w, plain):
    """plain: True -> int32 column ids, False -> the coded form; or a form name: 'pattern'
    (the default form: ring kernel), 'nomirror' (pattern ids without symmetric mirroring), 'nostage'
    (pattern form without the x-window staging kernels), 'stage' (k_csr_pat_stage instead of the
    ring kernel), 'ring2' (persistent ring kernel, 2 stages), 'rpt4' (4 rows per thread), 'wave' (two degrees per
    pass: the wave kernel), 'lag1' (the wave kernel at its smallest lag), 'wavep' / 'wavep1' (its persistent producer-warp
    form, default / smallest lag), 'nofill' (no
    earlier-tile mirrors moved into ELL padding), 'coded', 'plain'."""
    form = ("plain" if plain else "coded") if isinstance(plain, bool) else plain
    env = FORM_ENV.get(form)
    kv = [(e.split("=", 1) if "=" in e else (e, "1")) for e in env.split(",")] if env else []
    for key, val in kv:
        os.environ[key] = val
    try:
        return npc.create_from_workload(ctx, w, "csr")
    finally:
        for key, _ in kv:
            os.environ.pop(key, None)


WL = {"c3": lambda: W.config3(side=30), "c1": lambda: W.config1(side=64),
      "c3_ragged": lambda: W.config3(side=23)}  # 12,167 rows: a ragged last tile


@pytest.mark.parametrize("name", list(WL))
def test_coded_bitwise_equals_plain(ctx, name):
    w = WL[name]()
    n, nnz = w["n"], int(w["rowptr"][-1])
    opc, opp = make(ctx, w, False), make(ctx, w, True)
    mb_c, mb_p = npc.npc_operator_matrix_bytes(opc), npc.npc_operator_matrix_bytes(opp)
    assert mb_p == 12 * nnz + 4 * (n + 1)
    assert mb_c < 9.5 * nnz + 4 * (n + 1), (mb_c, nnz)  # coded: 9 B/nnz + small dictionaries
    x = np.random.default_rng(1).standard_normal(n)
    yc = torch.empty(n, dtype=torch.float64, device="cuda")
    yp = torch.empty_like(yc)
    npc.npc_apply_operator(opc, dev(x), yc)
    npc.npc_apply_operator(opp, dev(x), yp)
    assert torch.equal(yc, yp)
    orc = oracle.Operator(w)
    assert np.linalg.norm(yc.cpu().numpy() - orc.apply(x)) <= 1e-13 * np.linalg.norm(orc.apply(x))
    lo, hi = oracle.estimate_spectrum(orc, 20, W.lanczos_start(n))
    r = np.random.default_rng(2).uniform(-1, 1, n)
    zc, zp = torch.empty_like(yc), torch.empty_like(yc)
    os.environ["NPC_NO_CLUSTER"] = "1"  # config 1 would otherwise take the cluster-resident kernel
    try:
        pc, pp = npc.npc_set_poly(opc, 17, lo, hi, 1e-3), npc.npc_set_poly(opp, 17, lo, hi, 1e-3)
        npc.npc_apply_poly(pc, dev(r), zc)
        npc.npc_apply_poly(pp, dev(r), zp)
    finally:
        os.environ.pop("NPC_NO_CLUSTER", None)
    assert torch.equal(zc, zp)
    ref = oracle.cheb_apply(orc, 17, lo, hi, 1e-3, r)
    assert np.linalg.norm(zc.cpu().numpy() - ref) <= 1e-10 * np.linalg.norm(ref)


def test_unstructured_falls_back_to_plain(ctx):
    w = W.config4(n=12_000)  # kNN rows: thousands of distinct offsets per 256-row tile
    n, nnz = w["n"], int(w["rowptr"][-1])
    op = npc.create_from_workload(ctx, w, "csr")
    assert npc.npc_operator_matrix_bytes(op) == 12 * nnz + 4 * (n + 1)
    x = np.random.default_rng(3).standard_normal(n)
    y = torch.empty(n, dtype=torch.float64, device="cuda")
    npc.npc_apply_operator(op, dev(x), y)
    ref = oracle.Operator(w).apply(x)
    assert np.linalg.norm(y.cpu().numpy() - ref) <= 1e-13 * np.linalg.norm(ref)


def test_coded_pcg_matches_plain(ctx):
    """Whole PCG (graph-captured degree kernels) on the coded form: the same iterates."""
    w = W.config3(side=20)
    n = w["n"]
    res = []
    for plain in (False, True):
        op = make(ctx, w, plain)
        lo, hi = npc.npc_estimate_spectrum(op, 20, None)
        poly = npc.npc_set_poly(op, 20, lo, hi, 0.0)
        x = torch.zeros(n, dtype=torch.float64, device="cuda")
        st = npc.npc_pcg_solve(poly, op, dev(w["b"]), x, w["tol"], 5000)
        res.append((st["iters"], x))
    assert res[0][0] == res[1][0] and torch.equal(res[0][1], res[1][1])


def banded_spd(n, hb, seed):
    """SPD band matrix, half-bandwidth hb (2 hb + 1 entries per interior row), diagonally
    dominant: a coded matrix whose 512-row tiles exceed the staged kernel's shared memory."""
    rng = np.random.default_rng(seed)
    rows, cols, vals = [], [], []
    off = {}
    for i in range(n):
        for j in range(max(0, i - hb), min(n, i + hb + 1)):
            if j < i:
                v = off[(j, i)]
            elif j > i:
                v = off[(i, j)] = -rng.uniform(0.1, 1.0)
            else:
                continue
            rows.append(i), cols.append(j), vals.append(v)
    A = np.zeros((n, n))
    A[rows, cols] = vals
    A[np.arange(n), np.arange(n)] = -A.sum(axis=1) + 1.0
    rp = np.zeros(n + 1, dtype=np.int64)
    nz = A != 0
    rp[1:] = np.cumsum(nz.sum(axis=1))
    ci = np.nonzero(nz)[1].astype(np.int32)
    return dict(kind="csr", n=n, rowptr=rp.astype(np.int32), colidx=ci, vals=A[nz].astype(np.float64))


def test_coded_unstaged_tiles(ctx):
    """Tiles of 512 rows x 121 entries (62K entries, ~550 KB) take the coded kernel's
    non-staged form (codes and values read straight from HBM); bitwise equal to plain."""
    w = banded_spd(3000, 60, seed=4)
    n, nnz = w["n"], int(w["rowptr"][-1])
    opc, opp = make(ctx, w, False), make(ctx, w, True)
    assert npc.npc_operator_matrix_bytes(opc) < npc.npc_operator_matrix_bytes(opp)  # coded
    x = np.random.default_rng(5).standard_normal(n)
    yc = torch.empty(n, dtype=torch.float64, device="cuda")
    yp = torch.empty_like(yc)
    os.environ["NPC_NO_CLUSTER"] = "1"
    try:
        npc.npc_apply_operator(opc, dev(x), yc)
        npc.npc_apply_operator(opp, dev(x), yp)
        assert torch.equal(yc, yp)
        orc = oracle.Operator(w)
        ref = orc.apply(x)
        assert np.linalg.norm(yc.cpu().numpy() - ref) <= 1e-13 * np.linalg.norm(ref)
        lo, hi = oracle.estimate_spectrum(orc, 20, W.lanczos_start(n))
        r = np.random.default_rng(6).uniform(-1, 1, n)
        zc, zp = torch.empty_like(yc), torch.empty_like(yc)
        npc.npc_apply_poly(npc.npc_set_poly(opc, 9, lo, hi, 0.0), dev(r), zc)
        npc.npc_apply_poly(npc.npc_set_poly(opp, 9, lo, hi, 0.0), dev(r), zp)
        assert torch.equal(zc, zp)
        refz = oracle.cheb_apply(orc, 9, lo, hi, 0.0, r)
        assert np.linalg.norm(zc.cpu().numpy() - refz) <= 1e-10 * np.linalg.norm(refz)
    finally:
        os.environ.pop("NPC_NO_CLUSTER", None)
    assert nnz > 512 * 100


def empty_tile_csr(n=3000, first=18, empty_to=1600):
    """Rows [0, first) and [empty_to, n) hold a diagonal entry, rows [first, empty_to) are
    empty: whole 256-row (plain) and 512-row (coded) tiles with no entries, starting at entry
    offset 18 (= 2 mod 4 and not a multiple of 16), where the bulk copies' aligned spans are
    nonzero for an empty tile (the barrier used to wait for bytes never sent)."""
    lens = np.ones(n, dtype=np.int64)
    lens[first:empty_to] = 0
    rowptr = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
    rows = np.flatnonzero(lens)
    return dict(kind="csr", n=n, rowptr=rowptr, colidx=rows.astype(np.int32),
                vals=np.arange(1, len(rows) + 1, dtype=np.float64))


@pytest.mark.parametrize("plain", ["pattern", "coded", "plain"])
def test_empty_tiles_at_unaligned_offsets(ctx, plain):
    w = empty_tile_csr()
    op = make(ctx, w, plain)
    x = np.random.default_rng(2).standard_normal(w["n"])
    y = torch.empty(w["n"], dtype=torch.float64, device="cuda")
    npc.npc_apply_operator(op, dev(x), y)
    torch.cuda.synchronize()
    assert np.array_equal(y.cpu().numpy(), oracle.Operator(w).apply(x))
