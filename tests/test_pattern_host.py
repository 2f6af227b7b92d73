"""CPU: the host logic of the CSR operator's pattern form and ring layout (op_csr.cu:
build_pattern, pattern_ring_table, the descriptor/table packing), through the host-only
npc_pattern_check (include/npc.h).  It replays every ring tile's bulk-copy descriptors into a
NaN-filled staging buffer and sums the rows from the entry table in the kernel's order, so a
wrong window offset, gap, far-mirror window, padding fill, table dedup or byte count shows up
here -- without a GPU -- as a wrong y, a NaN, or an NPC_ERR_INTERNAL naming the tile and copy.
The reference is the plain oracle's y = A x (oracle/, PAPER.md:269-295 operator application)."""
import os

import numpy as np
import pytest

import oracle
import workloads as W
import paper_2208_01339_b200 as npc


def grid_csr(shape, diag, off):
    rp, ci, va = W.grid_laplacian_csr(shape, diag, off)
    n = int(np.prod(shape))
    return dict(kind="csr", n=n, rowptr=rp, colidx=ci, vals=va)


def banded(n, hb, seed):
    """Symmetric diagonally dominant band matrix, half-bandwidth hb."""
    rng = np.random.default_rng(seed)
    A = np.zeros((n, n))
    for d in range(1, hb + 1):
        v = -rng.uniform(0.1, 1.0, n - d)
        A[np.arange(n - d), np.arange(d, n)] = v
        A[np.arange(d, n), np.arange(n - d)] = v
    A[np.arange(n), np.arange(n)] = -A.sum(axis=1) + 1.0
    nz = A != 0
    rp = np.zeros(n + 1, dtype=np.int32)
    rp[1:] = np.cumsum(nz.sum(axis=1))
    return dict(kind="csr", n=n, rowptr=rp, colidx=np.nonzero(nz)[1].astype(np.int32), vals=A[nz].astype(np.float64))


def perturbed(w, row_hi):
    """Lower entries of rows < row_hi no longer equal their transposes: stored as own values."""
    w = dict(w)
    v = w["vals"].copy()
    rows = np.repeat(np.arange(w["n"]), np.diff(w["rowptr"]))
    v[(w["colidx"] < rows) & (rows < row_hi)] *= 1.0 + 1e-12
    w["vals"] = v
    return w


CASES = {
    "c3_30": lambda: W.config3(side=30),        # N^2 = 900 < 1,024: -N^2 mirrors as column gaps
    "c3_40": lambda: W.config3(side=40),        # N^2 = 1,600: far windows over two earlier tiles
    "c3_23": lambda: W.config3(side=23),        # ragged last tile (odd row count 903)
    "c3_21": lambda: W.config3(side=21),        # n = 9,261 odd: x window tails
    "c3_64": lambda: W.config3(side=64),        # 256 tiles, interior tables shared
    "c1_64": lambda: W.config1(side=64),        # 2D 5-point
    "c2_40": lambda: grid_csr((40, 40, 40), 6.0, -1.0),
    "band7": lambda: banded(4000, 7, seed=2),
    "c3_partial": lambda: perturbed(W.config3(side=24), 512),
}


def check(w, env=None):
    x = np.random.default_rng(5).standard_normal(w["n"])
    for k, v in (env or {}).items():
        os.environ[k] = v
    try:
        y, info = npc.npc_pattern_check(w["rowptr"], w["colidx"], w["vals"], x)
    finally:
        for k in (env or {}):
            os.environ.pop(k, None)
    ref = oracle.Operator(w).apply(x)
    assert np.all(np.isfinite(y)), "a row read a stage byte no copy wrote"
    err = np.abs(y - ref) / (np.abs(ref) + np.abs(w["vals"]).max() * np.abs(x).max())
    assert err.max() <= 1e-14, (err.max(), info)
    return info


@pytest.mark.parametrize("name", list(CASES))
def test_ring_layout_replays_to_the_operator(name):
    info = check(CASES[name]())
    assert info["pattern"] == 1
    assert info["ring"] == 1 and info["ring_tiles"] == info["tiles"], info
    assert 1 <= info["max_copies"] <= 31 and info["stage_bytes"] <= 110 * 1024, info


def test_ring_tables_are_shared_between_interior_tiles():
    info = check(W.config3(side=64))
    # 256 tiles of a 64^3 grid, only a handful of distinct (boundary) row-pattern tables
    assert info["ring_table_words"] < 0.1 * info["tiles"] * 300, info


def test_padding_fill_keeps_bytes_and_result():
    w = W.config3(side=30)
    a = check(w)
    b = check(w, {"NPC_CSR_NOFILL": "1"})
    assert a["own_values"] == b["own_values"]  # the fill uses padding slots only


@pytest.mark.parametrize("env", [{"NPC_CSR_NOMIRROR": "1"}, {"NPC_CSR_NORING": "1"}, {"NPC_CSR_NOSTAGE": "1"}])
def test_layout_knobs(env):
    info = check(W.config3(side=30), env)
    if "NPC_CSR_NOMIRROR" in env:
        assert info["ring"] == 1
    else:
        assert info["ring"] == 0 and info["ring_tiles"] == 0  # rows summed from the CSR arrays


def test_unstructured_is_not_pattern_form():
    w = W.config4(n=12_000)  # kNN rows: > 256 distinct patterns per tile
    with pytest.raises(npc.NpcError) as e:
        npc.npc_pattern_check(w["rowptr"], w["colidx"], w["vals"], np.ones(w["n"]))
    assert e.value.code == 9  # NPC_ERR_UNSUPPORTED
