"""CPU-only checks of libnpc: it builds for sm_100a, loads, exports every symbol include/npc.h
declares, and its host-side logic (coefficients, halo plans) is right.  No GPU compute."""
import os
import re

import numpy as np
import pytest

import oracle
import workloads as W

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def npc():
    from paper_2208_01339_b200 import build_lib
    build_lib.build()
    import paper_2208_01339_b200 as m
    m.lib()
    return m


def test_exports_every_declared_symbol(npc):
    hdr = open(os.path.join(ROOT, "include", "npc.h")).read()
    declared = set(re.findall(r"NPC_API\s+[\w\s\*]+?\b(npc_\w+)\s*\(", hdr))
    assert len(declared) >= 15
    lib = npc.lib()
    for name in sorted(declared):
        assert hasattr(lib, name), name
    # and the .so really is sm_100a code
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", npc.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_no_oracle_in_product():
    """The product path never imports or links the oracle (and vice versa)."""
    pkg = os.path.join(ROOT, "paper_2208_01339_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt and "npc_oracle" not in txt, f
    for f in os.listdir(os.path.join(ROOT, "oracle")):
        if f.endswith((".py", ".c")):
            lines = open(os.path.join(ROOT, "oracle", f)).read().splitlines()
            code = [ln for ln in lines if re.match(r"\s*(import|from|#include)\b", ln)]
            assert not any("paper_2208_01339_b200" in ln or "npc.h" in ln for ln in code), f


def test_version(npc):
    assert "sm_100a" in npc.npc_version()


@pytest.mark.parametrize("k,lmin,lmax,xi", [(1, 1.0, 3.0, 0.0), (10, 0.01, 8.0, 1e-3), (200, 1e-4, 12.0, 0.0),
                                            (63, 1.0, 1e5, 1e-4)])
def test_poly_coefficients_match_oracle_rho(npc, k, lmin, lmax, xi):
    tb, dl, sg, coef = npc.npc_poly_coefficients(k, lmin, lmax, xi)
    otb, odl, osg = oracle.cheb_params(lmin, lmax, xi)
    assert (tb, dl) == (otb, odl) and abs(sg - osg) <= 1e-15 * osg
    rho = oracle.cheb_rho(osg, k)
    # a_j = -2 rho_j/delta, b_j = 2 sigma rho_j, c_j = -rho_j rho_{j-1}, d_j = 2 rho_j/delta
    for j in range(1, k + 1):
        a, b, c, d = coef[j - 1]
        assert np.allclose([a, b, c, d], [-2 * rho[j] / odl, 2 * osg * rho[j], -rho[j] * rho[j - 1], 2 * rho[j] / odl],
                           rtol=1e-14, atol=0)


def test_fused_recurrence_equals_alg2_on_scalars(npc):
    """The fused per-degree form s_j = a A s_{j-1} + b s_{j-1} + c s_{j-2} + d r with the j=1,2
    folding used by the kernels reproduces Alg. 2 (the oracle) on a diagonal operator."""
    lam = np.linspace(0.05, 4.0, 37)
    for k in (0, 1, 2, 3, 17):
        tb, dl, sg, coef = npc.npc_poly_coefficients(k, 0.05, 4.0, 1e-3)
        r = np.ones_like(lam)
        if k == 0:
            s = r / tb
        else:
            sm2 = None
            sm1 = None
            for j in range(1, k + 1):
                a, b, c, d = coef[j - 1]
                if j == 1:
                    s = (a / tb) * lam * r + (b / tb + d) * r
                elif j == 2:
                    s = a * lam * sm1 + b * sm1 + (c / tb + d) * r
                else:
                    s = a * lam * sm1 + b * sm1 + c * sm2 + d * r
                sm2, sm1 = sm1, s
        op = oracle.Operator(dict(kind="csr", n=lam.size, rowptr=np.arange(lam.size + 1, dtype=np.int32),
                                  colidx=np.arange(lam.size, dtype=np.int32), vals=lam))
        ref = oracle.cheb_apply(op, k, 0.05, 4.0, 1e-3, r)
        assert np.allclose(s, ref, rtol=1e-12, atol=0)


def test_coefficient_errors(npc):
    with pytest.raises(npc.NpcError) as e:
        npc.npc_poly_coefficients(3, 2.0, 2.0, 0.0)
    assert e.value.name == "NPC_ERR_DEGENERATE_INTERVAL"
    with pytest.raises(npc.NpcError) as e:
        npc.npc_poly_coefficients(3, -1.0, 2.0, 0.0)
    assert e.value.name == "NPC_ERR_INVALID_ARGUMENT"


@pytest.mark.parametrize("nranks", [1, 2, 3, 4, 8])
def test_halo_plan_reproduces_column_sets(npc, nranks):
    w = W.config3(side=10, want_b=False)
    n = w["n"]
    starts = np.linspace(0, n, nranks + 1).astype(np.int64)
    for rank in range(nranks):
        r0, r1 = starts[rank], starts[rank + 1]
        rp = w["rowptr"][r0:r1 + 1] - w["rowptr"][r0]
        ci = w["colidx"][w["rowptr"][r0]:w["rowptr"][r1]]
        ids, counts = npc.npc_halo_plan(rp, ci, starts, rank)
        expect = np.unique(ci[(ci < r0) | (ci >= r1)])
        assert np.array_equal(ids, expect)
        owner = np.searchsorted(starts, expect, side="right") - 1
        assert np.array_equal(counts, np.bincount(owner, minlength=nranks))
        assert counts[rank] == 0
        if nranks > 1:  # 7-point z-slabs: only the two neighbouring planes are ghosts
            assert len(ids) <= 2 * 100


def test_halo_plan_rejects_bad_input(npc):
    with pytest.raises(npc.NpcError):
        npc.npc_halo_plan(np.array([0, 1], dtype=np.int32), np.array([5], dtype=np.int32),
                          np.array([0, 1, 2], dtype=np.int64), 0)  # column out of range


def test_pcg_stats_layout_matches_header(npc):
    """The binding's npc_pcg_stats mirrors include/npc.h field by field (ABI drift guard)."""
    hdr = open(os.path.join(ROOT, "include", "npc.h")).read()
    end = hdr.index("} npc_pcg_stats;")
    body = hdr[hdr.rindex("typedef struct {", 0, end) + len("typedef struct {"):end]
    body = re.sub(r"/\*.*?\*/", "", body, flags=re.S)
    names = re.findall(r"\b(\w+)\s*;", body)
    assert names == [f[0] for f in npc.PcgStats._fields_], (names, npc.PcgStats._fields_)
    assert "setup_seconds" in names and "solve_seconds" in names


def test_last_error_thread_and_null_context(npc):
    """A failing host-only call records its message for npc_last_error(NULL) (the calling
    thread); a context-less failure never touches a context's message."""
    with pytest.raises(npc.NpcError) as e:
        npc.npc_poly_coefficients(5, 2.0, 2.0, 0.0)
    assert e.value.name == "NPC_ERR_DEGENERATE_INTERVAL"
    msg = npc.npc_last_error(None)
    assert msg and msg in str(e.value)
    import threading
    other = []
    t = threading.Thread(target=lambda: other.append(npc.npc_last_error(None)))
    t.start()
    t.join()
    assert other == [""]  # thread-local


def test_estimate_spectrum_signature_has_seed(npc):
    hdr = open(os.path.join(ROOT, "include", "npc.h")).read()
    decl = re.search(r"npc_estimate_spectrum\((.*?)\);", hdr, re.S).group(1)
    assert "unsigned long long seed" in decl
    assert "NPC_DEFAULT_SEED 0x5EED" in hdr and npc.NPC_DEFAULT_SEED == 0x5EED == W.LANCZOS_SEED
