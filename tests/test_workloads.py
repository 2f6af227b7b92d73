"""Shape/structure checks of the seeded synthetic inputs (workloads/), CPU only."""
import numpy as np
import scipy.sparse as sp

import workloads as W


def _csr(w):
    return sp.csr_matrix((w["vals"], w["colidx"], w["rowptr"]), shape=(w["n"], w["n"]))


def test_config1_shape():
    w = W.config1()
    assert w["n"] == 4096 and w["rowptr"][-1] == 20224
    A = _csr(w)
    assert abs(A - A.T).max() == 0
    assert np.all(np.diff(w["colidx"][w["rowptr"][0]:w["rowptr"][1]]) > 0)
    assert w["b"].min() >= -1 and w["b"].max() <= 1


def test_config1_deterministic():
    assert np.array_equal(W.config1()["b"], W.config1()["b"])


def test_config3_structure_small():
    w = W.config3(side=10)
    A = _csr(w)
    n = w["n"]
    assert abs(A - A.T).max() == 0
    assert w["rowptr"][-1] == 7 * n - 6 * 10 * 10
    # diagonal dominance margin of each row = its boundary-face coefficients = b (x* = 1)
    d = A.diagonal()
    off = np.asarray(abs(A).sum(axis=1)).ravel() - d
    assert np.allclose(d - off, w["b"], rtol=1e-12, atol=1e-12)
    assert (w["b"] > 0).sum() == n - 8 ** 3
    for i in range(0, n, 97):
        cols = w["colidx"][w["rowptr"][i]:w["rowptr"][i + 1]]
        assert np.all(np.diff(cols) > 0)


def test_config3_full_size_counts():
    """nnz formula of the full 256^3 grid (not generated here: too big for the CPU suite)."""
    N = 256
    assert 7 * N ** 3 - 6 * N * N == 117_047_296


def test_config4_surrogate():
    w = W.config4(n=20_000)
    A = _csr(w)
    assert abs(A - A.T).max() < 1e-15
    assert np.array_equal(np.sort(w["perm"]), np.arange(w["n"]))
    deg = np.diff(w["rowptr"]) - 1
    assert deg.min() >= 16 and deg.max() <= 40
    assert np.allclose(np.asarray(A.sum(axis=1)).ravel(), 1e-3)  # L 1 = 0, + 1e-3 I


def test_config5_surrogate():
    w = W.config5(n=5000)
    lens = np.diff(w["browptr"])
    assert w["nb"] == 15000 and lens.min() == 2 and lens.max() == 4
    for q in range(0, w["nb"], 7):
        c = w["bcolidx"][w["browptr"][q]:w["browptr"][q + 1]]
        assert np.all(np.diff(c) > 0)
    assert w["d"].min() >= 1 and w["d"].max() <= 100 and 1 <= w["c"].min() and w["c"].max() <= 2


def test_dfn_generator_structure():
    """Structure of the synthetic DFN system (PAPER.md:668-688 bullets; SPEC generate_synthetic)."""
    w = W.dfn(40, seed=7)
    w2 = W.dfn(40, seed=7)
    for key in ("A", "Gh", "C", "B", "Gu"):  # deterministic
        for a, b in zip(w[key], w2[key]):
            assert np.array_equal(a, b)
    hb = w["hblk"]
    blk = np.searchsorted(hb, np.arange(w["nh"]), side="right") - 1
    for key in ("A", "Gh"):  # block-diagonal
        rp, ci, _ = w[key]
        rows = np.repeat(np.arange(w["nh"]), np.diff(rp))
        assert np.array_equal(blk[rows], blk[ci])
    rp, ci, cv = w["C"]  # C fracture-local: every column in one fracture block
    rows = np.repeat(np.arange(w["nh"]), np.diff(rp))
    for j in np.unique(ci)[:200]:
        assert len(set(blk[rows[ci == j]])) == 1
    brp, bci, bv = w["B"]
    assert brp[-1] >= rp[-1] and np.all(cv >= 0) and np.all(bv >= 0)
    # G^h symmetric with zero row sums (SPSD, rank-deficient); G^u symmetric tridiagonal per trace
    import scipy.sparse as sp
    Gh = sp.csr_matrix((w["Gh"][2], w["Gh"][1], w["Gh"][0]), shape=(w["nh"], w["nh"]))
    assert abs(Gh - Gh.T).max() == 0 and np.allclose(np.asarray(Gh.sum(axis=1)).ravel(), 0.0)
    Gu = sp.csr_matrix((w["Gu"][2], w["Gu"][1], w["Gu"][0]), shape=(w["n"], w["n"]))
    assert abs(Gu - Gu.T).max() == 0 and np.all(Gu.diagonal() == 2.0)
    assert w["alpha"] > 0 and w["b"].shape == (w["n"],)


def test_dfn_owner_order_is_a_symmetric_permutation():
    """dfn_owner_order renumbers u so each fracture's C columns are contiguous (the DSMat layout
    the multi-rank DFN operator needs); S_u is permuted symmetrically (checked on G^u, C, B, b)."""
    w = W.dfn(25, seed=9)
    w2 = W.dfn_owner_order(w)
    nh, nu = w["nh"], w["n"]
    hb = np.asarray(w["hblk"])
    blk = np.searchsorted(hb, np.arange(nh), side="right") - 1
    crp, cci, _ = w2["C"]
    rows = np.repeat(np.arange(nh), np.diff(crp))
    uoff = w2["uoff"]
    assert uoff[0] == 0 and uoff[-1] <= nu and np.all(np.diff(uoff) >= 0)
    assert np.all((uoff[blk[rows]] <= cci) & (cci < uoff[blk[rows] + 1]))
    # the same multiset of entries, columns permuted consistently with b
    import scipy.sparse as sp
    C1 = sp.csr_matrix((w["C"][2], w["C"][1], w["C"][0]), shape=(nh, nu))
    C2 = sp.csr_matrix((w2["C"][2], w2["C"][1], w2["C"][0]), shape=(nh, nu))
    G1 = sp.csr_matrix((w["Gu"][2], w["Gu"][1], w["Gu"][0]), shape=(nu, nu))
    G2 = sp.csr_matrix((w2["Gu"][2], w2["Gu"][1], w2["Gu"][0]), shape=(nu, nu))
    assert abs(G1.sum() - G2.sum()) < 1e-9 and abs(C1.sum() - C2.sum()) < 1e-9
    assert np.isclose(np.sort(w["b"]), np.sort(w2["b"])).all()
