"""CPU checks of bench.py's host logic (no GPU): the §8(d) byte model, the row partition of
the multi-GPU runs, the cached oracle golden lookup and the L2 / HBM peak files."""
import json
import os

import numpy as np
import pytest

import bench
import workloads as W

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_poly_bytes_counts_the_streams():
    """p_k(A) r: degree 1 reads r and writes s_1; degree 2 reads s_1, r and writes;
    degrees >= 3 read s_{j-1}, s_{j-2}, r and write, the matrix each degree."""
    M, V = 1000.0, 10.0
    assert bench.poly_bytes(M, V, 0) == 2 * V
    assert bench.poly_bytes(M, V, 1) == M + 2 * V
    assert bench.poly_bytes(M, V, 2) == 2 * M + 5 * V
    for k in (3, 10, 50):
        assert bench.poly_bytes(M, V, k) == k * M + 5 * V + (k - 2) * 4 * V
    # PCG step = iters x (p_k + A u + 10-stream update) + Lanczos + setup + final residual
    it, k, m = 7, 5, 20
    want = it * (bench.poly_bytes(M, V, k) + M + 2 * V + 10 * V) + m * (M + 9 * V) + 6 * V + M + 3 * V
    assert bench.solve_bytes(M, V, k, it, m) == want


def test_config3_byte_model_matches_survey():
    """Config 3 at 256^3: 117,047,296 nonzeros, 2,008.5 MB per degree."""
    w = W.config3(side=32)
    nnz = int(w["rowptr"][-1])
    assert bench.matrix_bytes(w, "csr") == nnz * 12 + (w["n"] + 1) * 4
    n = 256 ** 3
    nnz256 = 7 * n - 6 * 256 * 256  # 7-point rows minus the missing boundary neighbours
    assert nnz256 == 117_047_296
    per_degree = nnz256 * 12 + (n + 1) * 4 + 4 * 8 * n
    assert abs(per_degree / 1e6 - 2008.5) < 0.1


@pytest.mark.parametrize("ws", [1, 2, 3, 8])
def test_partition_rows_covers_the_grid_in_z_slabs(ws):
    w = W.config3(side=24)
    starts = [bench.partition_rows(w, 3, ws, r) for r in range(ws)]
    assert starts[0][0] == 0 and starts[-1][1] == w["n"]
    plane = 24 * 24
    for (a0, a1, zs), (b0, _, _) in zip(starts, starts[1:] + [(w["n"], None, None)]):
        assert a1 == b0 and a0 % plane == 0 and a1 % plane == 0  # whole z-planes, contiguous
        assert zs[1] == (a1 - a0) // plane


def test_oracle_golden_lookup():
    """The cached full-size oracle solve is found for its workload and k only."""
    g = bench.oracle_golden({"n": 256 ** 3, "name": "config3_256^3"}, 50, 0.0)
    if g is None:
        pytest.skip("golden not written")
    raw = json.load(open(os.path.join(ROOT, "tests", "golden", "config3_256_pcg_k50.json")))
    assert g["iters"] == raw["iters"] and g["seconds"] == round(raw["seconds_time_to_tol"], 1)
    assert bench.oracle_golden({"n": 256 ** 3, "name": "config3_256^3"}, 50, 1e-3) is None
    assert bench.oracle_golden({"n": 128 ** 3, "name": "config2_128^3"}, 30, 0.0) is None


def test_peaks_files():
    l2 = bench.l2_peaks()
    assert l2 is not None and l2["l2_random8B_sectors_per_s"] > 1e11 and l2["l2_copy_rw_gbs"] > 5000
    peak, src = bench.hbm_peak()
    assert 5000 < peak < 9000 and ("measured" in src or "fallback" in src)
