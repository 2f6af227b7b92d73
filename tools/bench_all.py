#!/usr/bin/env python
"""Per-config table (all five BASELINE.json configs, full size, 1 GPU): p_k(A) v time and
achieved algorithmic GB/s of the fused degree kernels, operator applications/s, PCG
time-to-tol and iterations.  Writes one JSON line per (config, k) and, with --md, a markdown
table.  Not the driver's bench line (bench.py is); this is the §8 coverage evidence.

    python tools/bench_all.py [--configs 1,2,3,4,5] [--reps 10] [--md profiles/configs_r01.md]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2208_01339_b200 as npc  # noqa: E402

KS = {1: [10], 2: [30], 3: [20, 50, 100], 4: [60], 5: [10, 50, 100, 200], 6: [30]}


def run(cfg, reps, ctx, kinds=None):
    t0 = time.time()
    w = bench.make_workload(cfg, None)
    gen_s = time.time() - t0
    out = []
    for kind in kinds or [bench.op_kind(w, cfg)]:
        op = npc.create_from_workload(ctx, w, kind)
        b = torch.tensor(w["b"], device="cuda")
        M = bench.matrix_bytes(w, kind)                 # format-independent §8(d) bytes
        # CSR: what its stored format streams (coded ids: 9 B/nnz); the other operators are
        # reported against their §8(d) floor
        Mf = npc.npc_operator_matrix_bytes(op) if kind == "csr" else M
        V = 8 * w["n"]
        lo, hi = npc.npc_estimate_spectrum(op, 20, None)
        for k in KS[cfg]:
            poly = npc.npc_set_poly(op, k, lo, hi, 0.0)
            z = torch.empty_like(b)
            npc.npc_apply_poly(poly, b, z)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(reps):
                npc.npc_apply_poly(poly, b, z)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / reps
            gbs = bench.poly_bytes(M, V, k) / (ms * 1e-3) / 1e9
            gbs_f = bench.poly_bytes(Mf, V, k) / (ms * 1e-3) / 1e9
            x = torch.zeros_like(b)
            tts = []
            for rep in range(3 if cfg != 3 else 1):  # time-to-tol: median of 3 (config 3: ~20 s, once)
                x.zero_()
                torch.cuda.synchronize()
                t1 = time.perf_counter()
                lo2, hi2 = npc.npc_estimate_spectrum(op, 20, None)
                p2 = npc.npc_set_poly(op, k, lo2, hi2, 0.0)
                st = npc.npc_pcg_solve(p2, op, b, x, w["tol"], 50000, raise_on_error=False)
                torch.cuda.synchronize()
                tts.append(time.perf_counter() - t1)
                if rep < 2 and cfg != 3:
                    p2.close()
            tt = sorted(tts)[len(tts) // 2]
            sb = bench.solve_bytes(M, V, k, st["iters"], 20)
            # the roofline that bounds this operator: HBM, except an L2-resident stencil (L2
            # copy rate) and the Schur operator (random L2 sectors: 2 nnz(B) per application)
            l2p = bench.l2_peaks() or {}
            bound, frac_bound = "hbm", round(gbs_f / bench.hbm_peak()[0], 3)
            if kind == "stencil" and 4 * V <= 0.75 * 126e6 and l2p:
                bound, frac_bound = "l2 copy", round(gbs_f / l2p["l2_copy_rw_gbs"], 3)
            elif kind == "schur" and l2p:
                sec = 2.0 * int(w["browptr"][-1]) * k / (ms * 1e-3)
                bound, frac_bound = "l2 random sectors", round(sec / l2p["l2_random8B_sectors_per_s"], 3)
            row = dict(config=cfg, name=w["name"], operator=kind, n=w["n"], k=k, apply_ms=round(ms, 4),
                       apply_gbs=round(gbs, 1), apply_gbs_format=round(gbs_f, 1),
                       frac_measured=round(gbs_f / bench.hbm_peak()[0], 3), bound=bound, frac_bound=frac_bound,
                       applications_per_s=round(k / (ms * 1e-3), 1), pcg_status=st["status"], iters=st["iters"],
                       relres_true=st["relres_true"], time_to_tol_s=round(tt, 4),
                       solve_gbs=round(sb / tt / 1e9, 1), lmin=lo2, lmax=hi2, gen_s=round(gen_s, 1))
            print(json.dumps(row), flush=True)
            out.append(row)
            p2.close()
            poly.close()
        op.close()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="1,2,3,4,5")
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--md", default=None)
    ap.add_argument("--kinds", default=None, help="e.g. csr,sell to compare storages where applicable")
    a = ap.parse_args()
    ctx = npc.npc_context_create(0)
    rows = []
    for c in [int(x) for x in a.configs.split(",")]:
        kinds = a.kinds.split(",") if a.kinds and c in (1, 3, 4) else None
        rows += run(c, a.reps, ctx, kinds)
    if a.md:
        with open(a.md, "w") as f:
            f.write("| config | operator | n | k | p_k(A)v ms | GB/s (alg., §8(d) bytes) | GB/s (stored format) | "
                    "frac of measured HBM (format) | bound | frac of that bound | applications/s | "
                    "PCG iters | time-to-tol s | solve GB/s | true relres |\n"
                    "|---|---|---|---|---|---|---|---|---|---|---|---|---|---|---|\n")
            for r in rows:
                f.write(f"| {r['name']} | {r['operator']} | {r['n']} | {r['k']} | {r['apply_ms']} | {r['apply_gbs']} | "
                        f"{r['apply_gbs_format']} | "
                        f"{r['frac_measured']} | {r['bound']} | {r['frac_bound']} | {r['applications_per_s']} | "
                        f"{r['iters']} | {r['time_to_tol_s']} | "
                        f"{r['solve_gbs']} | {r['relres_true']:.2e} |\n")


if __name__ == "__main__":
    main()
