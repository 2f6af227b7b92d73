#!/usr/bin/env python
"""Wall time of each phase of one bench step (estimate, set_poly, solve) for a config; tuning
aid for latency-bound (small) configs.   python tools/phase_times.py --config 1 --reps 20"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2208_01339_b200 as npc  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=1)
    ap.add_argument("--side", type=int, default=None)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--distributed", action="store_true", help="1-rank NCCL context (multi-rank path)")
    ap.add_argument("--reuse-poly", action="store_true", help="one poly for all reps (PCG graph cached)")
    ap.add_argument("--k", type=int, default=None)
    a = ap.parse_args()
    w = bench.make_workload(a.config, a.side)
    kind = bench.op_kind(w, a.config)
    ctx = npc.npc_context_create(0, 1, 0, npc.npc_get_unique_id() if a.distributed else None)
    op, _, _ = bench.create_operator(npc, ctx, w, kind, 1, 0, a.config)
    b = torch.tensor(w["b"], device="cuda")
    x = torch.zeros_like(b)
    t = {"estimate": [], "set_poly": [], "solve": []}
    poly = None
    for rep in range(a.reps + 3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        lo, hi = npc.npc_estimate_spectrum(op, 20, None)
        t1 = time.perf_counter()
        if poly is None or not a.reuse_poly:
            poly = npc.npc_set_poly(op, a.k or w["k"], lo, hi, 0.0)
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        x.zero_()
        st = npc.npc_pcg_solve(poly, op, b, x, w["tol"], 20000)
        torch.cuda.synchronize()
        t3 = time.perf_counter()
        if not a.reuse_poly:
            poly.close()
        if rep >= 3:
            t["estimate"].append(t1 - t0)
            t["set_poly"].append(t2 - t1)
            t["solve"].append(t3 - t2)
    print(w["name"], kind, "iters", st["iters"],
          {k: f"{1e3 * np.median(v):.3f} ms" for k, v in t.items()})


if __name__ == "__main__":
    main()
