#!/usr/bin/env python
"""Phases of bench.py's e2e step (create, H2D, estimate, set_poly, solve, D2H, close) for a
config; tuning aid.   python tools/e2e_phases.py --config 3"""
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
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--reps", type=int, default=2)
    a = ap.parse_args()
    w = bench.make_workload(a.config, None)
    kind = bench.op_kind(w, a.config)
    ctx = npc.npc_context_create(0)
    b_pin = torch.from_numpy(np.ascontiguousarray(w["b"])).pin_memory()
    x_pin = torch.empty(w["n"], dtype=torch.float64).pin_memory()
    for rep in range(a.reps):
        t = {}
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        op = npc.create_from_workload(ctx, w, kind)
        torch.cuda.synchronize(); t["create"] = time.perf_counter() - t0; t0 = time.perf_counter()
        bd = b_pin.to("cuda", non_blocking=True)
        xd = torch.zeros(w["n"], dtype=torch.float64, device="cuda")
        torch.cuda.synchronize(); t["h2d"] = time.perf_counter() - t0; t0 = time.perf_counter()
        lo, hi = npc.npc_estimate_spectrum(op, 20, None)
        t["estimate"] = time.perf_counter() - t0; t0 = time.perf_counter()
        p = npc.npc_set_poly(op, w["k"], lo, hi, 0.0)
        torch.cuda.synchronize(); t["set_poly"] = time.perf_counter() - t0; t0 = time.perf_counter()
        st = npc.npc_pcg_solve(p, op, bd, xd, w["tol"], 20000)
        torch.cuda.synchronize(); t["solve"] = time.perf_counter() - t0; t0 = time.perf_counter()
        x_pin.copy_(xd, non_blocking=True)
        torch.cuda.synchronize(); t["d2h"] = time.perf_counter() - t0; t0 = time.perf_counter()
        p.close()
        op.close()
        t["close"] = time.perf_counter() - t0
        print(rep, st["iters"], {k: round(v, 3) for k, v in t.items()}, "total", round(sum(t.values()), 3), flush=True)


if __name__ == "__main__":
    main()
