#!/usr/bin/env python
"""xi and spectrum-estimate sweep (DESIGN reading A12): PCG time-to-tolerance
and iterations of every BASELINE config for xi in {0, 1e-4, 1e-3, 1e-2} (Eq. thetamod,
PAPER.md:325-333) and Lanczos steps m in {20, 50, 100}.

Time-to-tol = npc_estimate_spectrum(m) + npc_set_poly + npc_pcg_solve (x0 = 0), median of
`--reps` solves, CUDA events on the library stream, operator created before (setup).

    python tools/xi_sweep.py --configs 1,2,3,4 --md profiles/r02_xi_sweep.md --jsonl profiles/r02_xi_sweep.jsonl
"""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2208_01339_b200 as npc  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="1,2,3,4")
    ap.add_argument("--xis", default="0,1e-4,1e-3,1e-2")
    ap.add_argument("--steps", default="20,50,100")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--side", type=int, default=None)
    ap.add_argument("--md", default=None)
    ap.add_argument("--jsonl", default=None)
    a = ap.parse_args()
    xis = [float(v) for v in a.xis.split(",")]
    msteps = [int(v) for v in a.steps.split(",")]
    ctx = npc.npc_context_create(0)
    stream = torch.cuda.current_stream()
    rows = []
    for cfg in [int(c) for c in a.configs.split(",")]:
        w = bench.make_workload(cfg, a.side if cfg in (2, 3) else None)
        kind = bench.op_kind(w, cfg)
        k = w["k"]
        op = npc.create_from_workload(ctx, w, kind)
        b = torch.tensor(w["b"], device="cuda")
        x = torch.zeros_like(b)
        for m in msteps:
            for xi in xis:
                ts, st = [], None
                for _ in range(a.reps):
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    torch.cuda.synchronize()
                    e0.record(stream)
                    lo, hi = npc.npc_estimate_spectrum(op, m, None)
                    poly = npc.npc_set_poly(op, k, lo, hi, xi)
                    x.zero_()
                    st = npc.npc_pcg_solve(poly, op, b, x, w["tol"], 20000, raise_on_error=False)
                    e1.record(stream)
                    torch.cuda.synchronize()
                    poly.close()
                    ts.append(e0.elapsed_time(e1))
                row = dict(config=cfg, workload=w["name"], kind=kind, k=k, lanczos_steps=m, xi=xi, lmin=lo, lmax=hi,
                           iters=st["iters"], converged=st["converged"], status=st["status"],
                           relres_true=st["relres_true"], time_to_tol_ms=round(statistics.median(ts), 3))
                rows.append(row)
                print(json.dumps(row), flush=True)
        op.close()
    if a.jsonl:
        with open(a.jsonl, "w") as f:
            for r in rows:
                f.write(json.dumps(r) + "\n")
    if a.md:
        with open(a.md, "w") as f:
            f.write("# xi / Lanczos-steps sweep (one B200; `tools/xi_sweep.py`)\n\n")
            f.write("PCG time-to-tol = estimate(m) + set_poly + solve, median of %d, CUDA events. "
                    "Best xi per (config, m) in bold.\n\n" % a.reps)
            f.write("| config | k | m | " + " | ".join(f"xi={x:g}: iters / ms" for x in xis) + " |\n")
            f.write("|---|---|---|" + "---|" * len(xis) + "\n")
            for cfg in sorted({r["config"] for r in rows}):
                for m in msteps:
                    sel = [r for r in rows if r["config"] == cfg and r["lanczos_steps"] == m]
                    if not sel:
                        continue
                    best = min((r for r in sel if r["converged"]), key=lambda r: r["time_to_tol_ms"], default=None)
                    cells = []
                    for xi in xis:
                        r = next(r for r in sel if r["xi"] == xi)
                        c = f"{r['iters']} / {r['time_to_tol_ms']:.1f}" + ("" if r["converged"] else " (no conv)")
                        cells.append(f"**{c}**" if best is not None and r is best else c)
                    f.write(f"| {cfg} ({sel[0]['workload']}) | {sel[0]['k']} | {m} | " + " | ".join(cells) + " |\n")


if __name__ == "__main__":
    main()
