#!/usr/bin/env python
"""Short, representative slice of the bench step for ncu: build the operator of a config,
run the spectrum estimate and `--iters` PCG iterations (not to tolerance), then `--applies`
extra p_k(A) r applications.  Used only for profiling (never a bench value).

    python tools/profile_step.py --config 3 --k 50 --iters 3 --applies 2
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2208_01339_b200 as npc  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--side", type=int, default=None)
    ap.add_argument("--kind", default=None)
    ap.add_argument("--k", type=int, default=None)
    ap.add_argument("--iters", type=int, default=3)
    ap.add_argument("--applies", type=int, default=2)
    a = ap.parse_args()
    w = bench.make_workload(a.config, a.side)
    kind = a.kind or bench.op_kind(w, a.config)
    k = a.k if a.k is not None else w["k"]
    ctx = npc.npc_context_create(0)
    op = npc.create_from_workload(ctx, w, kind)
    b = torch.tensor(w["b"], device="cuda")
    lo, hi = npc.npc_estimate_spectrum(op, 20, None)
    poly = npc.npc_set_poly(op, k, lo, hi, 0.0)
    x = torch.zeros_like(b)
    st = npc.npc_pcg_solve(poly, op, b, x, w["tol"], a.iters, raise_on_error=False)
    z = torch.empty_like(b)
    for _ in range(a.applies):
        npc.npc_apply_poly(poly, b, z)
    torch.cuda.synchronize()
    print("profile_step ok", kind, "k", k, "iters", st["iters"], "launches", npc.npc_launch_count(),
          "z norm", float(np.linalg.norm(z.cpu().numpy())))


if __name__ == "__main__":
    main()
