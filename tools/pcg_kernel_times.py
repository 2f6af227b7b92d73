#!/usr/bin/env python
"""Per-kernel device times inside a short PCG solve (maxit iterations, not to tolerance), from
CUPTI activity records via torch.profiler: which kernels the iteration spends its time in,
beside the degree steps (A.u with the delta partial, the update, the reductions).  Tuning aid
only; never a bench value.

    python tools/pcg_kernel_times.py --config 3 --k 50 --maxit 24
"""
import argparse
import collections
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2208_01339_b200 as npc  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--side", type=int, default=None)
    ap.add_argument("--kind", default=None)
    ap.add_argument("--k", type=int, default=50)
    ap.add_argument("--maxit", type=int, default=24)
    a = ap.parse_args()
    w = bench.make_workload(a.config, a.side)
    kind = a.kind or bench.op_kind(w, a.config)
    ctx = npc.npc_context_create(0)
    op, _, _ = bench.create_operator(npc, ctx, w, kind, 1, 0, a.config)
    lo, hi = npc.npc_estimate_spectrum(op, 20, None)
    poly = npc.npc_set_poly(op, a.k, lo, hi, 0.0)
    b = torch.tensor(w["b"], device="cuda")
    x = torch.zeros_like(b)
    npc.npc_pcg_solve(poly, op, b, x, 1e-30, a.maxit, raise_on_error=False)
    torch.cuda.synchronize()
    x.zero_()
    with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
        npc.npc_pcg_solve(poly, op, b, x, 1e-30, a.maxit, raise_on_error=False)
        torch.cuda.synchronize()
    tot = collections.defaultdict(lambda: [0, 0.0])
    for e in prof.events():
        if e.device_type == torch.autograd.DeviceType.CUDA:
            t = tot[e.name[:110]]
            t[0] += 1
            t[1] += e.device_time_total if hasattr(e, "device_time_total") else e.cuda_time_total
    allus = sum(v[1] for v in tot.values())
    for name, (cnt, us) in sorted(tot.items(), key=lambda kv: -kv[1][1]):
        print(f"{us / cnt:10.1f} us x {cnt:5d}  {100 * us / allus:5.1f}%  {name}")


if __name__ == "__main__":
    main()
