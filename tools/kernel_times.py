#!/usr/bin/env python
"""Per-kernel device times of p_k(A) r in a normal (non-ncu) run, from CUPTI activity records
via torch.profiler: warm caches, back-to-back launches, real clocks.  Tuning aid only.

    python tools/kernel_times.py --config 5 --k 10 --reps 5
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
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--side", type=int, default=None)
    ap.add_argument("--kind", default=None)
    ap.add_argument("--k", type=int, default=10)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--distributed", action="store_true", help="1-rank NCCL context (multi-rank path)")
    ap.add_argument("--interval", default=None, help="lo,hi instead of the Lanczos estimate (A/B of broken variants)")
    a = ap.parse_args()
    w = bench.make_workload(a.config, a.side)
    kind = a.kind or bench.op_kind(w, a.config)
    ctx = npc.npc_context_create(0, 1, 0, npc.npc_get_unique_id() if a.distributed else None)
    op, _, _ = bench.create_operator(npc, ctx, w, kind, 1, 0, a.config)
    lo, hi = (map(float, a.interval.split(","))) if a.interval else npc.npc_estimate_spectrum(op, 20, None)
    poly = npc.npc_set_poly(op, a.k, lo, hi, 0.0)
    b = torch.tensor(w["b"], device="cuda")
    z = torch.empty_like(b)
    for _ in range(3):
        npc.npc_apply_poly(poly, b, z)
    torch.cuda.synchronize()
    with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
        for _ in range(a.reps):
            npc.npc_apply_poly(poly, b, z)
        torch.cuda.synchronize()
    tot = collections.defaultdict(lambda: [0, 0.0])
    for e in prof.events():
        if e.device_type == torch.autograd.DeviceType.CUDA:
            t = tot[e.name[:70]]
            t[0] += 1
            t[1] += e.device_time_total if hasattr(e, "device_time_total") else e.cuda_time_total
    allus = sum(v[1] for v in tot.values())
    for name, (cnt, us) in sorted(tot.items(), key=lambda kv: -kv[1][1]):
        print(f"{us / cnt:10.1f} us x {cnt:5d}  {100 * us / allus:5.1f}%  {name}")


if __name__ == "__main__":
    main()
