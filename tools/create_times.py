#!/usr/bin/env python
"""Wall time of npc_create_operator per config (host conversion + uploads).
    python tools/create_times.py --configs 3,4,5,6"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2208_01339_b200 as npc  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="3,4,5,6")
    a = ap.parse_args()
    ctx = npc.npc_context_create(0)
    for c in [int(x) for x in a.configs.split(",")]:
        w = bench.make_workload(c, None)
        kind = bench.op_kind(w, c)
        ts = []
        for _ in range(2):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            op = npc.create_from_workload(ctx, w, kind)
            torch.cuda.synchronize()
            ts.append(time.perf_counter() - t0)
            op.close()
        print(f"config {c} {kind}: create {min(ts):.3f} s", flush=True)


if __name__ == "__main__":
    main()
