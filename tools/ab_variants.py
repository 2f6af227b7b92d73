#!/usr/bin/env python
"""A/B timing of library build variants (tuning experiments; never a bench value).

    python tools/ab_variants.py --config 4 --side 2000000 --k 60 --libs a.so,b.so

Each variant library is loaded in a fresh subprocess (NPC_LIB_PATH) and times `reps`
applications of p_k(A) r with CUDA events; prints one JSON line per variant.
"""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import sys, json, numpy as np, torch
sys.path.insert(0, ROOT)
import bench, paper_2208_01339_b200 as npc
import os, pickle
import hashlib
_wh = hashlib.sha1(open(os.path.join(ROOT, "workloads", "__init__.py"), "rb").read()).hexdigest()[:12]
cache = f"/tmp/npc_ab_workload_{CFG}_{SIDE}_{_wh}.pkl"  # per box and generator version, shared by the variants
if os.path.exists(cache):
    w = pickle.load(open(cache, "rb"))
else:
    w = bench.make_workload(CFG, SIDE)
    pickle.dump(w, open(cache + ".tmp", "wb"), protocol=4)
    os.replace(cache + ".tmp", cache)
kind = KIND or bench.op_kind(w, CFG)
ctx = npc.npc_context_create(0)
op = npc.create_from_workload(ctx, w, kind)
if os.environ.get("AB_INTERVAL"):  # fixed interval (variants whose operator is wrong on purpose)
    lo, hi = (float(v) for v in os.environ["AB_INTERVAL"].split(":"))
else:
    lo, hi = npc.npc_estimate_spectrum(op, 20, None)
poly = npc.npc_set_poly(op, K, lo, hi, 0.0)
b = torch.tensor(w["b"], device="cuda"); z = torch.empty_like(b)
for _ in range(3): npc.npc_apply_poly(poly, b, z)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(REPS): npc.npc_apply_poly(poly, b, z)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / REPS
M, V = bench.matrix_bytes(w, kind), 8 * w["n"]
print(json.dumps(dict(lib=npc.LIB_PATH, ms=ms, gbs=bench.poly_bytes(M, V, K) / (ms * 1e-3) / 1e9,
                      znorm=float(torch.linalg.norm(z)))))
"""


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--side", type=int, default=None)
    ap.add_argument("--kind", default=None)
    ap.add_argument("--k", type=int, default=60)
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--libs", default="paper_2208_01339_b200/libnpc.so")
    ap.add_argument("--envs", default="", help="'|'-separated env variants, e.g. '|NPC_DFN_M=1'")
    a = ap.parse_args()
    code = CHILD.replace("ROOT", repr(ROOT)).replace("CFG", str(a.config)).replace("SIDE", repr(a.side)) \
        .replace("KIND", repr(a.kind)).replace("REPS", str(a.reps)).replace("K,", f"{a.k},") \
        .replace("(M, V, K)", f"(M, V, {a.k})")
    for lib in a.libs.split(","):
        for ev in a.envs.split("|"):
            env = dict(os.environ, NPC_LIB_PATH=os.path.abspath(lib))
            env.update(kv.split("=", 1) for kv in ev.split(",") if kv)
            r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
            print(ev or "-", r.stdout.strip() or r.stderr[-2000:], flush=True)


if __name__ == "__main__":
    main()
