#!/usr/bin/env python
"""Summarise a bench.py JSON line from stdin (tuning runs)."""
import json
import sys

for raw in sys.stdin:
    raw = raw.strip()
    if not raw.startswith("{"):
        continue
    line = json.loads(raw)
    rf = line.get("roofline") or {}
    pc = line.get("pcg") or {}
    out = {k: line.get(k) for k in ("value", "ms_per_step", "step_ms", "parallelism", "clocks")}
    out.update(iters=pc.get("iters"), apps=pc.get("op_applications"), red=pc.get("reductions"), frac=rf.get("frac"))
    br = rf.get("step_breakdown") or {}
    if br:
        out["breakdown_ms"] = {k: v["ms"] for k, v in br.items()}
    print(json.dumps(out), flush=True)
