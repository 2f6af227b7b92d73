import sys, time, json
sys.path.insert(0, '/root/repo')
import numpy as np, torch, bench, paper_2208_01339_b200 as npc
import os
CFG = int(os.environ.get("EXP_CFG", "3")); w = bench.make_workload(CFG, None); kind = bench.op_kind(w, CFG); k = w["k"]
ctx = npc.npc_context_create(0)
op = npc.create_from_workload(ctx, w, kind)
b = torch.tensor(w['b'], device='cuda'); x = torch.zeros_like(b); z = torch.empty_like(b)
lo, hi = npc.npc_estimate_spectrum(op, 20, None)
poly = npc.npc_set_poly(op, k, lo, hi, 0.0)
M = bench.matrix_bytes(w, kind); V = 8 * w['n']
def iso(tag, reps=10):
    npc.npc_apply_poly(poly, b, z); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): npc.npc_apply_poly(poly, b, z)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(tag, 'isolated poly ms', round(ms, 3), 'GB/s', round(bench.poly_bytes(M, V, k) / ms / 1e6, 1), flush=True)
def pcg(tag, timing):
    npc.npc_context_set_timing(ctx, timing); npc.npc_context_get_timing(ctx)
    x.zero_(); t0 = time.perf_counter()
    st = npc.npc_pcg_solve(poly, op, b, x, 1e-8, 20000); torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    tm = npc.npc_context_get_timing(ctx); npc.npc_context_set_timing(ctx, False)
    per = tm['degree'][0] / max(tm['degree'][1] / k, 1) if timing else None
    print(tag, 'pcg s', round(dt, 3), 'iters', st['iters'], 'per-poly ms in step', per and round(per, 3),
          'GB/s', per and round(bench.poly_bytes(M, V, k) / per / 1e6, 1), flush=True)
iso('cold')
pcg('pcg1', True)
iso('hot')
pcg('pcg2-notiming', False)
iso('hot2')
pcg('pcg3', True)
