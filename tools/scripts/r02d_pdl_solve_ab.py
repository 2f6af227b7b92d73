import os, sys, time
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import torch, numpy as np
import bench, paper_2208_01339_b200 as npc
w = bench.make_workload(2, None)
ctx = npc.npc_context_create(0)
ref = None
for env in ("", "NPC_ST_PDL", "", "NPC_ST_PDL"):
    if env: os.environ[env] = "1"
    op, _, _ = bench.create_operator(npc, ctx, w, "stencil", 1, 0, 2)
    b = torch.tensor(w["b"], device="cuda")
    for rep in range(5):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        lo, hi = npc.npc_estimate_spectrum(op, 20, None)
        poly = npc.npc_set_poly(op, 30, lo, hi, 0.0)
        torch.cuda.synchronize(); t1 = time.perf_counter()
        x = torch.zeros_like(b)
        st = npc.npc_pcg_solve(poly, op, b, x, 1e-10, 5000)
        torch.cuda.synchronize(); t2 = time.perf_counter()
        if ref is None: ref = x.clone()
        print(env or "default", rep, "setup %.2f ms solve %.2f ms iters %d (lib solve_seconds %.2f ms) same bits as first solve: %s" % (1e3*(t1-t0), 1e3*(t2-t1), st["iters"], 1e3*st["solve_seconds"], bool(torch.equal(x, ref))))
    os.environ.pop(env, None) if env else None
