import os, sys, time
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import torch, numpy as np
import bench, paper_2208_01339_b200 as npc
ctx = npc.npc_context_create(0)
for cfg, side, kind, k in ((2, None, "stencil", 30), (3, 128, "csr", 50)):
    w = bench.make_workload(cfg, side)
    op, _, _ = bench.create_operator(npc, ctx, w, kind, 1, 0, cfg)
    b = torch.tensor(w["b"], device="cuda")
    for rep in range(6):
        lo, hi = npc.npc_estimate_spectrum(op, 20, None)
        poly = npc.npc_set_poly(op, k, lo, hi, 0.0)
        x = torch.zeros_like(b)
        torch.cuda.synchronize(); t1 = time.perf_counter()
        st = npc.npc_pcg_solve(poly, op, b, x, w["tol"], 20000)
        torch.cuda.synchronize(); t2 = time.perf_counter()
        print(os.environ.get("NPC_LIB_PATH", "default").split("/")[-1], "config", cfg, side or "", "rep", rep, "solve %.3f ms iters %d relres %.2e" % (1e3*(t2-t1), st["iters"], st["relres_true"]))
