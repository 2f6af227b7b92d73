import sys, numpy as np, torch, time
sys.path.insert(0, '/root/repo')
import oracle, workloads as W, paper_2208_01339_b200 as npc
ctx = npc.npc_context_create(0)
for side in [64, 128]:
    w = W.config3(side=side)
    orc = oracle.Operator(w)
    for kind in ['csr']:
        op = npc.create_from_workload(ctx, w, kind)
        b = torch.tensor(w['b'], device='cuda')
        ex = npc.npc_estimate_spectrum_ex(op, 20, None)
        lo, hi = npc.npc_estimate_spectrum(op, 20, None)
        for k in [20, 50, 100]:
            poly = npc.npc_set_poly(op, k, lo, hi, 0.0)
            x = torch.zeros_like(b)
            st = npc.npc_pcg_solve(poly, op, b, x, 1e-8, 20000, history=True, raise_on_error=False)
            h = st.pop('history')
            print(side, kind, k, ex, st, flush=True)
            if side <= 64:
                t = time.time()
                _, so = oracle.pcg(orc, w['b'], k, lo, hi, 0.0, tol=1e-8, maxit=20000)
                print('   oracle iters', so['iters'], 'oracle s', time.time() - t, flush=True)
