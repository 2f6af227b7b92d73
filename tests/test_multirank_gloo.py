"""Multi-rank host logic on CPU (gloo, world_size 2 and 4): the row-block partition, the
library's halo plan (npc_halo_plan, the same host code npc_create_operator runs per rank),
the ghost-id exchange that turns recv lists into send lists, and a distributed operator
application assembled from the plan equal the global oracle product.  The NCCL data path
itself needs GPUs (one per rank) and is not exercised here."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import workloads as W

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, ws, port, case, results):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=ws)
        import sys
        sys.path.insert(0, ROOT)
        import bench
        import paper_2208_01339_b200 as npc
        w = W.config3(side=12) if case == "c3" else W.config4(n=4000)
        n = w["n"]
        r0, r1, _ = bench.partition_rows(w, 3 if case == "c3" else 4, ws, rank)
        starts = [None] * ws
        dist.all_gather_object(starts, (r0, r1))
        row_starts = np.array([s[0] for s in starts] + [n], dtype=np.int64)
        assert all(starts[i][1] == starts[i + 1][0] for i in range(ws - 1))
        rp = w["rowptr"][r0:r1 + 1]
        rowptr = (rp - rp[0]).astype(np.int32)
        colidx = w["colidx"][rp[0]:rp[-1]]
        vals = w["vals"][rp[0]:rp[-1]]
        ghost_ids, recv_counts = npc.npc_halo_plan(rowptr, colidx, row_starts, rank)
        # exchange ghost id lists with the owners (what npc_create_operator does over NCCL)
        recv_off = np.concatenate([[0], np.cumsum(recv_counts)])
        want = [ghost_ids[recv_off[q]:recv_off[q + 1]].tolist() for q in range(ws)]
        all_want = [None] * ws
        dist.all_gather_object(all_want, want)
        send_idx = {q: np.array(all_want[q][rank], dtype=np.int64) - r0 for q in range(ws) if q != rank}
        for q, idx in send_idx.items():
            assert np.all((idx >= 0) & (idx < r1 - r0))
        # distributed y = A x: owned x + ghosts received through the plan
        x_glob = np.random.default_rng(42).standard_normal(n)
        x_own = x_glob[r0:r1]
        ghosts = np.zeros(len(ghost_ids))
        reqs = []
        for q in range(ws):
            if q == rank:
                continue
            if len(send_idx[q]):
                reqs.append(dist.isend(torch.from_numpy(np.ascontiguousarray(x_own[send_idx[q]])), q))
        for q in range(ws):
            if q == rank or recv_counts[q] == 0:
                continue
            buf = torch.zeros(int(recv_counts[q]), dtype=torch.float64)
            dist.recv(buf, q)
            ghosts[recv_off[q]:recv_off[q + 1]] = buf.numpy()
        for rq in reqs:
            rq.wait()
        # local columns: owned -> c - r0, ghost -> n_local + position in the sorted ghost list
        local = np.where((colidx >= r0) & (colidx < r1), colidx - r0,
                         (r1 - r0) + np.searchsorted(ghost_ids, colidx))
        xl = np.concatenate([x_own, ghosts])
        y = np.array([vals[rowptr[i]:rowptr[i + 1]] @ xl[local[rowptr[i]:rowptr[i + 1]]] for i in range(r1 - r0)])
        ref = oracle.Operator(w).apply(x_glob)[r0:r1]
        ok = np.allclose(y, ref, rtol=1e-13, atol=1e-13)
        # the interior/boundary split: rows with no ghost column can run before the halo arrives
        boundary = np.array([np.any(local[rowptr[i]:rowptr[i + 1]] >= r1 - r0) for i in range(r1 - r0)])
        if case == "c3" and ws > 1:
            plane = 12 * 12
            nb = boundary.sum()
            ok = ok and nb <= 2 * plane
        dist.barrier()
        results.put((rank, bool(ok), len(ghost_ids)))
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover
        results.put((rank, False, repr(e)))


@pytest.mark.parametrize("case", ["c3", "c4"])
@pytest.mark.parametrize("ws", [2, 4])
def test_distributed_spmv_from_halo_plan(case, ws):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, ws, port, case, q)) for r in range(ws)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(ws)]
    for p in procs:
        p.join(timeout=60)
    assert all(ok for _, ok, _ in res), res
    assert all(isinstance(g, int) and g > 0 for _, _, g in res), res
