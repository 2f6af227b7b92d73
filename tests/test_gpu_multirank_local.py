"""Multi-rank path on ONE B200: ranks are host threads sharing the GPU through the local
thread-group transport (npc_context_create_local).  Everything but the NCCL calls runs as in
the one-process-per-GPU deployment: the collective operator creation (row-start allgather,
ghost discovery, id exchange -> send lists), interior/boundary tile lists and dot-partial
offsets, the per-application halo, the distributed Lanczos and the single-reduction PCG with
its one-iteration-late convergence test.  Results are compared with the CPU oracle.
No rank ever waits on another on the device (host barriers after stream syncs only)."""
import threading

import numpy as np
import pytest

import oracle
import workloads as W

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import bench  # noqa: E402
import paper_2208_01339_b200 as npc  # noqa: E402

_group_id = [0]


def run_ranks(ws, fn, timeout=240):
    """Run fn(rank, ctx) on ws threads; return the per-rank results (re-raise failures)."""
    _group_id[0] += 1
    group = f"test-{_group_id[0]}"
    out, err = [None] * ws, [None] * ws

    def body(rank):
        ctx = None
        try:
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                ctx = npc.npc_context_create_local(0, ws, rank, group, s)
                out[rank] = fn(rank, ctx, s)
                s.synchronize()
        except BaseException as e:  # noqa: BLE001
            err[rank] = e
            if ctx is not None:
                ctx.close()  # aborts the group: peers leave their barriers with an error

    th = [threading.Thread(target=body, args=(r,), daemon=True) for r in range(ws)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout)
    assert not any(t.is_alive() for t in th), "a rank hung"
    for e in err:
        if e is not None:
            raise e
    return out


CASES = [("c3", "csr", 2), ("c3", "csr", 4), ("c3", "sell", 3), ("c2", "stencil", 2), ("c2", "stencil", 4),
         ("c4", "sell", 2), ("c4", "csr", 4), ("c5", "schur", 2), ("c5", "schur", 3), ("c6", "dfn", 2),
         ("c6", "dfn", 3)]
WL = {"c3": lambda: W.config3(side=24), "c2": lambda: W.config2(side=20), "c4": lambda: W.config4(n=20_000),
      "c5": lambda: W.config5(n=20_011), "c6": lambda: W.dfn_owner_order(W.dfn(61, seed=7))}
CFG = {"c3": 3, "c2": 2, "c4": 4, "c5": 5, "c6": 6}


@pytest.fixture(scope="module")
def wl():
    cache = {}

    def get(name):
        if name not in cache:
            cache[name] = WL[name]()
        return cache[name]
    return get


def run_nccl_one_rank(ws, fn):
    """One rank over a real 1-rank NCCL communicator: the multi-rank path with NCCL calls
    (allreduce / allgather / reduce-scatter, captured into the PCG graphs) on the B200."""
    assert ws == 1
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        ctx = npc.npc_context_create(0, 1, 0, npc.npc_get_unique_id(), s)
        try:
            out = fn(0, ctx, s)
            s.synchronize()
        finally:
            ctx.close()
    return [out]


@pytest.mark.timeout(600)
@pytest.mark.parametrize("name,kind,ws", CASES)
def test_multirank_apply_poly_lanczos_pcg(wl, name, kind, ws):
    check_case(wl, name, kind, ws, run_ranks)


# a distributed context on ONE rank (include/npc.h): the multi-rank path with empty halos,
# through the local transport and through a real NCCL communicator
ONE = [("c3", "csr"), ("c4", "sell"), ("c2", "stencil"), ("c5", "schur"), ("c6", "dfn")]


@pytest.mark.timeout(600)
@pytest.mark.parametrize("name,kind", ONE)
def test_distributed_one_rank_local(wl, name, kind):
    check_case(wl, name, kind, 1, run_ranks)


@pytest.mark.timeout(600)
@pytest.mark.parametrize("name,kind", ONE)
def test_distributed_one_rank_nccl(wl, name, kind):
    check_case(wl, name, kind, 1, run_nccl_one_rank)


def check_case(wl, name, kind, ws, runner):
    w = wl(name)
    orc = oracle.Operator(w)
    n = w["n"]
    lo_o, hi_o = oracle.estimate_spectrum(orc, 20, W.lanczos_start(n))
    k = 12
    r = np.random.default_rng(9).uniform(-1, 1, n)
    x = np.random.default_rng(10).standard_normal(n)
    ref_apply = orc.apply(x)
    ref_poly = oracle.cheb_apply(orc, k, lo_o, hi_o, 1e-3, r)
    _, st_o = oracle.pcg(orc, w["b"], k, lo_o, hi_o, 0.0, tol=w["tol"], maxit=5000)

    def fn(rank, ctx, stream):
        op, r0, r1 = bench.create_operator(npc, ctx, w, kind, ws, rank, CFG[name])
        dev = lambda a: torch.tensor(np.ascontiguousarray(a[r0:r1]), device="cuda")  # noqa: E731
        y = torch.empty(r1 - r0, dtype=torch.float64, device="cuda")
        npc.npc_apply_operator(op, dev(x), y)
        poly = npc.npc_set_poly(op, k, lo_o, hi_o, 1e-3)
        z = torch.empty_like(y)
        npc.npc_apply_poly(poly, dev(r), z)
        lo, hi = npc.npc_estimate_spectrum(op, 20, None)
        p2 = npc.npc_set_poly(op, k, lo, hi, 0.0)
        xs = torch.zeros_like(y)
        st = npc.npc_pcg_solve(p2, op, dev(w["b"]), xs, w["tol"], 5000)
        stream.synchronize()
        mb = npc.npc_operator_matrix_bytes(op)
        return dict(r0=r0, r1=r1, y=y.cpu().numpy(), z=z.cpu().numpy(), lo=lo, hi=hi, st=st, x=xs.cpu().numpy(),
                    mb=mb)

    res = runner(ws, fn)
    y = np.concatenate([q["y"] for q in res])
    z = np.concatenate([q["z"] for q in res])
    xs = np.concatenate([q["x"] for q in res])
    assert [q["r0"] for q in res] == sorted(q["r0"] for q in res) and res[-1]["r1"] == n
    if kind == "csr" and name == "c3":
        # z-slab ghosts have one offset per neighbour plane: the coded form (9 B/nnz) holds
        # across ranks too, boundary tiles included
        rp = w["rowptr"]
        for q in res:
            nnz = int(rp[q["r1"]] - rp[q["r0"]])
            assert q["mb"] < 9.5 * nnz + 4 * (q["r1"] - q["r0"] + 1), (q["mb"], nnz)
    # Schur: fp64 atomics + a reduce-scatter; DFN: explicit block inverses vs the oracle's
    # triangular solves -- summation order only
    assert np.linalg.norm(y - ref_apply) <= (1e-12 if kind in ("schur", "dfn") else 1e-13) * np.linalg.norm(ref_apply)
    assert np.linalg.norm(z - ref_poly) <= 1e-10 * np.linalg.norm(ref_poly)
    # every rank holds the same global scalars
    assert len({(q["lo"], q["hi"]) for q in res}) == 1
    assert abs(res[0]["hi"] - hi_o) <= 1e-6 * hi_o
    its = {q["st"]["iters"] for q in res}
    assert len(its) == 1 and abs(its.pop() - st_o["iters"]) <= 2
    assert all(q["st"]["converged"] and q["st"]["relres_true"] <= w["tol"] for q in res)
    assert np.linalg.norm(w["b"] - orc.apply(xs)) / np.linalg.norm(w["b"]) <= w["tol"]
    # distributed PCG: ||r_{i+1}||^2 is allreduced on a side stream while
    # p_k(A) r_{i+1} runs, so the block in flight at convergence is cut short and not counted;
    # two global reductions per iteration + b/x0, r0 and the true residual
    st = res[0]["st"]
    assert st["op_applications"] == st["iters"] * (k + 1) + 1
    assert st["reductions"] == 2 * st["iters"] + 3


@pytest.mark.timeout(600)
@pytest.mark.parametrize("kind", ["csr", "sell", "schur"])
def test_multirank_with_an_empty_rank(kind):
    """Edge case: a rank that owns no rows still takes part in every collective (halo plans,
    allreduces, the Schur allgather / reduce-scatter) and the result matches the oracle."""
    w = W.config5(n=9_000) if kind == "schur" else W.config3(side=14)
    orc = oracle.Operator(w)
    n = w["n"]
    cuts = [0, n // 2, n // 2, n]  # rank 1 owns nothing
    lo_o, hi_o = oracle.estimate_spectrum(orc, 20, W.lanczos_start(n))
    r = np.random.default_rng(12).uniform(-1, 1, n)
    ref = oracle.cheb_apply(orc, 8, lo_o, hi_o, 0.0, r)
    _, st_o = oracle.pcg(orc, w["b"], 8, lo_o, hi_o, 0.0, tol=w["tol"], maxit=5000)

    def fn(rank, ctx, stream):
        r0, r1 = cuts[rank], cuts[rank + 1]
        if kind == "schur":
            nb = w["nb"]
            q0, q1 = nb * rank // 3, nb * (rank + 1) // 3
            bp = w["browptr"][q0:q1 + 1]
            op = npc.npc_create_operator(ctx, "schur", n_local=r1 - r0, n_global=n, row_begin=r0, c=w["c"][r0:r1],
                                         b_rows_global=nb, b_row_begin=q0, b_n_local=q1 - q0,
                                         b_rowptr=(bp - bp[0]).astype(np.int32),
                                         b_colidx=w["bcolidx"][bp[0]:bp[-1]], b_vals=w["bvals"][bp[0]:bp[-1]],
                                         d=w["d"][q0:q1])
        else:
            rp = w["rowptr"][r0:r1 + 1]
            op = npc.npc_create_operator(ctx, kind, n_local=r1 - r0, n_global=n, row_begin=r0,
                                         rowptr=(rp - rp[0]).astype(np.int32), colidx=w["colidx"][rp[0]:rp[-1]],
                                         vals=w["vals"][rp[0]:rp[-1]], sell_C=32, sell_sigma=256)
        dev = lambda a: torch.tensor(np.ascontiguousarray(a[r0:r1]), device="cuda")  # noqa: E731
        poly = npc.npc_set_poly(op, 8, lo_o, hi_o, 0.0)
        z = torch.empty(r1 - r0, dtype=torch.float64, device="cuda")
        npc.npc_apply_poly(poly, dev(r), z)
        lo, hi = npc.npc_estimate_spectrum(op, 20, None)
        p2 = npc.npc_set_poly(op, 8, lo, hi, 0.0)
        xs = torch.zeros(r1 - r0, dtype=torch.float64, device="cuda")
        st = npc.npc_pcg_solve(p2, op, dev(w["b"]), xs, w["tol"], 5000)
        stream.synchronize()
        return dict(z=z.cpu().numpy(), x=xs.cpu().numpy(), st=st)

    res = run_ranks(3, fn)
    z = np.concatenate([q["z"] for q in res])
    assert np.linalg.norm(z - ref) <= 1e-10 * np.linalg.norm(ref)
    its = {q["st"]["iters"] for q in res}
    assert len(its) == 1 and abs(its.pop() - st_o["iters"]) <= 2
    xs = np.concatenate([q["x"] for q in res])
    assert np.linalg.norm(w["b"] - orc.apply(xs)) / np.linalg.norm(w["b"]) <= w["tol"]


# ---------------------------------------------------------------- single fused allreduce
FUSED = [("c3", "csr", 2, "local"), ("c2", "stencil", 3, "local"), ("c5", "schur", 2, "local"),
         ("c3", "csr", 1, "nccl"), ("c4", "sell", 1, "nccl"), ("c6", "dfn", 1, "nccl")]


@pytest.mark.timeout(600)
@pytest.mark.parametrize("name,kind,ws,transport", FUSED)
def test_pcg_single_fused_allreduce(wl, name, kind, ws, transport):
    """npc_context_set_fused_allreduce(1): ONE allreduce of {gamma, delta, ||r||^2} per PCG
    iteration (north star).  Same iterates as the default side-stream check --
    identical iteration count and solution -- but the exit is seen one (k+1)-application block
    late: op_applications = (iters + 1)(k + 1) + 1 (SURVEY §8(b) "naive single-allreduce
    exit"), reductions = iters + 1 (the block that sees the exit) + 3."""
    w = wl(name)
    orc = oracle.Operator(w)
    n = w["n"]
    lo_o, hi_o = oracle.estimate_spectrum(orc, 20, W.lanczos_start(n))
    k = 12
    _, st_o = oracle.pcg(orc, w["b"], k, lo_o, hi_o, 0.0, tol=w["tol"], maxit=5000)

    def fn(rank, ctx, stream):
        op, r0, r1 = bench.create_operator(npc, ctx, w, kind, ws, rank, CFG[name])
        b = torch.tensor(np.ascontiguousarray(w["b"][r0:r1]), device="cuda")
        poly = npc.npc_set_poly(op, k, lo_o, hi_o, 0.0)
        out = {}
        for fused in (False, True, True):  # the second fused solve replays the cached graph
            npc.npc_context_set_fused_allreduce(ctx, fused)
            xs = torch.zeros_like(b)
            st = npc.npc_pcg_solve(poly, op, b, xs, w["tol"], 5000)
            stream.synchronize()
            out[fused] = (st, xs.cpu().numpy())
        # maxit: the fused form stops after exactly maxit x-updates too
        xs = torch.zeros_like(b)
        stm = npc.npc_pcg_solve(poly, op, b, xs, 1e-14, 3, raise_on_error=False)
        assert stm["status"] != "NPC_SUCCESS" and stm["iters"] == 3 and not stm["converged"], stm
        return out

    res = (run_ranks if transport == "local" else run_nccl_one_rank)(ws, fn)
    st0, st1 = res[0][False][0], res[0][True][0]
    assert st0["iters"] == st1["iters"] and abs(st1["iters"] - st_o["iters"]) <= 2
    assert st1["converged"] and st1["relres_true"] <= w["tol"]
    assert st1["op_applications"] == (st1["iters"] + 1) * (k + 1) + 1
    assert st1["reductions"] == st1["iters"] + 1 + 3
    assert st0["reductions"] == 2 * st0["iters"] + 3
    x0 = np.concatenate([q[False][1] for q in res])
    x1 = np.concatenate([q[True][1] for q in res])
    # the two forms run the same arithmetic on the same data (the multi-rank Schur operator
    # accumulates B^T t with fp64 atomics, so its bits vary from run to run)
    if kind == "schur" and ws > 1:
        assert np.linalg.norm(x0 - x1) <= 1e-10 * np.linalg.norm(x0)
    else:
        assert np.array_equal(x0, x1)
    assert np.linalg.norm(w["b"] - orc.apply(x1)) / np.linalg.norm(w["b"]) <= w["tol"]
