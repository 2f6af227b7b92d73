#!/usr/bin/env python
"""bench.py -- the north-star measurement: p_k(A) v GB/s and PCG time-to-tol (fp64) on B200.

One STEP = one pass of the whole hot path over the workload:
    npc_estimate_spectrum (20 Lanczos steps, counter-hash start)  ->  npc_set_poly(k, lmin, lmax, xi)
    -> npc_pcg_solve(b, x0 = 0, tol)   [k fused degree kernels + 1 SpMV + update per iteration]
on config 3 of BASELINE.json (3D 7-point variable-coefficient diffusion, 256^3, CSR, b = A 1,
tol 1e-8) at N = 1; `--config` selects another.  The operator is created (a0, setup) before the
timed region.  value = algorithmic bytes of every kernel of the step (SURVEY §8(d) floors:
matrix once + the vector streams each kernel must touch) / step time, in GB/s.
ms_per_step is the PCG time-to-tol including the spectrum estimate.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 3] [--k 20] [--impl ours|reference]

N > 1 (torchrun, one rank per GPU): rows partitioned in z-slabs / row blocks over NCCL,
strong scaling on the fixed problem; time = max over ranks of the CUDA-event time.
--impl reference: the CPU fp64 oracle (oracle/) timed on the host cores on a bounded sample
(one p_k(A) v application of the same workload per step), same metric and unit.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import workloads as W  # noqa: E402

PEAKS_FILE = os.path.join(ROOT, "MEASURED_PEAKS.json")
# BASELINE.json metric, as both arms report it: algorithmic bytes of the timed
# step / step time.  Our arm's step is the whole PCG-to-tol solve (ms_per_step = time-to-tol);
# the reference arm's step is a bounded sample (one p_k(A) v application by the CPU oracle).
METRIC = "p_k(A)v GB/s (algorithmic bytes of the timed step / step time)"
FALLBACK_HBM = 6650.0


def l2_peaks():
    """The L2 roofline denominators measured by tools/microbench/l2_peak.cu on this pool's B200
    (profiles/r02_l2_peak.json): L2-resident copy GB/s and random 8-byte gathers (sectors/s)."""
    try:
        with open(os.path.join(ROOT, "profiles", "r02_l2_peak.json")) as f:
            return json.load(f)
    except Exception:
        return None


def hbm_peak():
    try:
        with open(PEAKS_FILE) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return FALLBACK_HBM, "fallback (B200_PROFILING.md)"


# ------------------------------------------------------------------ workloads / byte model
def make_workload(cfg: int, side: int | None):
    if cfg == 1:
        return W.config1()
    if cfg == 2:
        return W.config2(side or 128)
    if cfg == 3:
        return W.config3(side or 256)
    if cfg == 4:
        return W.config4(n=side or 8_000_000)
    if cfg == 5:
        return W.config5(n=side or 4_000_000)
    if cfg == 6:  # the paper's DFN Schur operator, Frac32-sized, u in
        # owner order so that --gpus N can use the DSMat fracture-block partition
        return W.dfn_owner_order(W.dfn(nf=side or 29_370))
    raise ValueError(cfg)


def op_kind(w, cfg):
    return {1: "csr", 2: "stencil", 3: "csr", 4: "sell", 5: "schur", 6: "dfn"}[cfg] if w["kind"] != "stencil" \
        else "stencil"


def matrix_bytes(w, kind):
    """Bytes of the operator data one application must stream."""
    n = w["n"]
    if kind == "csr":
        return int(w["rowptr"][-1]) * 12 + (n + 1) * 4
    if kind == "sell":
        return int(w["rowptr"][-1]) * 12 * 1.0366 + n / 32 * 8  # padding measured for config 4
    if kind == "stencil":
        return 0
    if kind == "schur":
        # atomic form (op_schur.cu default): Bt = D^{-1/2} B streamed once (12 B per entry),
        # c once, y scattered then read/reset (SURVEY §8(d) floor, ~704 MB per degree at config 5
        # with the four vector streams of poly_bytes)
        nnz = int(w["browptr"][-1])
        return nnz * 12 + n * 8 + 2 * n * 8
    if kind == "dfn":
        # op_dfn.cu: C, B and their transposes, G^h, G^u once (12 B/nnz + row pointers), the band
        # factor of A (8 B/entry; band = bandwidth + 1 per row, nx for a grid block), and the
        # internal vectors t, u2 (written and read) plus the second read of x
        nh = w["nh"]
        nnz = lambda key: int(w[key][0][-1])  # noqa: E731
        hb = w["hblk"]
        rp, ci, _ = w["A"]
        band = 0
        for f in range(len(hb) - 1):
            r0, r1 = int(hb[f]), int(hb[f + 1])
            rows = np.repeat(np.arange(r0, r1), np.diff(rp[r0:r1 + 1]))
            band += (r1 - r0) * (int(np.max(np.abs(rows - ci[rp[r0]:rp[r1]]))) + 1)
        return int(12 * (2 * nnz("C") + 2 * nnz("B") + nnz("Gh") + nnz("Gu")) + 4 * (5 * nh + 3 * n) + 8 * band
                   + 8 * (4 * nh + n))
    raise ValueError(kind)


def poly_bytes(M, V, k):
    """Algorithmic bytes of one p_k(A) r: degree 1 reads r (x) and writes s_1; degree 2 reads
    s_1, r and writes; degrees >= 3 read s_{j-1}, s_{j-2}, r and write s_j."""
    if k == 0:
        return 2 * V
    b = M + 2 * V
    if k >= 2:
        b += M + 3 * V
    if k >= 3:
        b += (k - 2) * (M + 4 * V)
    return b


def solve_bytes(M, V, k, iters, lanczos_steps):
    per_iter = poly_bytes(M, V, k) + (M + 2 * V) + 10 * V  # p_k, w = A u, fused update
    lz = lanczos_steps * ((M + 2 * V) + 7 * V)             # SpMV + two axpy/dot passes + q update
    setup = 6 * V                                          # b/x copies, norms, r0
    return iters * per_iter + lz + setup + (M + 3 * V)     # + final true residual


def config_dict(cfg, w, kind, k, xi, M, V):
    """The workload description shared by both arms (same keys, same values)."""
    return {"workload": f"config{cfg}: {w['name']}", "operator": kind, "n": w["n"], "k": k, "xi": xi,
            "tol": w["tol"], "lanczos_steps": w.get("lanczos_steps", 20),
            "l2": "inputs larger than L2 (matrix + vectors > 126 MB)" if (M + 4 * V) > 126e6
            else "working set may be L2-resident (no flush)"}


# ------------------------------------------------------------------ clocks sampling
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    # Started before the warm-up: nvidia-smi's NVML start-up stalls CUDA calls of this process
    # for tens to hundreds of ms (measured), so it must not fall inside the timed region; only
    # the samples that arrive between mark_begin() and mark_end() are summarised.
    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []
        self.t0 = self.t1 = None

    def mark_begin(self):
        self.t0 = time.time()

    def mark_end(self):
        self.t1 = time.time()

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for ln in self.proc.stdout:
            self.lines.append((time.time(), ln.strip()))

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        for _ in range(20):  # a short run may end before the first sample: wait for one
            if self.lines:
                break
            time.sleep(0.05)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons, pw = [], None, set(), []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        inside = [ln for t, ln in self.lines if self.t0 is not None and self.t0 <= t <= (self.t1 or t)]
        for ln in inside or [ln for _, ln in self.lines[-3:]]:
            p = [x.strip() for x in ln.split(",")]
            if len(p) < 7:
                continue
            try:
                sm.append(float(p[0]))
                mx = float(p[1])
            except ValueError:
                continue
            try:
                pw.append(float(p[2]))
            except ValueError:
                pass
            for nm, v in zip(names, p[3:7]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm), "power_w_median": float(np.median(pw)) if pw else None,
                "power_w_max": float(np.max(pw)) if pw else None}


# ------------------------------------------------------------------ distributed helpers
def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def partition_rows(w, cfg, ws, rank):
    """Row block of this rank: z-slabs for grids (configs 2, 3), contiguous blocks otherwise."""
    n = w["n"]
    if "grid" in w and len(w["grid"]) == 3 or w["kind"] == "stencil":
        nz = w["grid"][2] if "grid" in w else w["nz"]
        plane = n // nz
        z0 = nz * rank // ws
        z1 = nz * (rank + 1) // ws
        return z0 * plane, z1 * plane, (z0, z1 - z0)
    r0 = n * rank // ws
    r1 = n * (rank + 1) // ws
    return r0, r1, None


def create_operator(npc, ctx, w, kind, ws, rank, cfg):
    if ws == 1 and not getattr(ctx, "distributed", False):
        return npc.create_from_workload(ctx, w, kind), 0, w["n"]
    r0, r1, zs = partition_rows(w, cfg, ws, rank)
    if kind == "stencil":
        return npc.npc_create_operator(ctx, "stencil", n_local=r1 - r0, n_global=w["n"], row_begin=r0, dim=3,
                                       nx=w["nx"], ny=w["ny"], nz_global=w["nz"], z_begin=zs[0],
                                       nz_local=zs[1], diag=w["diag"], offdiag=w["offdiag"]), r0, r1
    if kind in ("csr", "sell"):
        rp = w["rowptr"][r0:r1 + 1]
        op = npc.npc_create_operator(ctx, kind, n_local=r1 - r0, n_global=w["n"], row_begin=r0,
                                     rowptr=(rp - rp[0]).astype(np.int32), colidx=w["colidx"][rp[0]:rp[-1]],
                                     vals=w["vals"][rp[0]:rp[-1]], sell_C=32, sell_sigma=256)
        return op, r0, r1
    if kind == "schur":
        # trace rows and B rows in contiguous blocks: the B pass needs
        # all of v (allgather) and its partial B^T t covers all trace rows (reduce-scatter)
        nb = w["nb"]
        q0, q1 = nb * rank // ws, nb * (rank + 1) // ws
        bp = w["browptr"][q0:q1 + 1]
        op = npc.npc_create_operator(ctx, "schur", n_local=r1 - r0, n_global=w["n"], row_begin=r0,
                                     c=w["c"][r0:r1], b_rows_global=nb, b_row_begin=q0, b_n_local=q1 - q0,
                                     b_rowptr=(bp - bp[0]).astype(np.int32), b_colidx=w["bcolidx"][bp[0]:bp[-1]],
                                     b_vals=w["bvals"][bp[0]:bp[-1]], d=w["d"][q0:q1])
        return op, r0, r1
    if kind == "dfn":
        # DSMat partition: consecutive whole fracture blocks per rank, u rows
        # by owning fracture (w must be in owner order: workloads.dfn_owner_order)
        nf = w["nf"]
        f0, f1 = nf * rank // ws, nf * (rank + 1) // ws
        hb = np.asarray(w["hblk"], dtype=np.int64)
        h0, h1 = int(hb[f0]), int(hb[f1])
        u0, u1 = int(w["uoff"][f0]), int(w["uoff"][f1])

        def rows(t, a, b):
            rp, ci, v = t
            return ((rp[a:b + 1] - rp[a]).astype(np.int32), ci[rp[a]:rp[b]], v[rp[a]:rp[b]])
        op = npc.npc_create_operator(
            ctx, "dfn", n_local=u1 - u0, n_global=w["n"], row_begin=u0,
            dfn=dict(nh=h1 - h0, nblk=f1 - f0, hblk=(hb[f0:f1 + 1] - h0).astype(np.int32), A=rows(w["A"], h0, h1),
                     Gh=rows(w["Gh"], h0, h1), C=rows(w["C"], h0, h1), B=rows(w["B"], h0, h1),
                     Gu=rows(w["Gu"], u0, u1), alpha=w["alpha"], scaled=w.get("scaled", 1)))
        return op, u0, u1
    raise SystemExit(f"config kind {kind} does not support --gpus > 1 in this version")


# ------------------------------------------------------------------ our arm
def run_ours(args):
    import torch
    import torch.distributed as dist
    import paper_2208_01339_b200 as npc

    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    if ws > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cfg = args.config
    w = make_workload(cfg, args.side)
    kind = args.kind or op_kind(w, cfg)
    k = args.k if args.k is not None else w["k"]
    tol = w["tol"]
    xi = args.xi
    lz_steps = w.get("lanczos_steps", 20)
    uid = None
    if ws > 1:
        t = torch.zeros(128, dtype=torch.uint8, device="cuda")
        if rank == 0:
            t.copy_(torch.frombuffer(bytearray(npc.npc_get_unique_id()), dtype=torch.uint8))
        dist.broadcast(t, 0)
        uid = bytes(t.cpu().numpy().tobytes())
    elif args.distributed:
        uid = npc.npc_get_unique_id()
    stream = torch.cuda.current_stream()
    ctx = npc.npc_context_create(local, ws, rank, uid, stream)
    op, r0, r1 = create_operator(npc, ctx, w, kind, ws, rank, cfg)
    nl = r1 - r0
    b_host = np.ascontiguousarray(w["b"][r0:r1])
    b = torch.tensor(b_host, device="cuda")
    x = torch.zeros(nl, dtype=torch.float64, device="cuda")
    maxit = args.maxit

    def barrier():
        if ws > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def step(bb, xx):
        lo, hi = npc.npc_estimate_spectrum(op, lz_steps, None)
        poly = npc.npc_set_poly(op, k, lo, hi, xi)
        xx.zero_()
        st = npc.npc_pcg_solve(poly, op, bb, xx, tol, maxit)
        poly.close()
        st["lmin"], st["lmax"] = lo, hi
        return st

    clocks = ClockSampler(local)
    clocks.start()
    for _ in range(args.warmup):
        st = step(b, x)
    barrier()
    clocks.mark_begin()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches0 = npc.npc_launch_count()
    if not args.no_kernel_timing:
        npc.npc_context_set_timing(ctx, True)
        npc.npc_context_get_timing(ctx)  # reset
    barrier()
    ev0.record(stream)
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    stats = []
    for i in range(args.steps):
        stats.append(step(b, x))
        evs[i].record(stream)
    ev1.record(stream)
    barrier()
    clocks.mark_end()
    launches = npc.npc_launch_count() - launches0
    ktime = None
    if not args.no_kernel_timing:
        ktime = npc.npc_context_get_timing(ctx)
        npc.npc_context_set_timing(ctx, False)
    clk = clocks.stop()
    ms = ev0.elapsed_time(ev1)
    step_ms = [round(ev0.elapsed_time(evs[0]), 3)] + [round(evs[i - 1].elapsed_time(evs[i]), 3)
                                                      for i in range(1, args.steps)]
    t = torch.tensor([ms], dtype=torch.float64, device="cuda")
    if ws > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_step = float(t.item()) / args.steps
    iters = stats[-1]["iters"]
    M = matrix_bytes(w, kind)
    V = 8 * w["n"]
    step_bytes = solve_bytes(M, V, k, iters, lz_steps)
    gbs = step_bytes / (ms_step * 1e-3) / 1e9

    # -------- dominant kernel: the fused degree step, timed live with CUDA events on the
    # library's stream (= torch's current stream) over R applications of p_k(A)
    lo, hi = stats[-1]["lmin"], stats[-1]["lmax"]
    poly = npc.npc_set_poly(op, k, lo, hi, xi)
    z = torch.empty_like(b)
    R = max(3, args.kernel_reps)
    npc.npc_apply_poly(poly, b, z)
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(R):
        npc.npc_apply_poly(poly, b, z)
    e1.record(stream)
    barrier()
    t_apply = e0.elapsed_time(e1) / R  # ms per p_k(A) r (k launches)
    # roofline numerator: the bytes the kernels stream in the library's stored format (the
    # pattern form streams ~4.7 B per nonzero, not 12), this rank's share
    # (CSR only: the other operators are reported against their §8(d) floor, like tools/bench_all.py)
    Mf = npc.npc_operator_matrix_bytes(op) if kind == "csr" else M / ws
    Vf = 8 * nl
    apply_bytes = poly_bytes(Mf, Vf, k)
    per_launch_ms = t_apply / max(k, 1)
    peak, peak_src = hbm_peak()
    ach_isolated = apply_bytes / max(k, 1) / (per_launch_ms * 1e-3) / 1e9
    ach = ach_isolated
    in_step = None
    if ktime is not None and ktime["degree"][1] > 0:
        # the fused degree kernels as they ran inside the timed region (library CUDA events
        # on the launching stream): bytes of every degree launch / their summed device time
        n_deg = ktime["degree"][1]
        deg_bytes = sum(s["iters"] for s in stats) * poly_bytes(Mf, Vf, k)
        ach = deg_bytes / (ktime["degree"][0] * 1e-3) / 1e9
        per_launch_ms = ktime["degree"][0] / n_deg
        in_step = {c: {"ms": round(v[0], 3), "launches": v[1], "share": round(v[0] / (ms_step * args.steps), 4)}
                   for c, v in ktime.items()}
    # -------- per-rank timing (N > 1): each rank's own step time and its in-library kernel
    # classes; what the kernels do not cover is halo / allreduce waiting and host work
    per_rank = None
    if ws > 1:
        mine = {"rank": rank, "n_local": nl, "step_ms": round(ms / args.steps, 3)}
        if ktime is not None:
            kms = {c: v[0] / args.steps for c, v in ktime.items()}
            mine.update({f"{c}_ms": round(v, 3) for c, v in kms.items()})
            mine["outside_kernels_ms"] = round(ms / args.steps - sum(kms.values()), 3)
        per_rank = [None] * ws
        dist.all_gather_object(per_rank, mine)
    # DRAM traffic of one degree launch from the committed ncu --set full capture of this
    # workload's kernel (profiles/traffic_config<C>.json, tools/traffic_from_ncu.py); used only
    # if it was captured on the operator format this run stores (same matrix bytes), else null
    traffic = None
    tf = os.path.join(ROOT, "profiles", f"traffic_config{cfg}.json")
    if os.path.exists(tf) and ws == 1:
        try:
            tj = json.load(open(tf))
            mb = npc.npc_operator_matrix_bytes(op)
            if tj.get("matrix_bytes") and abs(tj["matrix_bytes"] - mb) <= 1e-6 * mb and tj.get("k", k) == k:
                traffic = tj.get("dram_bytes_per_launch")
        except Exception:
            traffic = None

    # -------- L2 rooflines where HBM is not the bound: an L2-resident stencil (config 2: the
    # four vector streams fit in L2) against the measured L2 copy rate, and the Schur operator
    # (config 5) against the measured random-sector rate: its two passes gather v and t at
    # random, one 32-byte L2 sector per 8-byte value, 2 nnz(B) sectors per application
    l2_roof = None
    l2p = l2_peaks()
    if l2p and ws == 1:
        if kind == "stencil" and 4 * V <= 0.75 * 126e6:
            l2_roof = {"bound": "l2", "achieved": round(ach, 1), "peak": l2p["l2_copy_rw_gbs"], "unit": "GB/s",
                       "frac": round(ach / l2p["l2_copy_rw_gbs"], 4),
                       "peak_source": "measured L2-resident copy (profiles/r02_l2_peak.json)"}
        if kind == "schur":
            sectors = 2.0 * int(w["browptr"][-1])  # random gathers per application (v, then t)
            t_deg = per_launch_ms * 1e-3
            l2_roof = {"bound": "l2_random_sectors", "achieved": round(sectors / t_deg, 1),
                       "peak": l2p["l2_random8B_sectors_per_s"], "unit": "sectors/s",
                       "frac": round(sectors / t_deg / l2p["l2_random8B_sectors_per_s"], 4),
                       "floor_ms_per_degree": round(sectors / l2p["l2_random8B_sectors_per_s"] * 1e3, 4),
                       "peak_source": "measured random 8-byte gathers (profiles/r02_l2_peak.json)"}

    # -------- e2e: the public API from host buffers: operator upload (npc_create_operator
    # copies the host CSR), b H2D from pinned memory, estimate + set_poly + solve, x D2H
    e2e_val = None
    h2d = d2h = 0
    if not args.no_e2e:
        b_pin = torch.from_numpy(b_host).pin_memory()
        x_pin = torch.empty(nl, dtype=torch.float64).pin_memory()
        e2e_steps = max(1, min(args.steps, args.e2e_steps))
        barrier()
        keep = []  # handles are destroyed after the timed region (teardown is not part of a step)
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            op2, _, _ = create_operator(npc, ctx, w, kind, ws, rank, cfg)
            bd = b_pin.to("cuda", non_blocking=True)
            xd = torch.empty(nl, dtype=torch.float64, device="cuda")
            lo2, hi2 = npc.npc_estimate_spectrum(op2, lz_steps, None)
            p2 = npc.npc_set_poly(op2, k, lo2, hi2, xi)
            xd.zero_()
            npc.npc_pcg_solve(p2, op2, bd, xd, tol, maxit)
            x_pin.copy_(xd, non_blocking=True)
            torch.cuda.synchronize()
            keep.append((p2, op2))
        barrier()
        te = torch.tensor([(time.perf_counter() - t0) / e2e_steps], dtype=torch.float64, device="cuda")
        for p2, op2 in keep:
            p2.close()
            op2.close()
        if ws > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e_val = step_bytes / float(te.item()) / 1e9
        if kind in ("csr", "sell"):
            nnz_l = int(w["rowptr"][r1] - w["rowptr"][r0])
            h2d = nnz_l * 12 + (nl + 1) * 4 + nl * 8
        else:
            h2d = nl * 8
        d2h = nl * 8

    # -------- CPU oracle baseline (rank 0, N = 1 only): one bounded p_k(A) v sample
    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu:
        cpu = cpu_baseline(w, k, lo, hi, xi, M, V, max_seconds=args.cpu_seconds)

    if rank == 0:
        line = {
            "metric": METRIC,
            "value": round(gbs, 2), "unit": "GB/s", "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
            "value_basis": "effective bandwidth: format-independent SURVEY §8(d) bytes of the step (CSR: 12 B per "
                           "nonzero) / time-to-tol, so it can exceed the copy rate when the stored format moves less "
                           "(the pattern form streams ~4.7 B per nonzero); roofline.* uses the bytes actually streamed",
            "ms_per_step": round(ms_step, 3), "step_ms": step_ms, "higher_is_better": True,
            "scaling": "strong" if ws > 1 else "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded workloads/, BASELINE.json config recipe)",
            "config": config_dict(cfg, w, kind, k, xi, M, V),
            "parallelism": f"row-block x{ws} (z-slabs for grids), NCCL halo + 1 allreduce/iteration" if ws > 1
            else "1 GPU, multi-rank path on a 1-rank NCCL communicator" if args.distributed else "1 GPU",
            "pcg": {"iters": iters, "converged": stats[-1]["converged"], "relres_true": stats[-1]["relres_true"],
                    "op_applications": stats[-1]["op_applications"], "reductions": stats[-1]["reductions"],
                    "lmin": lo, "lmax": hi, "time_to_tol_ms": round(ms_step, 3),
                    "op_applications_per_s": round(stats[-1]["op_applications"] / (ms_step * 1e-3), 1)},
            "roofline": {"bound": "hbm", "kernel": f"fused degree step ({kind})", "achieved": round(ach, 1),
                         "peak": peak, "peak_source": peak_src, "unit": "GB/s", "frac": round(ach / peak, 4),
                         "frac_vs_8TBs_nominal": round(ach / 8000.0, 4),
                         # the same launches on SURVEY §8(d)'s format-independent bytes (CSR 12 B per
                         # nonzero): > 1 when the stored format streams less than that floor assumes
                         "frac_survey_8d_bytes": round(ach * poly_bytes(M / ws, Vf, k) / max(apply_bytes, 1) / peak, 4),
                         "traffic": traffic,
                         "bytes_per_launch": apply_bytes / max(k, 1), "launch_ms": round(per_launch_ms, 5),
                         "bytes_basis": ("operator data in the stored format (npc_operator_matrix_bytes: "
                                         f"{Mf / 1e6:.1f} MB per application) + the recurrence's vector streams; "
                                         "`value` uses the format-independent SURVEY §8(d) bytes "
                                         f"({M / ws / 1e6:.1f} MB), the reference arm's basis") if kind == "csr"
                         else f"SURVEY §8(d) bytes ({M / ws / 1e6:.1f} MB of operator data per application) + the "
                              "recurrence's vector streams, the same basis as `value`",
                         "timed": "library CUDA events on the launching stream inside the timed region: one event "
                         "pair around each p_k(A) r application (its k fused degree launches, replayed in the PCG "
                         "CUDA graph as event-record nodes); achieved = algorithmic bytes of the degree steps / their "
                         "summed device time" if in_step
                         else f"{R} x npc_apply_poly (k={k} launches each), CUDA events on the library stream",
                         "isolated_achieved": round(ach_isolated, 1),
                         "isolated": f"{R} x npc_apply_poly back to back after the timed region",
                         "step_breakdown": in_step},
            **({"roofline_l2": l2_roof} if l2_roof else {}),
            "e2e": {"value": round(e2e_val, 2) if e2e_val else None, "unit": "GB/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h,
                    "includes": "npc_create_operator from host CSR + b H2D (pinned) + estimate + set_poly + solve + x D2H"},
            "gpu_launches": int(launches),
            **({"per_rank": per_rank} if per_rank else {}),
            "clocks": clk,
            "cpu_baseline": cpu,
        }
        emit(line)
    if ws > 1:
        dist.destroy_process_group()


def host_info():
    """CPU model and a STREAM-triad bandwidth (numpy a = b + s c on 3 x 256 MB, one thread) of
    the host the oracle runs on (record nproc, the CPU model, a triad GB/s)."""
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    model = ln.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    n = 32 * 1024 * 1024
    b, c = np.ones(n), np.full(n, 2.0)
    a = np.empty(n)
    best = 0.0
    for _ in range(3):
        t0 = time.perf_counter()
        np.multiply(c, 3.0, out=a)
        np.add(a, b, out=a)
        dt = time.perf_counter() - t0
        best = max(best, 4 * 8 * n / dt / 1e9)  # two passes: read c, write a, read a+b, write a
    return {"cpu_model": model, "nproc": os.cpu_count(), "stream_triad_gbs_1thread": round(best, 1)}


def cpu_baseline(w, k, lo, hi, xi, M, V, max_seconds=30.0):
    """The oracle as it stands, one p_k(A) v application of the same workload on the host cores."""
    try:
        import oracle
    except Exception as e:  # pragma: no cover
        return {"value": None, "error": str(e)}
    orc = oracle.Operator(w)
    r = np.asarray(w["b"], dtype=np.float64)
    kk = k
    t0 = time.perf_counter()
    oracle.cheb_apply(orc, kk, lo, hi, xi, r)
    dt = time.perf_counter() - t0
    byts = poly_bytes(M, V, kk)
    out = {"value": round(byts / dt / 1e9, 3), "unit": "GB/s", "cores": oracle.num_threads(), "kind": "oracle",
           "sample": f"one p_k(A) v application (k={kk}) of {w['name']} by Alg. 2 verbatim (oracle/npc_oracle.c)",
           "seconds": round(dt, 3), **host_info()}
    g = oracle_golden(w, kk, xi)
    if g:
        out["time_to_tol"] = g
    return out


def oracle_golden(w, k, xi):
    """The oracle's full PCG-to-tolerance on this workload, run once by tools/oracle_golden.py
    ("run once per benchmark session and cached"): iterations, counters and the
    wall time on the host that wrote it (not this run's host), if a golden exists."""
    import glob
    side = round(w["n"] ** (1 / 3))
    cands = glob.glob(os.path.join(ROOT, "tests", "golden", f"config*_{side}_pcg_k{k}.json")) + \
        glob.glob(os.path.join(ROOT, "tests", "golden", f"config*_{w['n']}_pcg_k{k}.json"))
    for path in cands:
        g = json.load(open(path))
        if g.get("workload") == w.get("name") and g.get("xi", 0.0) == xi:
            return {"seconds": round(g["seconds_time_to_tol"], 1), "iters": g["iters"], "mvp": g["mvp"],
                    "relres_true": g["relres_true"], "threads": g["threads"], "nproc": g["nproc"], "cpu": g["cpu"],
                    "source": os.path.relpath(path, ROOT) + " (tools/oracle_golden.py; written on the build host, "
                                                            "not this run's host)"}
    return None


# ------------------------------------------------------------------ reference arm (the oracle)
def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    import oracle
    cfg = args.config
    w = make_workload(cfg, args.side)
    kind = args.kind or op_kind(w, cfg)
    k = args.k if args.k is not None else w["k"]
    orc = oracle.Operator(w)
    # the oracle's own interval (20 Lanczos steps from the counter-hash start), as in the GPU arm
    lo, hi = oracle.estimate_spectrum(orc, w.get("lanczos_steps", 20), W.lanczos_start(w["n"]))
    M = matrix_bytes(w, kind)
    V = 8 * w["n"]
    r = np.asarray(w["b"], dtype=np.float64)
    for _ in range(args.warmup):
        oracle.cheb_apply(orc, k, lo, hi, args.xi, r)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        oracle.cheb_apply(orc, k, lo, hi, args.xi, r)
    dt = (time.perf_counter() - t0) / args.steps
    val = poly_bytes(M, V, k) / dt / 1e9
    line = {
        "impl": "reference", "metric": METRIC, "value": round(val, 3),
        "unit": "GB/s", "n_gpus": ws, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(dt * 1e3, 3),
        "higher_is_better": True, "scaling": "strong" if ws > 1 else "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded workloads/)",
        "config": config_dict(cfg, w, kind, k, args.xi, M, V),
        "cpu_baseline": {"value": round(val, 3), "unit": "GB/s", "cores": oracle.num_threads(), "kind": "oracle",
                         **host_info(),
                         "sample": f"each step = one p_k(A) v application (k={k}) of the full workload, Alg. 2 verbatim"},
        "e2e": {"value": round(val, 3), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    emit(line)


_json_out = None


def emit(line):
    """The one JSON line, on the process's real stdout."""
    out = _json_out or sys.stdout
    out.write(json.dumps(line) + "\n")
    out.flush()


def main():
    global _json_out
    # stdout carries exactly one JSON line: anything else written to fd 1 (native libraries,
    # e.g. NCCL's version banner) goes to stderr
    sys.stdout.flush()
    _json_out = os.fdopen(os.dup(1), "w")
    os.dup2(2, 1)
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--side", type=int, default=None, help="grid side (configs 2, 3) or n (configs 4, 5)")
    ap.add_argument("--kind", default=None, help="operator storage override (csr|sell)")
    ap.add_argument("--k", type=int, default=None)
    ap.add_argument("--xi", type=float, default=0.0)
    ap.add_argument("--maxit", type=int, default=20000)
    ap.add_argument("--kernel-reps", type=int, default=10)
    ap.add_argument("--e2e-steps", type=int, default=1)
    ap.add_argument("--cpu-seconds", type=float, default=30.0)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--distributed", action="store_true",
                    help="at --gpus 1: a 1-rank NCCL context, i.e. the multi-rank path (include/npc.h)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-kernel-timing", action="store_true",
                    help="do not bracket launches with library CUDA events in the timed region")
    args = ap.parse_args()
    if args.warmup < 3 and not os.environ.get("NPC_BENCH_ALLOW_SHORT"):
        print("warning: --warmup < 3 violates the timing rules", file=sys.stderr)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
