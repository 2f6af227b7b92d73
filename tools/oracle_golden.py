"""Write oracle PCG goldens for full-size BASELINE configs ("The full config-3
oracle PCG runs once ... and is cached for parity").

Imports ONLY oracle/ (the CPU fp64 reference, O2 Lanczos + O5 textbook PCG with Alg. 2) and
workloads/ (the seeded generators).  Nothing here touches the CUDA path: the numbers it
writes are the oracle's, and tests/test_gpu_fullsize.py compares the GPU solve with them.

    OMP_NUM_THREADS=6 python tools/oracle_golden.py --config 3 --side 256 --k 50
    python tools/oracle_golden.py --config 4 --k 60

Output: tests/golden/config{C}_{size}_pcg_k{K}.json with the iteration count, counters, the
true residual, the oracle's spectrum estimate, the wall time and thread count (the
cpu_baseline time-to-tolerance), the sha256 of oracle/npc_oracle.c and of the workload
arrays (so a test can refuse a stale golden).
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import platform
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import oracle  # noqa: E402
import workloads as W  # noqa: E402


def workload_sha(w: dict) -> str:
    """sha256 over the arrays that define the operator and the right-hand side."""
    h = hashlib.sha256()
    for key in ("rowptr", "colidx", "vals", "b", "c", "browptr", "bcolidx", "bvals", "d"):
        if key in w and w[key] is not None:
            h.update(key.encode())
            h.update(np.ascontiguousarray(w[key]).tobytes())
    return h.hexdigest()


def oracle_sha() -> str:
    with open(os.path.join(ROOT, "oracle", "npc_oracle.c"), "rb") as f:
        return hashlib.sha256(f.read()).hexdigest()


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor()


def make(config: int, side: int | None, n: int | None):
    if config == 3:
        return W.config3(side or 256)
    if config == 4:
        return W.config4(n=n or 8_000_000)
    if config == 2:
        return W.config2(side or 128)
    if config == 5:
        return W.config5(n=n or 4_000_000)
    raise SystemExit(f"config {config} not supported")


def golden_path(config: int, w: dict, k: int, xi: float) -> str:
    size = f"{round(w['n'] ** (1 / 3))}" if config in (2, 3) else f"{w['n']}"
    tag = "" if xi == 0.0 else f"_xi{xi:g}"
    return os.path.join(ROOT, "tests", "golden", f"config{config}_{size}_pcg_k{k}{tag}.json")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--side", type=int, default=None)
    ap.add_argument("--n", type=int, default=None)
    ap.add_argument("--k", type=int, default=50)
    ap.add_argument("--xi", type=float, default=0.0)
    ap.add_argument("--maxit", type=int, default=20000)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()

    t0 = time.time()
    w = make(a.config, a.side, a.n)
    t_gen = time.time() - t0
    orc = oracle.Operator(w)
    t1 = time.time()
    lo, hi = oracle.estimate_spectrum(orc, 20, W.lanczos_start(w["n"]))
    t_est = time.time() - t1
    print(f"[golden] config {a.config} n={w['n']} generated in {t_gen:.1f}s; lanczos {t_est:.1f}s "
          f"lmin={lo:.6e} lmax={hi:.6e}; PCG k={a.k} xi={a.xi} on {oracle.num_threads()} threads ...", flush=True)
    t2 = time.time()
    _, st = oracle.pcg(orc, w["b"], a.k, lo, hi, a.xi, tol=w["tol"], maxit=a.maxit)
    t_pcg = time.time() - t2
    out = dict(
        config=a.config, workload=w["name"], n=int(w["n"]), k=a.k, xi=a.xi, tol=w["tol"], maxit=a.maxit,
        lanczos_steps=20, lmin=lo, lmax=hi,
        iters=st["iters"], converged=st["converged"], breakdown=st["breakdown"], mvp=st["mvp"], ddot=st["ddot"],
        true_checks=st["true_checks"], relres_recursive=st["relres_recursive"], relres_true=st["relres_true"],
        seconds_estimate=t_est, seconds_pcg=t_pcg, seconds_time_to_tol=t_est + t_pcg,
        threads=oracle.num_threads(), nproc=os.cpu_count(), cpu=cpu_model(),
        oracle_sha256=oracle_sha(), workload_sha256=workload_sha(w),
        written_by="tools/oracle_golden.py (imports oracle/ and workloads/ only)",
        when=time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime()),
    )
    path = a.out or golden_path(a.config, w, a.k, a.xi)
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
