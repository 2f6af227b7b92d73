"""paper_2208_01339_b200 -- Python binding of libnpc (include/npc.h), argument marshalling only.

Every step of the hot path (the fused degree kernels, PCG, Lanczos, halo exchange) runs in
libnpc.so (hand-written CUDA for sm_100a).  PyTorch is used by callers for device memory and
streams; this module only converts tensors/arrays to pointers and checks status codes.  There
is no fallback: if libnpc.so is missing or cannot load, every call raises.

Names mirror the C ABI: npc_context_create, npc_create_operator, npc_estimate_spectrum,
npc_set_poly, npc_apply_poly, npc_pcg_solve, npc_apply_operator, ... (see include/npc.h for
argument meaning, layout, ownership and errors).
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("NPC_LIB_PATH") or os.path.join(_HERE, "libnpc.so")  # override: A/B variants

NPC_OP_CSR, NPC_OP_SELL, NPC_OP_STENCIL, NPC_OP_SCHUR, NPC_OP_CALLBACK, NPC_OP_DFN = range(6)
STATUS = {0: "NPC_SUCCESS", 1: "NPC_ERR_INVALID_ARGUMENT", 2: "NPC_ERR_DIMENSION",
          3: "NPC_ERR_DEGENERATE_INTERVAL", 4: "NPC_ERR_NOT_CONVERGED", 5: "NPC_ERR_BREAKDOWN",
          6: "NPC_ERR_CUDA", 7: "NPC_ERR_NCCL", 8: "NPC_ERR_OUT_OF_MEMORY", 9: "NPC_ERR_UNSUPPORTED",
          10: "NPC_ERR_INTERNAL"}
KIND = {"csr": NPC_OP_CSR, "sell": NPC_OP_SELL, "stencil": NPC_OP_STENCIL, "schur": NPC_OP_SCHUR,
        "callback": NPC_OP_CALLBACK, "dfn": NPC_OP_DFN}


class NpcError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"{STATUS.get(code, code)}: {msg}")
        self.code = code
        self.name = STATUS.get(code, str(code))


APPLY_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p)


class OperatorDesc(C.Structure):
    _fields_ = [
        ("kind", C.c_int), ("n_global", C.c_longlong), ("row_begin", C.c_longlong), ("n_local", C.c_int),
        ("rowptr", C.c_void_p), ("colidx", C.c_void_p), ("vals", C.c_void_p),
        ("sell_C", C.c_int), ("sell_sigma", C.c_int),
        ("stencil_dim", C.c_int), ("nx", C.c_int), ("ny", C.c_int), ("nz_global", C.c_int),
        ("z_begin", C.c_int), ("nz_local", C.c_int), ("diag", C.c_double), ("offdiag", C.c_double),
        ("c", C.c_void_p), ("b_rows_global", C.c_longlong), ("b_row_begin", C.c_longlong),
        ("b_n_local", C.c_int), ("b_rowptr", C.c_void_p), ("b_colidx", C.c_void_p),
        ("b_vals", C.c_void_p), ("d", C.c_void_p),
        ("apply", APPLY_FN), ("user", C.c_void_p),
        ("dfn_nh", C.c_longlong), ("dfn_nblk", C.c_int), ("dfn_hblk", C.c_void_p),
        ("a_rowptr", C.c_void_p), ("a_colidx", C.c_void_p), ("a_vals", C.c_void_p),
        ("gh_rowptr", C.c_void_p), ("gh_colidx", C.c_void_p), ("gh_vals", C.c_void_p),
        ("c_rowptr", C.c_void_p), ("c_colidx", C.c_void_p), ("c_vals", C.c_void_p),
        ("bm_rowptr", C.c_void_p), ("bm_colidx", C.c_void_p), ("bm_vals", C.c_void_p),
        ("gu_rowptr", C.c_void_p), ("gu_colidx", C.c_void_p), ("gu_vals", C.c_void_p),
        ("dfn_alpha", C.c_double), ("dfn_scaled", C.c_int),
    ]


class PcgStats(C.Structure):
    _fields_ = [("iters", C.c_int), ("converged", C.c_int), ("op_applications", C.c_longlong),
                ("reductions", C.c_longlong), ("relres_recursive", C.c_double),
                ("relres_true", C.c_double), ("setup_seconds", C.c_double), ("solve_seconds", C.c_double),
                ("history", C.POINTER(C.c_double))]


_lib = None


def lib():
    """Load libnpc.so (raises if it is missing: there is no fallback path)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"libnpc.so not built ({LIB_PATH}); run `python -m paper_2208_01339_b200.build_lib`")
        L = C.CDLL(LIB_PATH)
        P, I, D, LL = C.c_void_p, C.c_int, C.c_double, C.c_longlong
        sig = {
            "npc_context_create": [I, I, I, P, P, C.POINTER(P)],
            "npc_context_destroy": [P],
            "npc_get_unique_id": [P],
            "npc_create_operator": [P, C.POINTER(OperatorDesc), C.POINTER(P)],
            "npc_destroy_operator": [P],
            "npc_operator_matrix_bytes": [P, C.POINTER(D)],
            "npc_apply_operator": [P, P, P],
            "npc_estimate_spectrum": [P, I, P, C.c_ulonglong, C.POINTER(D), C.POINTER(D)],
            "npc_estimate_spectrum_ex": [P, I, P, C.c_ulonglong, P],
            "npc_set_poly": [P, I, D, D, D, C.POINTER(P)],
            "npc_set_poly_newton": [P, I, D, D, D, C.POINTER(P)],
            "npc_destroy_poly": [P],
            "npc_apply_poly": [P, P, P],
            "npc_pcg_solve": [P, P, P, P, D, I, C.POINTER(PcgStats)],
            "npc_halo_plan": [I, P, P, I, P, I, C.POINTER(I), P, P],
            "npc_pattern_check": [I, P, P, P, P, P, P],
            "npc_poly_coefficients": [I, D, D, D, C.POINTER(D), C.POINTER(D), C.POINTER(D), P],
            "npc_context_set_timing": [P, I],
            "npc_context_set_fused_allreduce": [P, I],
            "npc_context_create_local": [I, I, I, C.c_char_p, P, C.POINTER(P)],
            "npc_context_get_timing": [P, P, P],
            "npc_poly_set_lowrank": [P, I, P],
            "npc_ritz_vectors": [P, I, I, P, P, P],
        }
        for name, args in sig.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = C.c_int
        L.npc_last_error.restype = C.c_char_p
        L.npc_last_error.argtypes = [P]
        L.npc_version.restype = C.c_char_p
        L.npc_launch_count.restype = C.c_ulonglong
        _lib = L
    return _lib


def npc_last_error(ctx=None) -> str:
    """Message of the last failing call on ctx (a Context), or on this thread (None)."""
    return lib().npc_last_error(ctx.h if ctx is not None else None).decode(errors="replace")


def _check(code):
    if code != 0:
        raise NpcError(code, lib().npc_last_error(None).decode(errors="replace"))


def _ptr(t):
    """Device pointer of a torch tensor (fp64, contiguous) or None."""
    if t is None:
        return None
    import torch
    assert t.dtype == torch.float64 and t.is_contiguous() and t.is_cuda, "expected a contiguous fp64 CUDA tensor"
    return C.c_void_p(t.data_ptr())


def _host(a, dt):
    a = np.ascontiguousarray(a, dtype=dt)
    return a, a.ctypes.data_as(C.c_void_p)


def npc_version() -> str:
    return lib().npc_version().decode()


def npc_launch_count() -> int:
    return int(lib().npc_launch_count())


def npc_get_unique_id() -> bytes:
    buf = (C.c_ubyte * 128)()
    _check(lib().npc_get_unique_id(C.cast(buf, C.c_void_p)))
    return bytes(buf)


class Context:
    def __init__(self, handle, stream):
        self.h = handle
        self.stream = stream
        self.distributed = False

    def close(self):
        if self.h:
            lib().npc_context_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def npc_context_create(device: int = 0, nranks: int = 1, rank: int = 0, unique_id: bytes | None = None,
                       stream=None) -> Context:
    """stream: a torch.cuda.Stream (default: torch's current stream on `device`)."""
    import torch
    if stream is None:
        stream = torch.cuda.current_stream(device)
    uid = None
    if unique_id is not None:
        assert len(unique_id) == 128
        uid = C.cast(C.create_string_buffer(unique_id, 128), C.c_void_p)
    h = C.c_void_p()
    # torch's default stream is the legacy NULL stream (handle 0); NULL means "library-owned
    # stream" in the C ABI, so pass cudaStreamLegacy (0x1) to enqueue on torch's stream.
    handle = stream.cuda_stream or 0x1
    _check(lib().npc_context_create(device, nranks, rank, uid, C.c_void_p(handle), C.byref(h)))
    c = Context(h, stream)
    c.distributed = unique_id is not None  # include/npc.h: a transport makes the context distributed
    return c


def npc_context_create_local(device: int, nranks: int, rank: int, group: str, stream=None) -> Context:
    """Rank `rank` of a local thread group (testing transport; see include/npc.h)."""
    import torch
    if stream is None:
        stream = torch.cuda.current_stream(device)
    h = C.c_void_p()
    handle = stream.cuda_stream or 0x1
    _check(lib().npc_context_create_local(device, nranks, rank, group.encode(), C.c_void_p(handle), C.byref(h)))
    c = Context(h, stream)
    c.distributed = True
    return c


TIMING_CLASSES = ("degree", "operator", "update", "reduce", "vector")


def npc_context_set_timing(ctx: Context, enable: bool = True):
    _check(lib().npc_context_set_timing(ctx.h, int(bool(enable))))


def npc_context_set_fused_allreduce(ctx: Context, enable: bool = True):
    """PCG on a distributed context: one {gamma, delta, ||r||^2} allreduce per iteration."""
    _check(lib().npc_context_set_fused_allreduce(ctx.h, int(bool(enable))))


def npc_context_get_timing(ctx: Context) -> dict:
    """{class: (device ms, launches)} accumulated since the last get (resets)."""
    ms = np.zeros(len(TIMING_CLASSES))
    cnt = np.zeros(len(TIMING_CLASSES), dtype=np.int64)
    _check(lib().npc_context_get_timing(ctx.h, ms.ctypes.data_as(C.c_void_p), cnt.ctypes.data_as(C.c_void_p)))
    return {c: (float(m), int(k)) for c, m, k in zip(TIMING_CLASSES, ms, cnt)}


class Operator:
    def __init__(self, ctx, handle, n_local, keep):
        self.ctx, self.h, self.n_local, self._keep = ctx, handle, n_local, keep

    def close(self):
        if self.h:
            lib().npc_destroy_operator(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def npc_create_operator(ctx: Context, kind, *, n_local, n_global=0, row_begin=0, rowptr=None, colidx=None,
                        vals=None, sell_C=0, sell_sigma=0, dim=3, nx=0, ny=0, nz_global=1, z_begin=0,
                        nz_local=None, diag=0.0, offdiag=0.0, c=None, b_rows_global=0, b_row_begin=0,
                        b_n_local=0, b_rowptr=None, b_colidx=None, b_vals=None, d=None, apply=None,
                        user=None, dfn=None) -> Operator:
    """Host arrays (numpy) are copied by the library.  `apply` (callback kind) is a Python
    callable (x_ptr, y_ptr, stream_ptr) -> int, kept alive by the returned Operator."""
    desc = OperatorDesc()
    desc.kind = KIND[kind] if isinstance(kind, str) else int(kind)
    desc.n_local, desc.n_global, desc.row_begin = int(n_local), int(n_global), int(row_begin)
    keep = []

    def arr(a, dt):
        if a is None:
            return None
        a2, p = _host(a, dt)
        keep.append(a2)
        return p

    desc.rowptr, desc.colidx, desc.vals = arr(rowptr, np.int32), arr(colidx, np.int32), arr(vals, np.float64)
    desc.sell_C, desc.sell_sigma = int(sell_C), int(sell_sigma)
    desc.stencil_dim, desc.nx, desc.ny, desc.nz_global = int(dim), int(nx), int(ny), int(nz_global)
    desc.z_begin = int(z_begin)
    desc.nz_local = int(nz_global if nz_local is None else nz_local)
    desc.diag, desc.offdiag = float(diag), float(offdiag)
    desc.c = arr(c, np.float64)
    desc.b_rows_global, desc.b_row_begin, desc.b_n_local = int(b_rows_global), int(b_row_begin), int(b_n_local)
    desc.b_rowptr, desc.b_colidx = arr(b_rowptr, np.int32), arr(b_colidx, np.int32)
    desc.b_vals, desc.d = arr(b_vals, np.float64), arr(d, np.float64)
    if dfn is not None:
        # dfn = dict(nh, nblk, hblk, A=(rowptr, colidx, vals), Gh=..., C=..., B=..., Gu=..., alpha, scaled)
        desc.dfn_nh, desc.dfn_nblk = int(dfn["nh"]), int(dfn["nblk"])
        desc.dfn_hblk = arr(dfn["hblk"], np.int32)
        for key, pre in (("A", "a"), ("Gh", "gh"), ("C", "c"), ("B", "bm"), ("Gu", "gu")):
            rp, ci, v = dfn[key]
            setattr(desc, pre + "_rowptr", arr(rp, np.int32))
            setattr(desc, pre + "_colidx", arr(ci, np.int32))
            setattr(desc, pre + "_vals", arr(v, np.float64))
        desc.dfn_alpha, desc.dfn_scaled = float(dfn["alpha"]), int(dfn.get("scaled", 1))
    if apply is not None:
        cb = APPLY_FN(lambda u, x, y, s: int(apply(x, y, s)))
        keep.append(cb)
        desc.apply = cb
        desc.user = user
    h = C.c_void_p()
    _check(lib().npc_create_operator(ctx.h, C.byref(desc), C.byref(h)))
    return Operator(ctx, h, int(n_local), keep if apply is not None else [])


def npc_operator_matrix_bytes(op: Operator) -> float:
    b = C.c_double()
    _check(lib().npc_operator_matrix_bytes(op.h, C.byref(b)))
    return b.value


def npc_apply_operator(op: Operator, x, y):
    _check(lib().npc_apply_operator(op.h, _ptr(x), _ptr(y)))


NPC_DEFAULT_SEED = 0x5EED


def npc_estimate_spectrum(op: Operator, nsteps: int = 20, v0=None, seed: int = NPC_DEFAULT_SEED):
    lo, hi = C.c_double(), C.c_double()
    _check(lib().npc_estimate_spectrum(op.h, int(nsteps), _ptr(v0), int(seed), C.byref(lo), C.byref(hi)))
    return lo.value, hi.value


def npc_estimate_spectrum_ex(op: Operator, nsteps: int = 20, v0=None, seed: int = NPC_DEFAULT_SEED):
    """-> dict(theta_min, theta_max, rho, steps)."""
    out = np.zeros(4)
    _check(lib().npc_estimate_spectrum_ex(op.h, int(nsteps), _ptr(v0), int(seed), out.ctypes.data_as(C.c_void_p)))
    return dict(theta_min=out[0], theta_max=out[1], rho=out[2], steps=int(out[3]))


class Poly:
    def __init__(self, op, handle, degree, lmin, lmax, xi):
        self.op, self.h, self.degree, self.lmin, self.lmax, self.xi = op, handle, degree, lmin, lmax, xi

    def close(self):
        if self.h:
            lib().npc_destroy_poly(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def npc_set_poly(op: Operator, degree: int, lmin: float, lmax: float, xi: float = 0.0) -> Poly:
    h = C.c_void_p()
    _check(lib().npc_set_poly(op.h, int(degree), float(lmin), float(lmax), float(xi), C.byref(h)))
    return Poly(op, h, degree, lmin, lmax, xi)


def npc_set_poly_newton(op: Operator, nlev: int, lmin: float, lmax: float, xi: float = 0.0) -> Poly:
    """Newton variant (Alg. 1), degree 2^nlev - 1."""
    h = C.c_void_p()
    _check(lib().npc_set_poly_newton(op.h, int(nlev), float(lmin), float(lmax), float(xi), C.byref(h)))
    return Poly(op, h, (1 << nlev) - 1, lmin, lmax, xi)


def npc_poly_set_lowrank(poly: Poly, V=None):
    """Low-rank correction P = p_k(A) + V (V^T A V)^{-1} V^T.  V: fp64 CUDA tensor of shape
    (p, n_local) (vector j = V[j]), or None / p = 0 to remove it."""
    if V is None:
        _check(lib().npc_poly_set_lowrank(poly.h, 0, None))
        return
    assert V.dim() == 2, "V must be (p, n_local)"
    _check(lib().npc_poly_set_lowrank(poly.h, int(V.shape[0]), _ptr(V)))
    poly._lowrank_V = V  # not needed by the library (it copies); kept for introspection


def npc_ritz_vectors(op: Operator, nsteps: int, p: int, v0=None):
    """-> (theta numpy[p], V CUDA tensor (p, n_local)): Ritz pairs of the p smallest Ritz values
    of an nsteps-step fully reorthogonalised Lanczos."""
    import torch
    V = torch.empty((p, op.n_local), dtype=torch.float64, device="cuda")
    th = (C.c_double * p)()
    _check(lib().npc_ritz_vectors(op.h, int(nsteps), int(p), _ptr(v0), _ptr(V), th))
    return np.array(th[:], dtype=np.float64), V


def npc_apply_poly(poly: Poly, r, z):
    _check(lib().npc_apply_poly(poly.h, _ptr(r), _ptr(z)))


def npc_pcg_solve(poly: Poly | None, op: Operator, b, x, tol: float, maxit: int, history: bool = False,
                  raise_on_error: bool = True) -> dict:
    st = PcgStats()
    hist = None
    if history:
        hist = np.zeros(maxit + 1)
        st.history = hist.ctypes.data_as(C.POINTER(C.c_double))
    code = lib().npc_pcg_solve(poly.h if poly is not None else None, op.h, _ptr(b), _ptr(x), float(tol),
                               int(maxit), C.byref(st))
    out = dict(status=STATUS.get(code, code), iters=st.iters, converged=bool(st.converged),
               op_applications=st.op_applications, reductions=st.reductions,
               relres_recursive=st.relres_recursive, relres_true=st.relres_true,
               setup_seconds=st.setup_seconds, solve_seconds=st.solve_seconds)
    if history:
        out["history"] = hist[: st.iters + 1]
    if raise_on_error and code not in (0,):
        raise NpcError(code, lib().npc_last_error(op.ctx.h if hasattr(op, "ctx") else None).decode(errors="replace")
                       + f" (stats {out})")
    return out


def npc_poly_coefficients(degree: int, lmin: float, lmax: float, xi: float):
    tb, dl, sg = C.c_double(), C.c_double(), C.c_double()
    coef = np.zeros(4 * max(degree, 1))
    _check(lib().npc_poly_coefficients(int(degree), float(lmin), float(lmax), float(xi), C.byref(tb), C.byref(dl),
                                       C.byref(sg), coef.ctypes.data_as(C.c_void_p)))
    return tb.value, dl.value, sg.value, coef[: 4 * degree].reshape(degree, 4)


def npc_halo_plan(rowptr, colidx, row_starts, rank: int):
    rp, prp = _host(rowptr, np.int32)
    ci, pci = _host(colidx if colidx is not None and len(colidx) else np.zeros(1), np.int32)
    rs, prs = _host(row_starts, np.int64)
    nranks = len(rs) - 1
    n_local = len(rp) - 1
    ng = C.c_int(0)
    _check(lib().npc_halo_plan(n_local, prp, pci, nranks, prs, rank, C.byref(ng), None, None))
    ids = np.zeros(max(ng.value, 1), dtype=np.int64)
    counts = np.zeros(nranks, dtype=np.int32)
    cap = C.c_int(ng.value)
    _check(lib().npc_halo_plan(n_local, prp, pci, nranks, prs, rank, C.byref(cap), ids.ctypes.data_as(C.c_void_p),
                               counts.ctypes.data_as(C.c_void_p)))
    return ids[: ng.value], counts


PATTERN_INFO = ("pattern", "ring", "tiles", "ring_tiles", "max_copies", "stage_bytes", "ring_table_words",
                "own_values")


def npc_pattern_check(rowptr, colidx, vals, x):
    """Host-only layout check of the CSR pattern form (include/npc.h): returns (y = A x evaluated
    by replaying the ring layout on the host, info dict)."""
    rp, prp = _host(rowptr, np.int32)
    n = len(rp) - 1
    ci, pci = _host(colidx if len(colidx) else np.zeros(1), np.int32)
    va, pva = _host(vals if len(vals) else np.zeros(1), np.float64)
    xx, pxx = _host(x, np.float64)
    y = np.zeros(max(n, 1))
    info = np.zeros(8, dtype=np.int64)
    _check(lib().npc_pattern_check(n, prp, pci, pva, pxx, y.ctypes.data_as(C.c_void_p),
                                   info.ctypes.data_as(C.c_void_p)))
    return y[:n], dict(zip(PATTERN_INFO, (int(v) for v in info)))


# ---------------------------------------------------------------- convenience (marshalling)
def create_from_workload(ctx: Context, w: dict, kind: str | None = None) -> Operator:
    """Create an operator from a workloads/ dict (single rank).  kind overrides w['kind']
    (e.g. 'sell' for a CSR workload)."""
    k = kind or w["kind"]
    if k in ("csr", "sell"):
        return npc_create_operator(ctx, k, n_local=w["n"], n_global=w["n"], rowptr=w["rowptr"], colidx=w["colidx"],
                                   vals=w["vals"], sell_C=w.get("sell_C", 32), sell_sigma=w.get("sell_sigma", 256))
    if k == "stencil":
        nz = w.get("nz", 1) if w["dim"] == 3 else 1
        return npc_create_operator(ctx, "stencil", n_local=w["n"], n_global=w["n"], dim=w["dim"], nx=w["nx"],
                                   ny=w["ny"], nz_global=nz, nz_local=nz, diag=w["diag"], offdiag=w["offdiag"])
    if k == "schur":
        return npc_create_operator(ctx, "schur", n_local=w["n"], n_global=w["n"], c=w["c"], b_rows_global=w["nb"],
                                   b_n_local=w["nb"], b_rowptr=w["browptr"], b_colidx=w["bcolidx"],
                                   b_vals=w["bvals"], d=w["d"])
    if k == "dfn":
        return npc_create_operator(ctx, "dfn", n_local=w["n"], n_global=w["n"],
                                   dfn=dict(nh=w["nh"], nblk=w["nf"], hblk=w["hblk"], A=w["A"], Gh=w["Gh"], C=w["C"],
                                            B=w["B"], Gu=w["Gu"], alpha=w["alpha"], scaled=w.get("scaled", 1)))
    raise ValueError(k)
