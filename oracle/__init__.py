"""ctypes wrapper of the CPU fp64 oracle (oracle/npc_oracle.c).

TEST INFRASTRUCTURE ONLY: importable from tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs.  The product path (paper_2208_01339_b200) never
imports this package, and this package never imports the product.

Every function names the PAPER.md passage it follows; see npc_oracle.c for the pins.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "npc_oracle.c")
_LIB = os.path.join(_HERE, "liborc.so")
CFLAGS = ["-O2", "-fno-fast-math", "-ffp-contract=off", "-fopenmp", "-shared", "-fPIC", "-std=c11"]


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (plain C, no GPU)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *CFLAGS, "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


class _Op(C.Structure):
    _fields_ = [
        ("kind", C.c_int), ("n", C.c_long),
        ("rowptr", C.c_void_p), ("colidx", C.c_void_p), ("vals", C.c_void_p),
        ("dim", C.c_int), ("nx", C.c_int), ("ny", C.c_int), ("nz", C.c_int),
        ("diag", C.c_double), ("offdiag", C.c_double),
        ("c", C.c_void_p), ("nb", C.c_long),
        ("browptr", C.c_void_p), ("bcolidx", C.c_void_p), ("bvals", C.c_void_p), ("d", C.c_void_p),
        ("tmp", C.c_void_p),
        ("nh", C.c_long), ("nblk", C.c_int), ("hblk", C.c_void_p),
        ("Arp", C.c_void_p), ("Aci", C.c_void_p), ("Av", C.c_void_p),
        ("Ghrp", C.c_void_p), ("Ghci", C.c_void_p), ("Ghv", C.c_void_p),
        ("Crp", C.c_void_p), ("Cci", C.c_void_p), ("Cv", C.c_void_p),
        ("Brp", C.c_void_p), ("Bci", C.c_void_p), ("Bv", C.c_void_p),
        ("Gurp", C.c_void_p), ("Guci", C.c_void_p), ("Guv", C.c_void_p),
        ("alpha", C.c_double), ("scaled", C.c_int),
        ("Lfac", C.c_void_p), ("Loff", C.c_void_p), ("ds", C.c_void_p), ("dwork", C.c_void_p),
    ]


class _Stats(C.Structure):
    _fields_ = [("iters", C.c_int), ("converged", C.c_int), ("breakdown", C.c_int),
                ("mvp", C.c_longlong), ("ddot", C.c_longlong),
                ("relres_recursive", C.c_double), ("relres_true", C.c_double), ("true_checks", C.c_int)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        P = C.c_void_p
        D = C.c_double
        _lib.orc_op_apply.argtypes = [C.POINTER(_Op), P, P]
        _lib.orc_cheb_params.argtypes = [D, D, D, P, P, P]
        _lib.orc_cheb_rho.argtypes = [D, C.c_int, P]
        _lib.orc_cheb_apply.argtypes = [C.POINTER(_Op), C.c_int, D, D, D, P, P, P]
        _lib.orc_newton_zeta.argtypes = [D, D, D, C.c_int, P]
        _lib.orc_newton_apply.argtypes = [C.POINTER(_Op), C.c_int, D, D, D, P, P, P]
        _lib.orc_lanczos.argtypes = [C.POINTER(_Op), C.c_int, P, P, P, P]
        _lib.orc_pcg.argtypes = [C.POINTER(_Op), C.c_int, D, D, D, P, P, D, C.c_int, P, C.POINTER(_Stats),
                                 C.c_int, P, P]
        _lib.orc_lowrank_setup.argtypes = [C.POINTER(_Op), C.c_int, P, P, P]
        _lib.orc_lowrank_apply.argtypes = [C.POINTER(_Op), C.c_int, D, D, D, C.c_int, P, P, P, P, P]
        _lib.orc_lanczos_full.argtypes = [C.POINTER(_Op), C.c_int, P, P, P, P, P]
        _lib.orc_num_threads.restype = C.c_int
        _lib.orc_dfn_setup.argtypes = [C.POINTER(_Op)]
        _lib.orc_dfn_free.argtypes = [C.POINTER(_Op)]
    return _lib


def _p(a):
    return a.ctypes.data_as(C.c_void_p) if a is not None else None


class Operator:
    """Holds the numpy arrays alive and the C descriptor of an operator (O1)."""

    def __init__(self, w: dict, scaled: bool = True):
        """scaled (DFN only): the operator is D_S^{-1/2} S_u D_S^{-1/2},
        the one the polynomial is applied to; False gives S_u itself."""
        self.w = w
        self._dfn = False
        op = _Op()
        kind = w["kind"]
        op.n = int(w["n"])
        self._keep = []

        def arr(a, dt):
            a = np.ascontiguousarray(a, dtype=dt)
            self._keep.append(a)
            return _p(a)

        if kind == "csr":
            op.kind = 0
            op.rowptr = arr(w["rowptr"], np.int32)
            op.colidx = arr(w["colidx"], np.int32)
            op.vals = arr(w["vals"], np.float64)
        elif kind == "stencil":
            op.kind = 1
            op.dim, op.nx, op.ny = int(w["dim"]), int(w["nx"]), int(w["ny"])
            op.nz = int(w.get("nz", 1))
            op.diag, op.offdiag = float(w["diag"]), float(w["offdiag"])
        elif kind == "schur":
            op.kind = 2
            op.c = arr(w["c"], np.float64)
            op.nb = int(w["nb"])
            op.browptr = arr(w["browptr"], np.int32)
            op.bcolidx = arr(w["bcolidx"], np.int32)
            op.bvals = arr(w["bvals"], np.float64)
            op.d = arr(w["d"], np.float64)
            op.tmp = arr(np.zeros(op.nb), np.float64)
        elif kind == "dfn":
            op.kind = 3
            op.nh, op.nblk = int(w["nh"]), int(w["nf"])
            op.hblk = arr(w["hblk"], np.int32)
            for key, (rp, ci, v) in (("A", w["A"]), ("Gh", w["Gh"]), ("C", w["C"]), ("B", w["B"]),
                                     ("Gu", w["Gu"])):
                setattr(op, key + "rp", arr(rp, np.int32))
                setattr(op, key + "ci", arr(ci, np.int32))
                setattr(op, key + "v", arr(v, np.float64))
            op.alpha = float(w["alpha"])
            op.scaled = 1 if scaled else 0
        else:
            raise ValueError(kind)
        self.op = op
        self.n = op.n
        if kind == "dfn":
            st = lib().orc_dfn_setup(C.byref(op))
            self._dfn = True
            if st:
                raise ValueError(f"orc_dfn_setup failed ({st}: -1 A block not SPD, -2 A not block-diagonal, "
                                 f"-3 diag(S_u) <= 0)")

    def dfn_diag(self):
        """D_S = diag(S_u) by Alg. 4, computed at setup."""
        assert self._dfn
        return np.ctypeslib.as_array(C.cast(self.op.ds, C.POINTER(C.c_double)), shape=(self.n,)).copy()

    def __del__(self):
        if getattr(self, "_dfn", False) and _lib is not None:
            _lib.orc_dfn_free(C.byref(self.op))
            self._dfn = False

    def apply(self, x):
        """y = A x (O1)."""
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.empty(self.n)
        assert lib().orc_op_apply(C.byref(self.op), _p(x), _p(y)) == 0
        return y


def cheb_params(alpha, beta, xi):
    """(theta_bar, delta, sigma): PAPER.md:240-241 with Eq. thetamod, reading A1."""
    t, d, s = C.c_double(), C.c_double(), C.c_double()
    st = lib().orc_cheb_params(alpha, beta, xi, C.byref(t), C.byref(d), C.byref(s))
    if st:
        raise ValueError(f"invalid interval ({st})")
    return t.value, d.value, s.value


def cheb_rho(sigma, m):
    """rho_0..rho_m by Eq. rhocheb."""
    rho = np.empty(m + 1)
    lib().orc_cheb_rho(sigma, m, _p(rho))
    return rho


def cheb_apply(op: Operator, m, alpha, beta, xi, r):
    """p_m(A) r by Alg. 2 verbatim."""
    r = np.ascontiguousarray(r, dtype=np.float64)
    out = np.empty(op.n)
    work = np.empty(3 * op.n)
    st = lib().orc_cheb_apply(C.byref(op.op), m, alpha, beta, xi, _p(r), _p(out), _p(work))
    if st:
        raise ValueError(f"cheb_apply failed ({st})")
    return out


def newton_zeta(alpha, beta, xi, nlev):
    z = np.empty(nlev + 1)
    assert lib().orc_newton_zeta(alpha, beta, xi, nlev, _p(z)) == 0
    return z


def newton_apply(op: Operator, nlev, alpha, beta, xi, r):
    """P_nlev r by Alg. 1 step 4, zeta_1 with alpha' = theta_bar - delta."""
    r = np.ascontiguousarray(r, dtype=np.float64)
    out = np.empty(op.n)
    work = np.empty(3 * op.n * max(nlev, 1) + op.n)
    assert lib().orc_newton_apply(C.byref(op.op), nlev, alpha, beta, xi, _p(r), _p(out), _p(work)) == 0
    return out


def lanczos(op: Operator, m, v0):
    """m-step Lanczos from v0 (O2). Returns (alphas, betas) of T_s (s = steps taken)."""
    v0 = np.ascontiguousarray(v0, dtype=np.float64)
    a = np.zeros(m)
    b = np.zeros(m)
    work = np.empty(3 * op.n)
    s = lib().orc_lanczos(C.byref(op.op), m, _p(v0), _p(a), _p(b), _p(work))
    assert s >= 0
    return a[:s], b[:s]


def ritz_extremes(alphas, betas):
    """Extreme eigenvalues of the Lanczos tridiagonal T_s (LAPACK via scipy: a library
    primitive standing for 'eigenvalues of T_m')."""
    from scipy.linalg import eigvalsh_tridiagonal
    ev = eigvalsh_tridiagonal(alphas, betas[: len(alphas) - 1])
    return float(ev[0]), float(ev[-1])


def ritz_upper(alphas, betas):
    """(theta_max, rho): the largest Ritz value of T_s and its residual norm
    ||A y - theta y|| = beta_s |e_s^T s| (s = normalised eigenvector of T_s for theta_max;
    beta_s = the last Lanczos beta, 0 on an invariant subspace).  theta_max + rho is the
    upper estimate of lambda_max used for the polynomial interval (reading A11)."""
    from scipy.linalg import eigh_tridiagonal
    s = len(alphas)
    ev, vec = eigh_tridiagonal(alphas, betas[: s - 1], select="i", select_range=(s - 1, s - 1))
    return float(ev[0]), float(abs(betas[s - 1]) * abs(vec[-1, 0]))


def estimate_spectrum(op: Operator, m, v0):
    """(lmin, lmax) for the polynomial: lmin = smallest Ritz value, lmax = theta_max + rho."""
    a, b = lanczos(op, m, v0)
    lo, _ = ritz_extremes(a, b)
    th, rho = ritz_upper(a, b)
    return lo, th + rho


class LowRank:
    """V (n x p) and the Cholesky factor L of V^T A V: the low-rank spectral correction
    P = P_0 + V (V^T A V)^{-1} V^T of PAPER.md:483-508 (O8)."""

    def __init__(self, op: Operator, V):
        V = np.asarray(V, dtype=np.float64)
        if V.ndim == 1:
            V = V[:, None]
        assert V.shape[0] == op.n
        self.p = V.shape[1]
        self.Vc = np.ascontiguousarray(V.T)  # column j contiguous (column-major n x p)
        self.L = np.zeros((self.p, self.p))
        work = np.empty(op.n)
        if lib().orc_lowrank_setup(C.byref(op.op), self.p, _p(self.Vc), _p(self.L), _p(work)) != 0:
            raise ValueError("V^T A V is not SPD")


def lowrank_apply(op: Operator, m, alpha, beta, xi, lr: LowRank, r):
    """(p_m(A) + V (V^T A V)^{-1} V^T) r  (O8)."""
    r = np.ascontiguousarray(r, dtype=np.float64)
    out = np.empty(op.n)
    work = np.empty(3 * op.n)
    st = lib().orc_lowrank_apply(C.byref(op.op), m, alpha, beta, xi, lr.p, _p(lr.Vc), _p(lr.L), _p(r), _p(out),
                                 _p(work))
    if st:
        raise ValueError(f"lowrank_apply failed ({st})")
    return out


def lanczos_full(op: Operator, m, v0):
    """m-step Lanczos with full reorthogonalisation; returns (alphas, betas, Q) with Q the
    n x (s+1) basis (s = steps taken; the last column is valid only if beta_s > 0)."""
    v0 = np.ascontiguousarray(v0, dtype=np.float64)
    a = np.zeros(m)
    b = np.zeros(m)
    Q = np.zeros((m + 1, op.n))
    w = np.empty(op.n)
    s = lib().orc_lanczos_full(C.byref(op.op), m, _p(v0), _p(a), _p(b), _p(Q), _p(w))
    assert s >= 0
    return a[:s], b[:s], Q[: s + 1].T


def ritz_vectors(op: Operator, m, p, v0):
    """(theta[p], V n x p): Ritz pairs of the p smallest Ritz values of the fully
    reorthogonalised m-step Lanczos (the tridiagonal eigenproblem via LAPACK through scipy,
    a library primitive)."""
    from scipy.linalg import eigh_tridiagonal
    a, b, Q = lanczos_full(op, m, v0)
    s = len(a)
    ev, S = eigh_tridiagonal(a, b[: s - 1])
    return ev[:p], Q[:, :s] @ S[:, :p]


def pcg(op: Operator, b, m, alpha=None, beta=None, xi=0.0, tol=1e-8, maxit=10000, x0=None,
        history=False, lowrank: LowRank | None = None):
    """Textbook PCG (O5) preconditioned by p_m(A) (m < 0: none), plus the low-rank
    correction V (V^T A V)^{-1} V^T when `lowrank` is given (O8).  Returns (x, stats dict)."""
    b = np.ascontiguousarray(b, dtype=np.float64)
    x = np.zeros(op.n) if x0 is None else np.array(x0, dtype=np.float64)
    hist = np.zeros(maxit + 1) if history else None
    st = _Stats()
    if m >= 0:
        assert alpha is not None and beta is not None
    lr_p, lr_V, lr_L = (lowrank.p, _p(lowrank.Vc), _p(lowrank.L)) if lowrank is not None else (0, None, None)
    lib().orc_pcg(C.byref(op.op), m, float(alpha or 0.0), float(beta or 0.0), float(xi), _p(b), _p(x),
                  tol, maxit, _p(hist), C.byref(st), lr_p, lr_V, lr_L)
    out = dict(iters=st.iters, converged=bool(st.converged), breakdown=bool(st.breakdown),
               mvp=st.mvp, ddot=st.ddot, relres_recursive=st.relres_recursive,
               relres_true=st.relres_true, true_checks=st.true_checks)
    if history:
        out["history"] = hist[: st.iters + 1]
    return x, out


def num_threads() -> int:
    return int(lib().orc_num_threads())
