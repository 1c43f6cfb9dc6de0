"""Sparse kernels and primitive solvers on the device (drop-in for dppflow.linalg).

Every entry point runs on the B200 through libdpp (reference linalg.py):
  spmv            -> CSR SpMV kernel                 (linalg.py:27-32)
  gmres           -> device GMRES(m), host Givens     (linalg.py:65-165)
  ilu0/apply_ilu0 -> sync-free ILU(0) + SpTRSV        (linalg.py:178-227)
  diag_lump       -> diagonal extraction              (linalg.py:234-241)
  schur_selfp     -> ordered SpGEMM, scipy rounding   (linalg.py:244-254)
  amg_setup/vcycle-> device smoothed aggregation AMG  (linalg.py:279-400)
Inputs may be scipy matrices (uploaded) or device handles; results that the
reference returns as scipy matrices are exported back to scipy.
"""

from __future__ import annotations

import ctypes as ct
from dataclasses import dataclass, field

import numpy as np
import scipy.io
import scipy.sparse as sp

from . import _native as N
from ._native import ZeroPivotError  # noqa: F401  (public name, reference linalg.py:23)
from .device import DeviceCsr, as_device

CsrMatrix = sp.csr_matrix


def spmv(A, x: np.ndarray) -> np.ndarray:
    """y = A @ x on the device with the reference's shape check."""
    x = np.asarray(x)
    if A.shape[1] != x.shape[0]:
        raise ValueError(f"dimension mismatch: {A.shape} @ {x.shape}")
    return as_device(A) @ x


def write_matrix_market(path, obj) -> None:
    if sp.issparse(obj) or isinstance(obj, DeviceCsr):
        obj = obj.to_scipy() if isinstance(obj, DeviceCsr) else obj
        scipy.io.mmwrite(str(path), sp.coo_matrix(obj))
        return
    arr = np.asarray(obj)
    scipy.io.mmwrite(str(path), arr.reshape(-1, 1) if arr.ndim == 1 else arr)


def read_matrix_market(path):
    out = scipy.io.mmread(str(path))
    if sp.issparse(out):
        return out.tocsr()
    arr = np.asarray(out)
    return arr.ravel() if 1 in arr.shape else arr


# ----------------------------------------------------------------------------- GMRES

@dataclass
class KrylovStats:
    iterations: int
    relative_residual: float
    converged: bool
    wall_time_s: float
    reason: str = "converged"
    history: list = field(default_factory=list)
    cycles: int = 0
    pc_applies: int = 0
    matvecs: int = 0


_REASONS = {0: "converged", 1: "max_iter", 2: "stagnation"}


def _stats(s: N.KrylovStatsC, hist) -> KrylovStats:
    return KrylovStats(s.iterations, float(s.relative_residual), bool(s.converged),
                       float(s.wall_time_s), _REASONS[s.reason], list(hist), s.cycles,
                       s.pc_applies, s.matvecs)


def _host_cb(fn, n):
    def cb(inp, out, _u):
        x = np.ctypeslib.as_array(inp, shape=(n,)).copy()
        y = np.asarray(fn(x), dtype=np.float64)
        ct.memmove(out, y.ctypes.data, 8 * n)
    return N.APPLY_FN(cb)


def gmres(operator, b: np.ndarray, *, preconditioner=None, rtol: float = 1e-7,
          max_iter: int = 1000, restart: int = 30, x0: np.ndarray | None = None):
    """Left-preconditioned restarted GMRES on the device (reference linalg.py:65-165).

    `operator`: scipy / dense / DeviceCsr matrix (device SpMV) or a callable
    (evaluated on the host through a callback).  `preconditioner`: a device
    Preconditioner (blocksolve), a callable (host callback), or None.
    """
    from .blocksolve import Preconditioner
    b = N.f64(b)
    n = b.shape[0]
    A = Acb = None
    if callable(operator) and not (sp.issparse(operator) or isinstance(operator, (DeviceCsr, np.ndarray))):
        Acb = _host_cb(operator, n)
    else:
        A = as_device(operator)
    pc = pcb = None
    if isinstance(preconditioner, Preconditioner):
        pc = preconditioner.handle()
    elif preconditioner is not None:
        pcb = _host_cb(preconditioner, n)
    x = np.empty(n)
    x0a = None if x0 is None else N.f64(x0)
    st = N.KrylovStatsC()
    hist = np.empty(max(int(max_iter), 1))
    null_cb = N.APPLY_FN()
    N.call("dpp_gmres", N.ctx(), None if A is None else A.h, Acb or null_cb, None, pc,
           pcb or null_cb, None, n, N.ptr(b), N.ptr(x0a), N.ptr(x), float(rtol), int(max_iter),
           int(restart), ct.byref(st), N.ptr(hist), len(hist))
    return x, _stats(st, hist[:st.iterations])


# ----------------------------------------------------------------------------- ILU(0)

class Ilu0Factorization:
    """ILU(0) factors held on the device; L/U exported to scipy on access."""

    def __init__(self, handle, n):
        self.h = handle
        self.n = n
        self._L = self._U = None

    def _export(self):
        lh, uh = ct.c_void_p(), ct.c_void_p()
        N.call("dpp_ilu0_factors", self.h, ct.byref(lh), ct.byref(uh))
        self._L, self._U = DeviceCsr(lh).to_scipy(), DeviceCsr(uh).to_scipy()

    @property
    def L(self) -> sp.csr_matrix:
        if self._L is None:
            self._export()
        return self._L

    @property
    def U(self) -> sp.csr_matrix:
        if self._U is None:
            self._export()
        return self._U

    def __del__(self):
        if getattr(self, "h", None) is not None and N._lib is not None:
            N.lib().dpp_ilu0_destroy(self.h)
            self.h = None


def ilu0(A) -> Ilu0Factorization:
    """Zero-fill incomplete LU on A's stored pattern (reference linalg.py:178-222)."""
    if A.shape[0] != A.shape[1]:
        raise ValueError("ilu0 requires a square matrix")
    d = as_device(A)
    h = ct.c_void_p()
    N.call("dpp_ilu0_create", N.ctx(), d.h, ct.byref(h))
    return Ilu0Factorization(h, A.shape[0])


def apply_ilu0(fact: Ilu0Factorization, r: np.ndarray) -> np.ndarray:
    r = N.f64(r)
    z = np.empty(fact.n)
    N.call("dpp_ilu0_apply", fact.h, N.ptr(r), N.ptr(z))
    return z


# ----------------------------------------------------------------------------- selfp

def diag_lump(A) -> np.ndarray:
    if A.shape[0] != A.shape[1]:
        raise ValueError("diag_lump requires a square matrix")
    d = np.empty(A.shape[0])
    dA = as_device(A)          # keep the device copy alive across the call
    N.call("dpp_diag", N.ctx(), dA.h, N.ptr(d))
    if np.any(d == 0.0):
        raise ZeroPivotError("zero diagonal entry in diag_lump")
    return d


def schur_selfp(D, C, diagA: np.ndarray, B) -> sp.csr_matrix:
    """S = D - C diag(diagA)^-1 B with scipy's accumulation order (bitwise)."""
    diagA = N.f64(diagA)
    if np.any(diagA == 0.0):
        raise ZeroPivotError("zero entry in diagA")
    if C.shape[1] != len(diagA) or B.shape[0] != len(diagA) or D.shape != (C.shape[0], B.shape[1]):
        raise ValueError("schur_selfp: non-conforming block dimensions")
    h = ct.c_void_p()
    dD, dC, dB = as_device(D), as_device(C), as_device(B)
    N.call("dpp_schur_selfp", N.ctx(), dD.h, dC.h, N.ptr(diagA), dB.h, ct.byref(h))
    return DeviceCsr(h).to_scipy()


# ----------------------------------------------------------------------------- AMG

@dataclass
class AmgLevel:
    A: sp.csr_matrix
    P: sp.csr_matrix | None
    lower: sp.csr_matrix | None
    upper: sp.csr_matrix | None
    aggregates: np.ndarray | None = None
    rho: float | None = None


class AmgHierarchy:
    """Device hierarchy; levels exported to scipy on access (reference linalg.py:265-276)."""

    def __init__(self, handle):
        self.h = handle
        n = ct.c_int()
        N.call("dpp_amg_levels", handle, ct.byref(n))
        self._count = n.value
        self._levels = None
        self.coarse_lu = None   # the coarsest solve is a device dense inverse

    @property
    def level_count(self) -> int:
        return self._count

    @property
    def levels(self):
        if self._levels is None:
            out = []
            for l in range(self._count):
                a, p = ct.c_void_p(), ct.c_void_p()
                rho = ct.c_double()
                coarse = l + 1 == self._count
                N.call("dpp_amg_level", self.h, l, ct.byref(a), ct.byref(p), None, ct.byref(rho))
                A0 = DeviceCsr(a, owner=self).to_scipy()
                if not coarse:
                    agg = np.empty(A0.shape[0], dtype=np.int64)
                    N.call("dpp_amg_level", self.h, l, None, None, N.ptr(agg), None)
                    P = DeviceCsr(p, owner=self).to_scipy()
                    nl = AmgLevel(A0, P, sp.tril(A0, k=0, format="csr"), sp.triu(A0, k=0, format="csr"),
                                  agg, float(rho.value))
                else:
                    nl = AmgLevel(A0, None, None, None)
                out.append(nl)
            self._levels = out
        return self._levels

    def __del__(self):
        if getattr(self, "h", None) is not None and N._lib is not None:
            N.lib().dpp_amg_destroy(self.h)
            self.h = None


def strength_aggregates(A, theta: float = 0.5, *, path: str = "auto") -> np.ndarray:
    """Greedy aggregation over the strength graph (reference linalg.py:279-324
    _strength_aggregates): int64 aggregate id per row.  path: "auto" (device passes from
    32768 rows), "host" (greedy loop over the device-built strength graph) or "device"."""
    if A.shape[0] != A.shape[1]:
        raise ValueError("aggregation requires a square matrix")
    dA = as_device(A)
    agg = np.empty(A.shape[0], dtype=np.int64)
    nagg = ct.c_int64()
    N.call("dpp_strength_aggregates", N.ctx(), dA.h, float(theta), {"auto": 0, "host": 1, "device": 2}[path],
           N.ptr(agg), ct.byref(nagg))
    return agg


def amg_setup(A, *, theta: float = 0.5, omega: float = 2.0 / 3.0, max_coarse: int = 64,
              max_levels: int = 25) -> AmgHierarchy:
    """Smoothed-aggregation hierarchy on the device (reference linalg.py:341-380)."""
    if A.shape[0] != A.shape[1]:
        raise ValueError("amg_setup requires a square matrix")
    h = ct.c_void_p()
    dA = as_device(A)
    N.call("dpp_amg_create", N.ctx(), dA.h, float(theta), float(omega), int(max_coarse),
           int(max_levels), N.RANDN, None, ct.byref(h))
    return AmgHierarchy(h)


def amg_vcycle(hierarchy: AmgHierarchy, r: np.ndarray) -> np.ndarray:
    """One V(1,1) cycle with zero initial guess (reference linalg.py:398-400)."""
    r = N.f64(r)
    z = np.empty_like(r)
    N.call("dpp_amg_vcycle", hierarchy.h, N.ptr(r), N.ptr(z))
    return z
