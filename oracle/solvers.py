"""Oracle: GMRES(m), ILU(0), selfp Schur, aggregation AMG, split-tree composition.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Restates reference linalg.py:
  :65-165   left-preconditioned restarted GMRES (MGS, Givens, true-residual exit,
            stagnation factor 0.9999, happy breakdown 1e-14)
  :178-227  ILU(0) (numeric loop in oracle/csrc/oracle_kernels.c) and its apply
  :234-254  diag lump and the selfp triple product
  :279-400  smoothed-aggregation AMG setup (aggregation loop in C) and V(1,1)
and reference blocksolve.py:43-86 (option listings), :119-210 (parser),
:227-294 (recursive additive / Schur-full composition), :346-360 (solve).
Arithmetic goes through the same numpy / scipy kernels as the reference so the
results are bitwise reproducible on the same host.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
import time
from dataclasses import dataclass, replace

import numpy as np
import scipy.linalg
import scipy.sparse as sp
from scipy.sparse.linalg import spsolve_triangular

from .forms import FIELDS, monolithic_view

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "liboracle.so")
_lib = None


def build_c(force=False):
    """Compile oracle/csrc into oracle/_build/liboracle.so (gcc, no FMA contraction)."""
    src = os.path.join(_HERE, "csrc", "oracle_kernels.c")
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
        os.makedirs(os.path.dirname(_LIB_PATH), exist_ok=True)
        subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fPIC", "-shared", src,
                               "-o", _LIB_PATH, "-lm"])
    return _LIB_PATH


def _c():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build_c())
        P = ctypes.c_void_p
        _lib.o_ilu0.argtypes = [ctypes.c_int, P, P, P, P]
        _lib.o_ilu0.restype = ctypes.c_int
        _lib.o_aggregate.argtypes = [ctypes.c_int, P, P, P, ctypes.c_double, P]
        _lib.o_aggregate.restype = ctypes.c_int64
    return _lib


def _ptr(a):
    return a.ctypes.data_as(ctypes.c_void_p)


class ZeroPivotError(RuntimeError):
    pass


class OptionError(ValueError):
    pass


# --------------------------------------------------------------------------- GMRES

@dataclass
class Stats:
    iterations: int
    relative_residual: float
    converged: bool
    wall_time_s: float
    reason: str = "converged"
    history: list = None
    cycles: int = 0
    pc_applies: int = 0
    matvecs: int = 0


def gmres(A, b, *, preconditioner=None, rtol=1e-7, max_iter=1000, restart=30, x0=None):
    t0 = time.perf_counter()
    cnt = {"mv": 0, "pc": 0}

    def mv(v):
        cnt["mv"] += 1
        return A(v) if callable(A) else A @ v

    def pc(v):
        cnt["pc"] += 1
        return v if preconditioner is None else preconditioner(v)

    b = np.asarray(b, dtype=float)
    n = b.shape[0]
    x = np.zeros(n) if x0 is None else np.array(x0, dtype=float)
    nb = np.linalg.norm(b)
    if nb == 0.0:
        return np.zeros(n), Stats(0, 0.0, True, time.perf_counter() - t0, history=[])
    nmb = np.linalg.norm(pc(b))
    hist, its, reason, conv, prev, cycles = [], 0, "max_iter", False, None, 0
    while its < max_iter:
        r = b - mv(x)
        rel = np.linalg.norm(r) / nb
        if rel <= rtol:
            conv, reason = True, "converged"
            break
        if prev is not None and rel >= prev * 0.9999:
            reason = "stagnation"
            break
        prev = rel
        z = pc(r)
        beta = np.linalg.norm(z)
        if beta == 0.0:
            conv, reason = True, "converged"
            break
        cycles += 1
        m = min(restart, max_iter - its)
        V = np.zeros((m + 1, n))
        H = np.zeros((m + 1, m))
        cs, sn, g = np.zeros(m), np.zeros(m), np.zeros(m + 1)
        g[0] = beta
        V[0] = z / beta
        k, happy = 0, False
        for j in range(m):
            w = pc(mv(V[j]))
            for i in range(j + 1):
                H[i, j] = V[i] @ w
                w -= H[i, j] * V[i]
            H[j + 1, j] = np.linalg.norm(w)
            if H[j + 1, j] > 1e-14 * beta:
                V[j + 1] = w / H[j + 1, j]
            else:
                happy = True
            for i in range(j):
                t = cs[i] * H[i, j] + sn[i] * H[i + 1, j]
                H[i + 1, j] = -sn[i] * H[i, j] + cs[i] * H[i + 1, j]
                H[i, j] = t
            d = np.hypot(H[j, j], H[j + 1, j])
            cs[j], sn[j] = (1.0, 0.0) if d == 0 else (H[j, j] / d, H[j + 1, j] / d)
            H[j, j] = cs[j] * H[j, j] + sn[j] * H[j + 1, j]
            H[j + 1, j] = 0.0
            g[j + 1] = -sn[j] * g[j]
            g[j] = cs[j] * g[j]
            its += 1
            k = j + 1
            hist.append(abs(g[j + 1]) / nmb)
            if happy or abs(g[j + 1]) <= rtol * nmb:
                break
        R = np.triu(H[:k, :k])
        try:
            y = np.linalg.solve(R, g[:k])
        except np.linalg.LinAlgError:
            y = np.linalg.lstsq(R, g[:k], rcond=None)[0]
        x = x + V[:k].T @ y
        if happy:
            rel = np.linalg.norm(b - mv(x)) / nb
            if rel <= rtol or rel < 1e-13:
                conv, reason = True, "converged"
                break
    final = np.linalg.norm(b - mv(x)) / nb
    if final <= rtol:
        conv, reason = True, "converged"
    return x, Stats(its, float(final), conv, time.perf_counter() - t0, reason, hist, cycles,
                    cnt["pc"], cnt["mv"])


# --------------------------------------------------------------------------- ILU(0)

@dataclass
class Ilu0:
    L: sp.csr_matrix
    U: sp.csr_matrix


def ilu0(A):
    A = sp.csr_matrix(A, copy=True)
    A.sort_indices()
    if A.shape[0] != A.shape[1]:
        raise ValueError("ilu0 requires a square matrix")
    n = A.shape[0]
    ip = np.ascontiguousarray(A.indptr, dtype=np.int32)
    ix = np.ascontiguousarray(A.indices, dtype=np.int32)
    data = np.ascontiguousarray(A.data, dtype=np.float64)
    bad = np.zeros(1, dtype=np.int64)
    rc = _c().o_ilu0(n, _ptr(ip), _ptr(ix), _ptr(data), _ptr(bad))
    if rc == 1:
        raise ZeroPivotError("missing diagonal entry in sparsity pattern")
    if rc == 2:
        raise ZeroPivotError(f"zero pivot at row {int(bad[0])}")
    A = sp.csr_matrix((data, A.indices, A.indptr), shape=A.shape)
    L = sp.tril(A, k=-1, format="csr") + sp.eye(n, format="csr")
    U = sp.triu(A, k=0, format="csr")
    L.sort_indices()
    U.sort_indices()
    return Ilu0(L, U)


def apply_ilu0(f: Ilu0, r):
    y = spsolve_triangular(f.L, r, lower=True, unit_diagonal=True)
    return spsolve_triangular(f.U, y, lower=False)


# --------------------------------------------------------------------------- selfp

def diag_lump(A):
    if A.shape[0] != A.shape[1]:
        raise ValueError("diag_lump requires a square matrix")
    d = np.asarray(A.diagonal())
    if np.any(d == 0.0):
        raise ZeroPivotError("zero diagonal entry in diag_lump")
    return d


def schur_selfp(D, C, dA, B):
    dA = np.asarray(dA)
    if np.any(dA == 0.0):
        raise ZeroPivotError("zero entry in diagA")
    if C.shape[1] != len(dA) or B.shape[0] != len(dA) or D.shape != (C.shape[0], B.shape[1]):
        raise ValueError("schur_selfp: non-conforming block dimensions")
    S = (D - C @ sp.diags(1.0 / dA) @ B).tocsr()
    S.sum_duplicates()
    S.sort_indices()
    return S


# --------------------------------------------------------------------------- AMG

@dataclass
class Level:
    A: sp.csr_matrix
    P: sp.csr_matrix | None
    lower: sp.csr_matrix | None
    upper: sp.csr_matrix | None
    agg: np.ndarray | None = None
    rho: float | None = None


@dataclass
class Hierarchy:
    levels: list
    coarse_lu: tuple

    @property
    def level_count(self):
        return len(self.levels)


def aggregate(A, theta):
    A = sp.csr_matrix(A)
    n = A.shape[0]
    ip = np.ascontiguousarray(A.indptr, dtype=np.int32)
    ix = np.ascontiguousarray(A.indices, dtype=np.int32)
    dv = np.ascontiguousarray(A.data, dtype=np.float64)
    agg = np.empty(n, dtype=np.int64)
    _c().o_aggregate(n, _ptr(ip), _ptr(ix), _ptr(dv), float(theta), _ptr(agg))
    return agg


def spectral_radius(A, iterations=10):
    M = sp.diags(1.0 / A.diagonal()) @ A
    x = np.random.default_rng(12345).standard_normal(A.shape[0])
    x /= np.linalg.norm(x)
    for _ in range(iterations):
        y = M @ x
        nrm = np.linalg.norm(y)
        if nrm == 0.0:
            return 1.0
        x = y / nrm
    return max(float(np.linalg.norm(M @ x)), 1e-8)


def amg_setup(A, *, theta=0.5, omega=2.0 / 3.0, max_coarse=64, max_levels=25):
    A = sp.csr_matrix(A)
    if A.shape[0] != A.shape[1]:
        raise ValueError("amg_setup requires a square matrix")
    if np.any(A.diagonal() == 0.0):
        raise ZeroPivotError("structurally singular input: zero diagonal entry")
    levels, cur = [], A
    while cur.shape[0] > max_coarse and len(levels) < max_levels - 1:
        agg = aggregate(cur, theta)
        nc = int(agg.max()) + 1
        if nc >= cur.shape[0]:
            if cur.shape[0] > 5000:
                raise RuntimeError("aggregation stalled on a large operator")
            break
        n = cur.shape[0]
        P0 = sp.csr_matrix((np.ones(n), (np.arange(n), agg)), shape=(n, nc))
        Dinv = sp.diags(1.0 / cur.diagonal())
        rho = spectral_radius(cur)
        P = (P0 - (2.0 * omega / rho) * (Dinv @ (cur @ P0))).tocsr()
        levels.append(Level(cur, P, sp.tril(cur, k=0, format="csr"), sp.triu(cur, k=0, format="csr"),
                            agg, rho))
        cur = (P.T @ cur @ P).tocsr()
        cur.sum_duplicates()
    levels.append(Level(cur, None, None, None))
    return Hierarchy(levels, scipy.linalg.lu_factor(cur.toarray()))


def _sgs(lv, x, b):
    x = x + spsolve_triangular(lv.lower, b - lv.A @ x, lower=True)
    return x + spsolve_triangular(lv.upper, b - lv.A @ x, lower=False)


def _vc(h, l, b):
    lv = h.levels[l]
    if lv.P is None:
        return scipy.linalg.lu_solve(h.coarse_lu, b)
    x = _sgs(lv, np.zeros_like(b), b)
    rc = lv.P.T @ (b - lv.A @ x)
    x = x + lv.P @ _vc(h, l + 1, rc)
    return _sgs(lv, x, b)


def amg_vcycle(h, r):
    return _vc(h, 0, np.asarray(r, dtype=float))


# --------------------------------------------------------------------------- options

SCALE_SPLIT_OPTIONS = """
-ksp_type gmres -pc_type fieldsplit -pc_fieldsplit_0_fields 0,1 -pc_fieldsplit_1_fields 2,3
-pc_fieldsplit_type additive
-fieldsplit_0_ksp_type preonly -fieldsplit_0_pc_type fieldsplit -fieldsplit_0_pc_fieldsplit_type schur
-fieldsplit_0_pc_fieldsplit_schur_fact_type full -fieldsplit_0_pc_fieldsplit_schur_precondition selfp
-fieldsplit_0_fieldsplit_0_ksp_type preonly -fieldsplit_0_fieldsplit_0_pc_type bjacobi
-fieldsplit_0_fieldsplit_1_ksp_type preonly -fieldsplit_0_fieldsplit_1_pc_type hypre
-fieldsplit_1_ksp_type preonly -fieldsplit_1_pc_type fieldsplit -fieldsplit_1_pc_fieldsplit_type schur
-fieldsplit_1_pc_fieldsplit_schur_fact_type full -fieldsplit_1_pc_fieldsplit_schur_precondition selfp
-fieldsplit_1_fieldsplit_0_ksp_type preonly -fieldsplit_1_fieldsplit_0_pc_type bjacobi
-fieldsplit_1_fieldsplit_1_ksp_type preonly -fieldsplit_1_fieldsplit_1_pc_type hypre
""".split()

FIELD_SPLIT_OPTIONS = """
-ksp_type gmres -pc_type fieldsplit -pc_fieldsplit_0_fields 0,2 -pc_fieldsplit_1_fields 1,3
-pc_fieldsplit_type schur -pc_fieldsplit_schur_fact_type full -pc_fieldsplit_schur_precondition selfp
-fieldsplit_0_ksp_type preonly -fieldsplit_0_pc_type bjacobi
-fieldsplit_1_ksp_type preonly -fieldsplit_1_pc_type fieldsplit -fieldsplit_1_pc_fieldsplit_type additive
-fieldsplit_1_fieldsplit_0_ksp_type preonly -fieldsplit_1_fieldsplit_0_pc_type hypre
-fieldsplit_1_fieldsplit_1_ksp_type preonly -fieldsplit_1_fieldsplit_1_pc_type hypre
""".split()


@dataclass(frozen=True)
class Leaf:
    pc_type: str
    split: object = None


@dataclass(frozen=True)
class Node:
    groups: tuple
    split_type: str
    children: tuple
    schur_fact_type: str | None = None
    schur_precondition: str | None = None


@dataclass(frozen=True)
class Config:
    split: Node
    ksp_type: str = "gmres"
    rtol: float = 1e-7
    restart: int = 30
    max_iter: int = 1000


def _pairs(tokens):
    if isinstance(tokens, str):
        tokens = tokens.split()
    flat = [t for tok in tokens for t in str(tok).split()]
    out, i = {}, 0
    while i < len(flat):
        k = flat[i]
        if not k.startswith("-"):
            raise OptionError(f"expected an option starting with '-', got {k!r}")
        if i + 1 >= len(flat) or flat[i + 1].startswith("-"):
            raise OptionError(f"option {k} is missing a value")
        if k[1:] in out:
            raise OptionError(f"duplicate option {k}")
        out[k[1:]] = flat[i + 1]
        i += 2
    return out


def _take(o, k, allowed=None):
    if k not in o:
        raise OptionError(f"missing required option -{k}")
    v = o.pop(k)
    if allowed is not None and v not in allowed:
        raise OptionError(f"-{k} {v} is not supported")
    return v


def _fields(v):
    try:
        return tuple(int(t) for t in v.split(","))
    except ValueError as e:
        raise OptionError(f"malformed field list {v!r}") from e


def _split(o, pre, groups):
    st = _take(o, f"{pre}pc_fieldsplit_type", {"additive", "schur"})
    fact = prec = None
    if st == "schur":
        fact = _take(o, f"{pre}pc_fieldsplit_schur_fact_type", {"full"})
        prec = _take(o, f"{pre}pc_fieldsplit_schur_precondition", {"selfp"})
    kids = []
    for i, g in enumerate(groups):
        c = f"{pre}fieldsplit_{i}_"
        _take(o, f"{c}ksp_type", {"preonly"})
        pt = _take(o, f"{c}pc_type", {"bjacobi", "hypre", "fieldsplit"})
        if pt == "fieldsplit":
            if len(g) != 2:
                raise OptionError("nested fieldsplit needs exactly 2 fields")
            kids.append(Leaf("fieldsplit", _split(o, c, ((g[0],), (g[1],)))))
        else:
            kids.append(Leaf("amg" if pt == "hypre" else pt))
    return Node(tuple(groups), st, tuple(kids), fact, prec)


def parse_options(tokens):
    o = _pairs(tokens)
    ksp = _take(o, "ksp_type", {"gmres"})
    _take(o, "pc_type", {"fieldsplit"})
    g0 = _fields(_take(o, "pc_fieldsplit_0_fields"))
    g1 = _fields(o.pop("pc_fieldsplit_1_fields")) if "pc_fieldsplit_1_fields" in o else \
        tuple(f for f in range(4) if f not in g0)
    for g in (g0, g1):
        if len(g) != 2 or len(set(g)) != 2:
            raise OptionError(f"field group {g} must contain exactly 2 distinct fields")
    if sorted(g0 + g1) != [0, 1, 2, 3]:
        raise OptionError("field groups do not partition the four fields")
    node = _split(o, "", (g0, g1))
    if o:
        raise OptionError("unsupported option(s): " + ", ".join("-" + k for k in sorted(o)))
    return Config(node, ksp)


def method_config(method, rtol=1e-7, restart=30, max_iter=1000):
    t = {"scale": SCALE_SPLIT_OPTIONS, "field": FIELD_SPLIT_OPTIONS}.get(method)
    if t is None:
        raise ValueError(f"unknown method {method!r}")
    return replace(parse_options(t), rtol=rtol, restart=restart, max_iter=max_iter)


# --------------------------------------------------------------------------- composition

@dataclass
class Preconditioner:
    apply: object
    description: str
    setup_time_s: float
    parts: dict = None

    def __call__(self, r):
        return self.apply(r)


def _sub(M, r, c):
    return M[r][:, c].tocsr()


def _leaf(inner, M, fids, sizes, parts):
    if inner.pc_type == "bjacobi":
        f = ilu0(M)
        parts.setdefault("ilu", []).append(f)
        return (lambda r: apply_ilu0(f, r)), "bjacobi/ilu0"
    if inner.pc_type == "amg":
        h = amg_setup(M)
        parts.setdefault("amg", []).append(h)
        return (lambda r: amg_vcycle(h, r)), f"amg[{h.level_count}]"
    return _node(inner.split, M, fids, sizes, parts)


def _node(node, M, fids, sizes, parts):
    off = np.cumsum([0] + [sizes[f] for f in fids])
    loc = {f: np.arange(off[i], off[i + 1]) for i, f in enumerate(fids)}
    gA, gB = node.groups
    iA = np.concatenate([loc[f] for f in gA])
    iB = np.concatenate([loc[f] for f in gB])
    A, D = _sub(M, iA, iA), _sub(M, iB, iB)
    if node.split_type == "additive":
        pa, da = _leaf(node.children[0], A, gA, sizes, parts)
        pb, db = _leaf(node.children[1], D, gB, sizes, parts)

        def add(r):
            z = np.zeros_like(r)
            z[iA] = pa(r[iA])
            z[iB] = pb(r[iB])
            return z
        return add, f"additive({da}, {db})"
    B, C = _sub(M, iA, iB), _sub(M, iB, iA)
    S = schur_selfp(D, C, diag_lump(A), B)
    parts.setdefault("schur", []).append(S)
    pa, da = _leaf(node.children[0], A, gA, sizes, parts)
    ps, ds = _leaf(node.children[1], S, gB, sizes, parts)

    def full(r):
        zA = pa(r[iA])
        zB = ps(r[iB] - C @ zA)
        zA = zA - pa(B @ zB)
        z = np.zeros_like(r)
        z[iA] = zA
        z[iB] = zB
        return z
    return full, f"schur-full({da}, selfp->{ds})"


def build_preconditioner(bs, config, monolithic=None):
    t0 = time.perf_counter()
    K = monolithic if monolithic is not None else monolithic_view(bs)[0]
    sz = bs.field_sizes
    sizes = {i: sz[FIELDS[i]] for i in range(4)}
    parts = {}
    ap, desc = _node(config.split, K, (0, 1, 2, 3), sizes, parts)
    return Preconditioner(ap, desc, time.perf_counter() - t0, parts)


@dataclass
class Report:
    x: np.ndarray
    stats: Stats
    assembly_s: float
    solve_s: float
    total_s: float
    method: str
    pc_setup_s: float = 0.0

    @property
    def converged(self):
        return self.stats.converged


def solve(bs, config):
    t0 = time.perf_counter()
    K, f = monolithic_view(bs)
    pc = build_preconditioner(bs, config, monolithic=K)
    x, st = gmres(K, f, preconditioner=pc, rtol=config.rtol, max_iter=config.max_iter,
                  restart=config.restart)
    s = time.perf_counter() - t0
    a = getattr(bs, "wall_time_s", 0.0)
    return Report(x, st, a, s, a + s, pc.description, pc.setup_time_s)
