"""ctypes binding of libdpp.so (include/dpp.h).

The product path has no CPU fallback: if the CUDA library or a CUDA device is
missing, every entry point that needs the device raises DeviceUnavailable.
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("DPP_LIB") or os.path.join(_HERE, "libdpp.so")

DPP_OK, DPP_ERR_CUDA, DPP_ERR_VALUE, DPP_ERR_ZERO_PIVOT, DPP_ERR_RUNTIME, DPP_ERR_ALLOC = range(6)
KINDS = {"tri": 0, "quad": 1, "tet": 2, "hex": 3}
FORMS = {"hdiv": 0, "cgvms": 1, "dgvms": 2}


class DeviceUnavailable(RuntimeError):
    """libdpp or the CUDA device is missing -- there is no CPU fallback."""


class ZeroPivotError(RuntimeError):
    """Mirror of dppflow.linalg.ZeroPivotError (reference linalg.py:23-24)."""


class Params(C.Structure):
    _fields_ = [("mu", C.c_double), ("beta", C.c_double), ("k1", C.c_double), ("k2", C.c_double),
                ("eta_u", C.c_double), ("eta_p", C.c_double), ("gamma_b", C.c_double * 3)]


class Bc(C.Structure):
    _fields_ = [("n_pfacets", C.c_int64 * 2), ("pfacets", C.c_void_p * 2), ("p0", C.c_void_p * 2),
                ("n_vfacets", C.c_int64 * 2), ("vfacets", C.c_void_p * 2), ("vdata", C.c_void_p * 2),
                ("p0_kind", C.c_int32 * 2), ("p0_coef", (C.c_double * 4) * 2)]


class SplitNode(C.Structure):
    _fields_ = [("split_type", C.c_int), ("ngroup", C.c_int * 2), ("groups", (C.c_int * 2) * 2),
                ("child_type", C.c_int * 2), ("child_node", C.c_int * 2)]


class KrylovStatsC(C.Structure):
    _fields_ = [("iterations", C.c_int), ("cycles", C.c_int), ("converged", C.c_int),
                ("reason", C.c_int), ("pc_applies", C.c_int), ("matvecs", C.c_int),
                ("relative_residual", C.c_double), ("wall_time_s", C.c_double)]


class StepProfile(C.Structure):
    _fields_ = [("spmv_ms", C.c_double), ("pc_ms", C.c_double), ("spmv_bytes", C.c_double),
                ("pc_bytes", C.c_double), ("mgs_ms", C.c_double), ("pc_launches", C.c_int64)]


RANDN_FN = C.CFUNCTYPE(None, C.c_int64, C.POINTER(C.c_double), C.c_void_p)
APPLY_FN = C.CFUNCTYPE(None, C.POINTER(C.c_double), C.POINTER(C.c_double), C.c_void_p)

P = C.c_void_p
PP = C.POINTER(C.c_void_p)
I32, I64, D = C.c_int, C.c_int64, C.c_double

# name -> argtypes (restype is always int status)
SIGNATURES = {
    "dpp_version": [],
    "dpp_ctx_create": [I32, PP],
    "dpp_ctx_destroy": [P],
    "dpp_ctx_sync": [P],
    "dpp_timer_start": [P],
    "dpp_timer_stop": [P, C.POINTER(D)],
    "dpp_ctx_launches": [P, C.POINTER(I64)],
    "dpp_ctx_set_tri_jacobi": [P, I32],
    "dpp_csr_create": [P, I32, I32, I64, P, P, P, PP],
    "dpp_csr_info": [P, C.POINTER(I32), C.POINTER(I32), C.POINTER(I64)],
    "dpp_csr_download": [P, P, P, P],
    "dpp_csr_destroy": [P],
    "dpp_spmv": [P, P, P, P],
    "dpp_csr_plan": [P, I32],
    "dpp_mesh_generate": [I32, I32, I32, PP],
    "dpp_mesh_generate_device": [P, I32, I32, I32, PP],
    "dpp_mesh_from_arrays": [I32, I32, I32, I64, P, I64, P, PP],
    "dpp_mesh_counts": [P, C.POINTER(I64), C.POINTER(I64), C.POINTER(I64)],
    "dpp_mesh_export": [P] + [P] * 11,
    "dpp_mesh_destroy": [P],
    "dpp_mesh_release_device": [P],
    "dpp_facet_rule_size": [I32, I32, I32, C.POINTER(I32)],
    "dpp_facet_points": [P, P, I32, I64, P, P, P],
    "dpp_assemble": [P, P, I32, C.POINTER(Params), C.POINTER(Bc), PP],
    "dpp_assemble_ext": [P, P, I32, C.POINTER(Params), P, P, C.POINTER(Bc), PP],
    "dpp_field_evaluate": [P, P, I32, I32, P, I64, I32, P, P],
    "dpp_cell_points": [P, P, I32, P, P],
    "dpp_field_l2_error": [P, P, I32, I32, P, I64, I32, P, P, I32, P, P, C.POINTER(D)],
    "dpp_system_eliminate": [P, I32, I64, P, P],
    "dpp_mesh_upload_bytes": [P, C.POINTER(I64)],
    "dpp_system_from_blocks": [P, C.POINTER(P), C.POINTER(P), C.POINTER(I64), PP],
    "dpp_system_sizes": [P, C.POINTER(I64)],
    "dpp_system_block": [P, I32, PP],
    "dpp_system_rhs": [P, I32, P],
    "dpp_system_monolithic": [P, PP],
    "dpp_system_timing": [P, C.POINTER(D)],
    "dpp_system_destroy": [P],
    "dpp_ilu0_create": [P, P, PP],
    "dpp_ilu0_apply": [P, P, P],
    "dpp_ilu0_factors": [P, PP, PP],
    "dpp_ilu0_destroy": [P],
    "dpp_diag": [P, P, P],
    "dpp_schur_selfp": [P, P, P, P, P, PP],
    "dpp_amg_create": [P, P, D, D, I32, I32, RANDN_FN, P, PP],
    "dpp_amg_levels": [P, C.POINTER(I32)],
    "dpp_strength_aggregates": [P, P, D, I32, P, C.POINTER(I64)],
    "dpp_amg_level": [P, I32, PP, PP, P, C.POINTER(D)],
    "dpp_amg_vcycle": [P, P, P],
    "dpp_amg_destroy": [P],
    "dpp_pc_create": [P, P, C.POINTER(SplitNode), I32, RANDN_FN, P, PP],
    "dpp_pc_create_explicit": [P, P, P, C.POINTER(SplitNode), I32, RANDN_FN, P, PP],
    "dpp_pc_apply": [P, P, P],
    "dpp_pc_describe": [P, C.c_char_p, I32],
    "dpp_pc_setup_ms": [P, C.POINTER(D)],
    "dpp_pc_destroy": [P],
    "dpp_gmres": [P, P, APPLY_FN, P, P, APPLY_FN, P, I64, P, P, P, D, I32, I32,
                  C.POINTER(KrylovStatsC), P, I32],
    "dpp_solve": [P, P, P, D, I32, I32, P, C.POINTER(KrylovStatsC), P, I32],
    "dpp_peerbuf_create": [P, I64, PP],
    "dpp_peerbuf_export": [P, P],
    "dpp_peerbuf_open": [P, P, I64, PP],
    "dpp_peerbuf_write": [P, P, I64],
    "dpp_peerbuf_read": [P, P, I64],
    "dpp_peerbuf_destroy": [P],
    "dpp_shard_create": [P, I32, I64, P, P, P, I32, P, PP],
    "dpp_shard_spmv": [P, P, C.POINTER(P), P],
    "dpp_shard_profile": [P, P, C.POINTER(P), P, I32, C.POINTER(D), C.POINTER(D)],
    "dpp_shard_destroy": [P],
    "dpp_profile_step": [P, P, P, I32, I32, C.POINTER(StepProfile)],
}

_lib = None


def lib():
    """Load libdpp.so (fails loudly; there is no CPU fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise DeviceUnavailable(f"{LIB_PATH} is missing: run __graft_entry__.build() "
                                    "(or make -C paper_1808_08328_b200/csrc)")
        lib_ = C.CDLL(LIB_PATH)
        for name, args in SIGNATURES.items():
            fn = getattr(lib_, name)
            fn.argtypes = args
            fn.restype = C.c_int
        lib_.dpp_last_error.argtypes = []
        lib_.dpp_last_error.restype = C.c_char_p
        _lib = lib_
    return _lib


def check(rc):
    if rc == DPP_OK:
        return
    msg = lib().dpp_last_error().decode(errors="replace")
    if rc == DPP_ERR_ZERO_PIVOT:
        raise ZeroPivotError(msg)
    if rc == DPP_ERR_VALUE:
        raise ValueError(msg)
    if rc == DPP_ERR_CUDA:
        raise DeviceUnavailable(msg)
    if rc == DPP_ERR_ALLOC:
        raise MemoryError(msg)
    raise RuntimeError(msg)


def call(name, *args):
    check(getattr(lib(), name)(*args))


def ptr(a):
    return None if a is None else C.c_void_p(a.ctypes.data)


class _Ctx:
    def __init__(self):
        self.handle = None

    def get(self):
        if self.handle is None:
            h = C.c_void_p()
            dev = int(os.environ.get("DPP_DEVICE", os.environ.get("LOCAL_RANK", "0")))
            call("dpp_ctx_create", dev, C.byref(h))
            self.handle = h
        return self.handle


_CTX = _Ctx()


def ctx():
    """The process-wide device context (device = $DPP_DEVICE or $LOCAL_RANK or 0)."""
    return _CTX.get()


def launches():
    n = C.c_int64()
    call("dpp_ctx_launches", ctx(), C.byref(n))
    return int(n.value)


def sync():
    call("dpp_ctx_sync", ctx())


# power-iteration start vector of the reference (linalg.py:330): a fresh
# default_rng(12345) per call, so the vector depends on n only -- cached per n
_RANDN_CACHE = {}


def _randn(n, out, _user):
    n = int(n)
    v = _RANDN_CACHE.get(n)
    if v is None:
        v = np.random.default_rng(12345).standard_normal(n)
        if len(_RANDN_CACHE) < 64:
            _RANDN_CACHE[n] = v
    C.memmove(out, v.ctypes.data, 8 * n)


RANDN = RANDN_FN(_randn)


def f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def i32(a):
    return np.ascontiguousarray(a, dtype=np.int32)


def i64(a):
    return np.ascontiguousarray(a, dtype=np.int64)
