"""Device-resident CSR matrices and block systems (handles into libdpp)."""

from __future__ import annotations

import ctypes as C

import numpy as np
import scipy.sparse as sp

from . import _native as N

BLOCK_NAMES = ("k1_uu", "k1_up", "k1_pu", "k1_pp", "k2_uu", "k2_up", "k2_pu", "k2_pp",
               "k12_pp", "k21_pp")


def canonical(A) -> sp.csr_matrix:
    """scipy CSR with sorted, summed indices (a copy when the input is not canonical)."""
    A = sp.csr_matrix(A)
    if not A.has_canonical_format:
        A = A.copy()
        A.sum_duplicates()
    return A


class DeviceCsr:
    """A CSR matrix in HBM (scipy storage semantics: int32 indices, explicit zeros kept)."""

    def __init__(self, handle, owner=None):
        self.h = handle
        self._owner = owner          # keeps a borrowed view's parent alive
        r, c, z = C.c_int(), C.c_int(), C.c_int64()
        N.call("dpp_csr_info", handle, C.byref(r), C.byref(c), C.byref(z))
        self.shape = (r.value, c.value)
        self.nnz = int(z.value)

    @classmethod
    def from_scipy(cls, A) -> "DeviceCsr":
        A = canonical(A)
        ip, ix, v = N.i32(A.indptr), N.i32(A.indices), N.f64(A.data)
        h = C.c_void_p()
        N.call("dpp_csr_create", N.ctx(), A.shape[0], A.shape[1], len(v), N.ptr(ip), N.ptr(ix),
               N.ptr(v), C.byref(h))
        return cls(h)

    def to_scipy(self) -> sp.csr_matrix:
        ip = np.empty(self.shape[0] + 1, dtype=np.int32)
        ix = np.empty(self.nnz, dtype=np.int32)
        v = np.empty(self.nnz)
        N.call("dpp_csr_download", self.h, N.ptr(ip), N.ptr(ix), N.ptr(v))
        return sp.csr_matrix((v, ix, ip), shape=self.shape)

    def __matmul__(self, x):
        x = N.f64(x)
        if x.ndim != 1 or x.shape[0] != self.shape[1]:
            raise ValueError(f"dimension mismatch: {self.shape} @ {x.shape}")
        y = np.empty(self.shape[0])
        N.call("dpp_spmv", N.ctx(), self.h, N.ptr(x), N.ptr(y))
        return y

    def __del__(self):
        if getattr(self, "h", None) is not None and N._lib is not None:
            N.lib().dpp_csr_destroy(self.h)
            self.h = None


def as_device(A) -> DeviceCsr:
    if isinstance(A, DeviceCsr):
        return A
    if isinstance(A, np.ndarray) and A.ndim == 2:
        A = sp.csr_matrix(A)
    return DeviceCsr.from_scipy(A)


class DeviceSystem:
    """Ten blocks + four RHS segments in HBM (reference BlockSystem, assembly.py:48-99)."""

    def __init__(self, handle):
        self.h = handle
        s = (C.c_int64 * 4)()
        N.call("dpp_system_sizes", handle, s)
        self.sizes = tuple(int(v) for v in s)

    @classmethod
    def from_blocks(cls, blocks, rhs, sizes) -> "DeviceSystem":
        devs = [None if b is None else as_device(b) for b in blocks]
        arr = (C.c_void_p * 10)(*[None if d is None else d.h.value for d in devs])
        rh = [None if r is None else N.f64(r) for r in rhs]
        rarr = (C.c_void_p * 4)(*[None if r is None else r.ctypes.data for r in rh])
        sz = (C.c_int64 * 4)(*sizes)
        h = C.c_void_p()
        N.call("dpp_system_from_blocks", N.ctx(), arr, rarr, sz, C.byref(h))
        return cls(h)

    def block(self, i) -> DeviceCsr:
        h = C.c_void_p()
        N.call("dpp_system_block", self.h, i, C.byref(h))
        return DeviceCsr(h, owner=self)

    def rhs(self, field) -> np.ndarray:
        out = np.empty(self.sizes[field])
        N.call("dpp_system_rhs", self.h, field, N.ptr(out))
        return out

    def monolithic(self) -> DeviceCsr:
        h = C.c_void_p()
        N.call("dpp_system_monolithic", self.h, C.byref(h))
        return DeviceCsr(h, owner=self)

    def assembly_ms(self) -> float:
        t = C.c_double()
        N.call("dpp_system_timing", self.h, C.byref(t))
        return float(t.value)

    def __del__(self):
        if getattr(self, "h", None) is not None and N._lib is not None:
            N.lib().dpp_system_destroy(self.h)
            self.h = None
