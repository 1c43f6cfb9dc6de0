"""Structured meshes (drop-in for dppflow.mesh, reference mesh.py).

Numbering is produced by libdpp -- on the device (csrc/devmesh.cu: closed-form
vertices / cells, radix-sorted facet tuples, adjacency and geometry kernels) or,
without a GPU or for user-supplied cells, by the host builder (csrc/mesh.cpp) --
and is bit-exact with the reference (mesh.py:206-277, :106-167); the Mesh object
exposes the same numpy arrays and keeps the native handle whose device image the
assembler reads.
"""

from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass
from enum import Enum

import numpy as np

from . import _native as N

BOUNDARY = -1


class CellKind(str, Enum):
    TRI = "tri"
    QUAD = "quad"
    TET = "tet"
    HEX = "hex"

    @property
    def dim(self) -> int:
        return 2 if self in (CellKind.TRI, CellKind.QUAD) else 3

    @property
    def n_facets_per_cell(self) -> int:
        return {CellKind.TRI: 3, CellKind.QUAD: 4, CellKind.TET: 4, CellKind.HEX: 6}[self]


LOCAL_FACETS = {
    CellKind.TRI: ((0, 1), (0, 2), (1, 2)),
    CellKind.QUAD: ((0, 2), (1, 3), (0, 1), (2, 3)),
    CellKind.TET: ((0, 1, 2), (0, 1, 3), (0, 2, 3), (1, 2, 3)),
    CellKind.HEX: ((0, 2, 4, 6), (1, 3, 5, 7), (0, 1, 4, 5), (2, 3, 6, 7), (0, 1, 2, 3), (4, 5, 6, 7)),
}
_NODES = {CellKind.TRI: 3, CellKind.QUAD: 4, CellKind.TET: 4, CellKind.HEX: 8}
_FNODES = {CellKind.TRI: 2, CellKind.QUAD: 2, CellKind.TET: 3, CellKind.HEX: 4}


@dataclass(frozen=True)
class FacetRecord:
    vertices: tuple
    plus_cell: int
    minus_cell: int
    normal: np.ndarray
    measure: float
    center: np.ndarray

    @property
    def is_boundary(self) -> bool:
        return self.minus_cell == BOUNDARY


@dataclass(frozen=True)
class CellGeometry:
    origin: np.ndarray
    jacobian: np.ndarray
    det: float
    volume: float


class Mesh:
    """Immutable structured mesh of the unit domain (reference mesh.py:73-199)."""

    def __init__(self, dim, cell_kind, n_div, vertices, cells, _handle=None):
        self.dim = dim
        self.cell_kind = CellKind(cell_kind)
        self.n_div = n_div
        self.h = 1.0 / n_div
        if _handle is None:
            v = N.f64(vertices)
            c = N.i64(cells)
            h = C.c_void_p()
            N.call("dpp_mesh_from_arrays", dim, N.KINDS[self.cell_kind.value], n_div, len(v),
                   N.ptr(v), len(c), N.ptr(c), C.byref(h))
            _handle = h
        self._h = _handle
        self._export()

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and N._lib is not None:
            N.lib().dpp_mesh_destroy(h)

    def _export(self):
        nv, nc, nf = C.c_int64(), C.c_int64(), C.c_int64()
        N.call("dpp_mesh_counts", self._h, C.byref(nv), C.byref(nc), C.byref(nf))
        V, Cn, F, d = nv.value, nc.value, nf.value, self.dim
        k = self.cell_kind
        nloc = k.n_facets_per_cell
        self.vertices = np.empty((V, d))
        self.cells = np.empty((Cn, _NODES[k]), dtype=np.int64)
        self.facet_vertex_ids = np.empty((F, _FNODES[k]), dtype=np.int64)
        self.cell_facets = np.empty((Cn, nloc), dtype=np.int64)
        self.cell_facet_signs = np.empty((Cn, nloc), dtype=np.int8)
        self.facet_plus = np.empty(F, dtype=np.int64)
        self.facet_minus = np.empty(F, dtype=np.int64)
        self.facet_normals = np.empty((F, d))
        self.facet_measures = np.empty(F)
        self._J = np.empty((Cn, d, d))
        self._det = np.empty(Cn)
        N.call("dpp_mesh_export", self._h, *(N.ptr(a) for a in (
            self.vertices, self.cells, self.facet_vertex_ids, self.cell_facets, self.cell_facet_signs,
            self.facet_plus, self.facet_minus, self.facet_normals, self.facet_measures, self._J,
            self._det)))
        self.interior_facets = np.flatnonzero(self.facet_minus != BOUNDARY)
        self.boundary_facets = np.flatnonzero(self.facet_minus == BOUNDARY)
        self._facets = None

    @property
    def n_vertices(self) -> int:
        return len(self.vertices)

    @property
    def n_cells(self) -> int:
        return len(self.cells)

    @property
    def n_facets(self) -> int:
        return len(self.facet_vertex_ids)

    @property
    def facets(self):
        """FacetRecord list (reference mesh.py:131-134), built on demand."""
        if self._facets is None:
            pts = self.vertices[self.facet_vertex_ids]
            ctr = pts.mean(axis=1)
            self._facets = [FacetRecord(tuple(int(v) for v in self.facet_vertex_ids[f]),
                                        int(self.facet_plus[f]), int(self.facet_minus[f]),
                                        self.facet_normals[f], float(self.facet_measures[f]), ctr[f])
                            for f in range(self.n_facets)]
        return self._facets

    def jacobians(self):
        return self._J, self._det

    def boundary_vertices(self) -> np.ndarray:
        return np.unique(self.facet_vertex_ids[self.boundary_facets].ravel())

    def dump_text(self) -> str:
        lines = ["vertices"]
        lines += [" ".join(f"{x:.17g}" for x in p) for p in self.vertices]
        lines.append("cells")
        lines += [" ".join(str(int(i)) for i in cell) for cell in self.cells]
        return "\n".join(lines) + "\n"


def reference_measure(cell_kind) -> float:
    return {CellKind.TRI: 0.5, CellKind.QUAD: 1.0, CellKind.TET: 1.0 / 6.0,
            CellKind.HEX: 1.0}[CellKind(cell_kind)]


def generate_unit_mesh(dim: int, cell_kind, n_div: int) -> Mesh:
    """Structured mesh of the unit square/cube (reference mesh.py:206-277)."""
    cell_kind = CellKind(cell_kind)
    if n_div < 1:
        raise ValueError("n_div must be a positive integer")
    if cell_kind.dim != dim:
        raise ValueError(f"cell kind {cell_kind.value} is {cell_kind.dim}D, requested dim={dim}")
    h = C.c_void_p()
    ctx = _mesh_ctx()
    if ctx is not None:
        # built in HBM (csrc/devmesh.cu); the numpy arrays are read back from the device image
        N.call("dpp_mesh_generate_device", ctx, dim, N.KINDS[cell_kind.value], n_div, C.byref(h))
    else:
        N.call("dpp_mesh_generate", dim, N.KINDS[cell_kind.value], n_div, C.byref(h))
    return Mesh(dim, cell_kind, n_div, None, None, _handle=h)


def _mesh_ctx():
    """Where generate_unit_mesh numbers the mesh: $DPP_MESH = device | host | auto (default).

    auto: on the device when there is one; a box without a GPU can still number a mesh with the
    host builder (csrc/mesh.cpp, the same arrays bit for bit) -- assembling it needs the device.
    """
    mode = os.environ.get("DPP_MESH", "auto")
    if mode == "host":
        return None
    if mode not in ("auto", "device"):
        raise ValueError(f"DPP_MESH={mode!r}: expected device, host or auto")
    global _NO_DEVICE
    if mode == "auto" and _NO_DEVICE:
        return None
    try:
        return N.ctx()
    except N.DeviceUnavailable:
        if mode == "device":
            raise
        _NO_DEVICE = True
        return None


_NO_DEVICE = False


def facet_adjacency(mesh: Mesh):
    return mesh.facets


def cell_geometry(mesh: Mesh, cell_index: int) -> CellGeometry:
    if not 0 <= cell_index < mesh.n_cells:
        raise IndexError(f"cell index {cell_index} out of range")
    J, dets = mesh.jacobians()
    det = float(dets[cell_index])
    if det <= 0:
        raise RuntimeError(f"cell {cell_index} has non-positive Jacobian determinant")
    origin = mesh.vertices[mesh.cells[cell_index, 0]]
    return CellGeometry(origin, J[cell_index], det, det * reference_measure(mesh.cell_kind))
