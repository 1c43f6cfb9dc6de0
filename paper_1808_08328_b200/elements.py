"""Element families, formulations, reference quadrature (dppflow.elements API).

Host-side reference-element utilities (reference elements.py).  The device
assembler carries its own copies of these tables (csrc/assembly.cu); this
module serves user code that inspects rules or counts DoFs.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from enum import Enum

import numpy as np

from .mesh import CellKind


class ElementFamily(str, Enum):
    P1 = "p1"
    Q1 = "q1"
    DP0_DQ0 = "dp0_dq0"
    RT_TRI = "rt_tri"
    RT_QUAD = "rt_quad"
    RT_TET = "rt_tet"
    RT_HEX = "rt_hex"


class Formulation(str, Enum):
    HDIV = "hdiv"
    CG_VMS = "cgvms"
    DG_VMS = "dgvms"


SCALAR_FAMILY = {CellKind.TRI: ElementFamily.P1, CellKind.QUAD: ElementFamily.Q1,
                 CellKind.TET: ElementFamily.P1, CellKind.HEX: ElementFamily.Q1}
HDIV_FAMILY = {CellKind.TRI: ElementFamily.RT_TRI, CellKind.QUAD: ElementFamily.RT_QUAD,
               CellKind.TET: ElementFamily.RT_TET, CellKind.HEX: ElementFamily.RT_HEX}
_VECTOR_DIM = {ElementFamily.RT_TRI: 2, ElementFamily.RT_QUAD: 2, ElementFamily.RT_TET: 3,
               ElementFamily.RT_HEX: 3}
# vertex opposite each local facet (LOCAL_FACETS order) of the simplex flux bases
_TRI_OPPOSITE = ((0.0, 1.0), (1.0, 0.0), (0.0, 0.0))
_TET_OPPOSITE = ((0.0, 0.0, 1.0), (0.0, 1.0, 0.0), (1.0, 0.0, 0.0), (0.0, 0.0, 0.0))


def family_dim(family):
    """Vector dimension of an H(div) family, None for scalar families."""
    return _VECTOR_DIM.get(ElementFamily(family))


def is_vector_family(family) -> bool:
    return ElementFamily(family) in _VECTOR_DIM


def piola_map(geometry, reference_vector_values: np.ndarray) -> np.ndarray:
    """Contravariant Piola transform (J v_ref) / det J (reference elements.py:141-149)."""
    if geometry.det <= 0:
        raise ValueError("singular or inverted cell geometry")
    return np.einsum("ij,...j->...i", geometry.jacobian, reference_vector_values) / geometry.det


def piola_divergence(geometry, reference_divergences: np.ndarray) -> np.ndarray:
    if geometry.det <= 0:
        raise ValueError("singular or inverted cell geometry")
    return np.asarray(reference_divergences) / geometry.det


def eval_basis(family, points):
    """Reference basis at reference points (reference elements.py:79-138): scalar families ->
    (values (n, nd), gradients (n, nd, dim)); RT families -> (values (n, nd, dim), divergences
    (nd,)).  A host-side table utility; the device kernels (csrc/fields.cu, assembly.cu) carry
    the same formulas."""
    fam = ElementFamily(family)
    pts = np.atleast_2d(np.asarray(points, dtype=float))
    n, dim = pts.shape
    tol = 1e-12
    simplex = fam in (ElementFamily.P1, ElementFamily.RT_TRI, ElementFamily.RT_TET)
    inside = (np.all(pts >= -tol) and np.all(pts.sum(axis=-1) <= 1 + tol)) if simplex else \
        (np.all(pts >= -tol) and np.all(pts <= 1 + tol))
    if not inside:
        raise ValueError("reference point outside reference cell")
    if fam is ElementFamily.P1:
        vals = np.empty((n, dim + 1))
        vals[:, 0] = 1.0 - pts.sum(axis=1)
        vals[:, 1:] = pts
        grads = np.empty((n, dim + 1, dim))
        grads[:, 0, :] = -1.0
        grads[:, 1:, :] = np.eye(dim)
        return vals, grads
    if fam is ElementFamily.Q1:
        nd = 2 ** dim
        vals, grads = np.ones((n, nd)), np.ones((n, nd, dim))
        for a in range(nd):
            for axis in range(dim):
                s = (a >> axis) & 1
                f = pts[:, axis] if s else 1.0 - pts[:, axis]
                vals[:, a] *= f
                for other in range(dim):
                    grads[:, a, other] *= (1.0 if s else -1.0) if other == axis else f
        return vals, grads
    if fam is ElementFamily.DP0_DQ0:
        return np.ones((n, 1)), np.zeros((n, 1, dim))
    if dim != _VECTOR_DIM[fam]:
        raise ValueError("point dimension does not match element family")
    if fam is ElementFamily.RT_TRI:
        return pts[:, None, :] - np.array(_TRI_OPPOSITE)[None], np.full(3, 2.0)
    if fam is ElementFamily.RT_TET:
        return 2.0 * (pts[:, None, :] - np.array(_TET_OPPOSITE)[None]), np.full(4, 6.0)
    vals = np.zeros((n, 2 * dim, dim))
    for axis in range(dim):
        vals[:, 2 * axis, axis] = pts[:, axis] - 1.0
        vals[:, 2 * axis + 1, axis] = pts[:, axis]
    return vals, np.ones(2 * dim)


@dataclass(frozen=True)
class QuadratureRule:
    cell_kind: CellKind
    degree: int
    points: np.ndarray
    weights: np.ndarray


def gauss_legendre_01(n: int):
    x, w = np.polynomial.legendre.leggauss(n)
    return 0.5 * (x + 1.0), 0.5 * w


def quadrature_rule(cell_kind, degree: int) -> QuadratureRule:
    """Exact for total degree <= degree (reference elements.py:175-221)."""
    kind = CellKind(cell_kind)
    if not 0 <= degree <= 6:
        raise ValueError(f"unsupported quadrature degree {degree} (0..6)")
    deg = max(degree, 1)
    if kind in (CellKind.QUAD, CellKind.HEX):
        x, w = gauss_legendre_01(math.ceil((deg + 1) / 2))
        grids = np.meshgrid(*([x] * kind.dim), indexing="ij")
        wg = np.meshgrid(*([w] * kind.dim), indexing="ij")
        pts = np.column_stack([g.ravel() for g in grids])
        wts = np.ones(len(pts))
        for g in wg:
            wts *= g.ravel()
    elif kind is CellKind.TRI:
        if deg == 1:
            pts, wts = np.array([[1 / 3, 1 / 3]]), np.array([0.5])
        elif deg == 2:
            pts, wts = np.array([[1 / 6, 1 / 6], [2 / 3, 1 / 6], [1 / 6, 2 / 3]]), np.full(3, 1 / 6)
        else:
            u, wu = gauss_legendre_01(math.ceil((deg + 2) / 2))
            U, V = np.meshgrid(u, u, indexing="ij")
            WU, WV = np.meshgrid(wu, wu, indexing="ij")
            pts = np.column_stack([U.ravel(), (V * (1 - U)).ravel()])
            wts = (WU * WV * (1 - U)).ravel()
    else:
        if deg == 1:
            pts, wts = np.array([[0.25, 0.25, 0.25]]), np.array([1 / 6])
        elif deg == 2:
            a = (5.0 + 3.0 * math.sqrt(5.0)) / 20.0
            b = (5.0 - math.sqrt(5.0)) / 20.0
            pts, wts = np.array([[a, b, b], [b, a, b], [b, b, a], [b, b, b]]), np.full(4, 1 / 24)
        else:
            u, wu = gauss_legendre_01(math.ceil((deg + 3) / 2))
            U, V, W = (g.ravel() for g in np.meshgrid(u, u, u, indexing="ij"))
            WU, WV, WW = (g.ravel() for g in np.meshgrid(wu, wu, wu, indexing="ij"))
            pts = np.column_stack([U, V * (1 - U), W * (1 - U) * (1 - V)])
            wts = WU * WV * WW * (1 - U) ** 2 * (1 - V)
    return QuadratureRule(kind, deg, pts, wts)


def nodes_per_cell(cell_kind) -> int:
    return {CellKind.TRI: 3, CellKind.QUAD: 4, CellKind.TET: 4, CellKind.HEX: 8}[CellKind(cell_kind)]


def dof_count(formulation, mesh) -> int:
    """Total size over both networks (reference elements.py:228-236)."""
    f = Formulation(formulation)
    if f is Formulation.HDIV:
        return 2 * (mesh.n_facets + mesh.n_cells)
    per = 2 * mesh.dim + 2
    if f is Formulation.CG_VMS:
        return per * mesh.n_vertices
    return per * nodes_per_cell(mesh.cell_kind) * mesh.n_cells
