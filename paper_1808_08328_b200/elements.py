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
