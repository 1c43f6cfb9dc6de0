"""Discrete-field evaluation and L2 errors (TEST INFRASTRUCTURE ONLY; see oracle/__init__.py).

Restates reference assembly.py:591-644 (DiscreteField.evaluate_all, solution_fields) and
spectrum.py:149-176 (l2_error, field_errors) with numpy, on the oracle's mesh / block system.
Pinned by tests/golden/fields.json (generated from the unmodified reference by
tests/golden/make_golden_fields.py).
"""

from __future__ import annotations

import numpy as np

from .forms import FIELDS
from .geometry import eval_basis, quadrature_rule


def evaluate_all(mesh, formulation, name, coeffs, ref_points):
    """(C, nq) for pressures, (C, nq, dim) for velocities (reference assembly.py:600-633)."""
    pts = np.atleast_2d(ref_points)
    kind = getattr(mesh.cell_kind, "value", mesh.cell_kind)
    vel = name.startswith("u")
    dim = mesh.dim
    if formulation == "hdiv":
        if vel:
            Vref = eval_basis(kind, pts, hdiv=True)
            J, det = mesh.jacobians()
            wloc = mesh.cell_facet_signs * coeffs[mesh.cell_facets]
            return np.einsum("cij,qfj,cf->cqi", J, Vref, wloc) / det[:, None, None]
        return np.broadcast_to(coeffs[:, None], (mesh.n_cells, len(pts))).copy()
    N = eval_basis(kind, pts)
    N = N[0] if isinstance(N, tuple) else N
    nn = N.shape[1]
    if formulation == "cgvms":
        cf = coeffs.reshape(-1, dim)[mesh.cells] if vel else coeffs[mesh.cells]
    else:
        cf = coeffs.reshape(mesh.n_cells, nn, dim) if vel else coeffs.reshape(mesh.n_cells, nn)
    return np.einsum("qa,cai->cqi", N, cf) if vel else np.einsum("qa,ca->cq", N, cf)


def l2_error(mesh, formulation, name, coeffs, exact_field, quadrature_degree=4):
    """Reference spectrum.py:149-169."""
    kind = getattr(mesh.cell_kind, "value", mesh.cell_kind)
    rule = quadrature_rule(kind, quadrature_degree)
    pts, wts = (rule.points, rule.weights) if hasattr(rule, "points") else rule
    J, det = mesh.jacobians()
    origin = mesh.vertices[mesh.cells[:, 0]]
    X = origin[:, None, :] + np.einsum("cij,qj->cqi", J, pts)
    vals_h = evaluate_all(mesh, formulation, name, coeffs, pts)
    exact = np.asarray(exact_field(X.reshape(-1, mesh.dim))).reshape(vals_h.shape)
    diff2 = (vals_h - exact) ** 2
    if diff2.ndim == 3:
        diff2 = diff2.sum(axis=-1)
    return float(np.sqrt(np.einsum("q,cq,c->", wts, diff2, det)))


def field_errors(block_system, x, fields, quadrature_degree=4):
    """Reference spectrum.py:172-176 (x in (u1, p1, u2, p2) order)."""
    sizes = [block_system.size_of(f) for f in FIELDS] if hasattr(block_system, "size_of") else None
    if sizes is None:
        sizes = [len(block_system.rhs[f]) for f in FIELDS]
    out, start = {}, 0
    for name, n in zip(FIELDS, sizes):
        out[name] = l2_error(block_system.mesh, block_system.formulation, name, x[start:start + n],
                             fields.field(name), quadrature_degree)
        start += n
    return out
