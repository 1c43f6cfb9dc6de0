"""Oracle: structured unit meshes, reference elements and quadrature.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Restates, in vectorised numpy, the numbering contracts of
  reference mesh.py:39-44   (LOCAL_FACETS)
  reference mesh.py:106-167 (facet enumeration, plus/minus cells, normals)
  reference mesh.py:171-185 (affine Jacobians; det via numpy's LAPACK slogdet path)
  reference mesh.py:206-277 (vertex ids x-fastest, TRI diagonal split, Kuhn TETs)
and of the reference elements / quadrature of elements.py:79-138, 154-221.
Integer numbering is bit-exact with the reference (pinned by tests/golden).
"""

from __future__ import annotations

import itertools
import math

import numpy as np


class CellKind:
    TRI, QUAD, TET, HEX = "tri", "quad", "tet", "hex"
    DIM = {"tri": 2, "quad": 2, "tet": 3, "hex": 3}
    NODES = {"tri": 3, "quad": 4, "tet": 4, "hex": 8}


def _kind(k) -> str:
    return getattr(k, "value", k)


# local facet -> local vertex positions (reference mesh.py:39-44)
LOCAL_FACETS = {
    "tri": ((0, 1), (0, 2), (1, 2)),
    "quad": ((0, 2), (1, 3), (0, 1), (2, 3)),
    "tet": ((0, 1, 2), (0, 1, 3), (0, 2, 3), (1, 2, 3)),
    "hex": ((0, 2, 4, 6), (1, 3, 5, 7), (0, 1, 4, 5), (2, 3, 6, 7), (0, 1, 2, 3), (4, 5, 6, 7)),
}

REF_MEASURE = {"tri": 0.5, "quad": 1.0, "tet": 1.0 / 6.0, "hex": 1.0}


class OMesh:
    """Array-only mesh (vertices, cells, facet tables, Jacobians)."""

    def __init__(self, dim, kind, n_div, vertices, cells):
        self.dim, self.kind, self.n_div = dim, _kind(kind), n_div
        self.cell_kind = self.kind
        self.h = 1.0 / n_div
        self.vertices = np.asarray(vertices, dtype=float)
        self.cells = np.asarray(cells, dtype=np.int64)
        self._facets()
        J, det = self._jac()
        self.J, self.det = J, det

    @property
    def n_vertices(self):
        return len(self.vertices)

    @property
    def n_cells(self):
        return len(self.cells)

    @property
    def n_facets(self):
        return len(self.facet_vertex_ids)

    def jacobians(self):
        return self.J, self.det

    # -- facet table: sort-unique of sorted local vertex tuples ---------------
    def _facets(self):
        loc = np.array(LOCAL_FACETS[self.kind])          # (nf, nv)
        C, nf = len(self.cells), loc.shape[0]
        keys = np.sort(self.cells[:, loc], axis=2).reshape(C * nf, -1)
        cell = np.repeat(np.arange(C), nf)
        lf = np.tile(np.arange(nf), C)
        order = np.lexsort((lf, cell) + tuple(keys[:, k] for k in reversed(range(keys.shape[1]))))
        ks = keys[order]
        new = np.ones(len(ks), dtype=bool)
        new[1:] = np.any(ks[1:] != ks[:-1], axis=1)
        fid_sorted = np.cumsum(new) - 1
        nF = int(fid_sorted[-1]) + 1
        first = np.flatnonzero(new)
        count = np.diff(np.append(first, len(ks)))
        if np.any(count > 2):
            raise ValueError("facet shared by more than two cells")
        fid = np.empty(C * nf, dtype=np.int64)
        fid[order] = fid_sorted
        is_plus = np.zeros(len(ks), dtype=bool)
        is_plus[first] = True
        sign = np.empty(C * nf, dtype=np.int8)
        sign[order] = np.where(is_plus, 1, -1)
        self.facet_vertex_ids = ks[first].astype(np.int64)
        self.cell_facets = fid.reshape(C, nf)
        self.cell_facet_signs = sign.reshape(C, nf)
        self.facet_plus = cell[order][first].astype(np.int64)
        minus = np.full(nF, -1, dtype=np.int64)
        two = count == 2
        minus[two] = cell[order][first[two] + 1]
        self.facet_minus = minus
        self.interior_facets = np.flatnonzero(minus != -1)
        self.boundary_facets = np.flatnonzero(minus == -1)
        # geometry (reference mesh.py:145-167)
        pts = self.vertices[self.facet_vertex_ids]       # (F, nv, dim)
        center = pts.mean(axis=1)
        if self.dim == 2:
            t = pts[:, 1] - pts[:, 0]
            meas = np.sqrt(np.einsum("fi,fi->f", t, t))
            nrm = np.stack([t[:, 1], -t[:, 0]], axis=1) / meas[:, None]
        else:
            cr = np.cross(pts[:, 1] - pts[:, 0], pts[:, 2] - pts[:, 0])
            a2 = np.sqrt(np.einsum("fi,fi->f", cr, cr))
            nrm = cr / a2[:, None]
            meas = 0.5 * a2 if pts.shape[1] == 3 else a2
        cc = self.vertices[self.cells[self.facet_plus]].mean(axis=1)
        flip = np.einsum("fi,fi->f", nrm, center - cc) < 0
        nrm[flip] *= -1.0
        self.facet_normals, self.facet_measures, self.facet_centers = nrm, meas, center

    def _jac(self):
        v, c = self.vertices, self.cells
        if self.kind in ("tri", "tet"):
            J = np.stack([v[c[:, k + 1]] - v[c[:, 0]] for k in range(self.dim)], axis=-1)
        else:
            d = v[c[:, -1]] - v[c[:, 0]]
            J = np.zeros((len(c), self.dim, self.dim))
            for k in range(self.dim):
                J[:, k, k] = d[:, k]
        return J, np.linalg.det(J)


def generate_unit_mesh(dim, kind, n):
    kind = _kind(kind)
    if n < 1:
        raise ValueError("n_div must be a positive integer")
    if CellKind.DIM[kind] != dim:
        raise ValueError("cell kind / dim mismatch")
    xs = np.linspace(0.0, 1.0, n + 1)
    m = n + 1
    if dim == 2:
        jj, ii = np.meshgrid(np.arange(m), np.arange(m), indexing="ij")
        verts = np.stack([xs[ii.ravel()], xs[jj.ravel()]], axis=1)
        J, I = np.meshgrid(np.arange(n), np.arange(n), indexing="ij")
        I, J = I.ravel(), J.ravel()
        v00, v10, v01, v11 = J * m + I, J * m + I + 1, (J + 1) * m + I, (J + 1) * m + I + 1
        if kind == "quad":
            cells = np.stack([v00, v10, v01, v11], axis=1)
        else:
            cells = np.stack([np.stack([v00, v10, v11], 1), np.stack([v00, v11, v01], 1)],
                             axis=1).reshape(-1, 3)
    else:
        K3, J3, I3 = np.meshgrid(np.arange(m), np.arange(m), np.arange(m), indexing="ij")
        verts = np.stack([xs[I3.ravel()], xs[J3.ravel()], xs[K3.ravel()]], axis=1)
        K, J, I = (g.ravel() for g in np.meshgrid(np.arange(n), np.arange(n), np.arange(n),
                                                  indexing="ij"))

        def vid(i, j, k):
            return (k * m + j) * m + i

        if kind == "hex":
            cells = np.stack([vid(I + di, J + dj, K + dk)
                              for dk in (0, 1) for dj in (0, 1) for di in (0, 1)], axis=1)
        else:
            tets = []
            for perm in itertools.permutations((0, 1, 2)):
                step = np.zeros((3, 3), dtype=np.int64)
                pos = np.zeros(3, dtype=np.int64)
                corners = [pos.copy()]
                for ax in perm:
                    pos[ax] += 1
                    corners.append(pos.copy())
                ids = [vid(I + c[0], J + c[1], K + c[2]) for c in corners]
                parity = np.linalg.det(np.eye(3)[list(perm)].T)
                if parity < 0:
                    ids[1], ids[2] = ids[2], ids[1]
                tets.append(np.stack(ids, axis=1))
                del step
            cells = np.stack(tets, axis=1).reshape(-1, 4)
    mesh = OMesh(dim, kind, n, verts, cells)
    if np.any(mesh.det <= 0):
        raise RuntimeError("inverted cell")
    return mesh


# -- quadrature & bases (reference elements.py:154-221, 79-138) ---------------

def gauss01(n):
    x, w = np.polynomial.legendre.leggauss(n)
    return 0.5 * (x + 1.0), 0.5 * w


def quadrature_rule(kind, degree):
    """(points, weights) of the reference rule (elements.py:175-221)."""
    kind = _kind(kind)
    if degree < 0 or degree > 6:
        raise ValueError("unsupported quadrature degree")
    degree = max(degree, 1)
    if kind in ("quad", "hex"):
        d = CellKind.DIM[kind]
        x, w = gauss01(math.ceil((degree + 1) / 2))
        g = np.meshgrid(*([x] * d), indexing="ij")
        wg = np.meshgrid(*([w] * d), indexing="ij")
        pts = np.column_stack([a.ravel() for a in g])
        wts = np.ones(len(pts))
        for a in wg:
            wts *= a.ravel()
        return pts, wts
    if kind == "tri":
        if degree == 1:
            return np.array([[1 / 3, 1 / 3]]), np.array([0.5])
        if degree == 2:
            return (np.array([[1 / 6, 1 / 6], [2 / 3, 1 / 6], [1 / 6, 2 / 3]]), np.full(3, 1 / 6))
        n = math.ceil((degree + 2) / 2)
        u, wu = gauss01(n)
        U, V = np.meshgrid(u, u, indexing="ij")
        WU, WV = np.meshgrid(wu, wu, indexing="ij")
        return (np.column_stack([U.ravel(), (V * (1 - U)).ravel()]), (WU * WV * (1 - U)).ravel())
    if degree == 1:
        return np.array([[0.25, 0.25, 0.25]]), np.array([1 / 6])
    if degree == 2:
        a = (5.0 + 3.0 * math.sqrt(5.0)) / 20.0
        b = (5.0 - math.sqrt(5.0)) / 20.0
        return np.array([[a, b, b], [b, a, b], [b, b, a], [b, b, b]]), np.full(4, 1 / 24)
    n = math.ceil((degree + 3) / 2)
    u, wu = gauss01(n)
    U, V, W = (g.ravel() for g in np.meshgrid(u, u, u, indexing="ij"))
    WU, WV, WW = (g.ravel() for g in np.meshgrid(wu, wu, wu, indexing="ij"))
    return (np.column_stack([U, V * (1 - U), W * (1 - U) * (1 - V)]),
            WU * WV * WW * (1 - U) ** 2 * (1 - V))


def scalar_basis(kind, pts):
    """P1 / Q1 values (n, nd) and reference gradients (n, nd, dim)."""
    kind = _kind(kind)
    pts = np.atleast_2d(np.asarray(pts, dtype=float))
    n, d = pts.shape
    if kind in ("tri", "tet"):
        vals = np.empty((n, d + 1))
        vals[:, 0] = 1.0 - pts.sum(axis=1)
        vals[:, 1:] = pts
        grads = np.empty((n, d + 1, d))
        grads[:, 0, :] = -1.0
        grads[:, 1:, :] = np.eye(d)
        return vals, grads
    nd = 2 ** d
    vals = np.ones((n, nd))
    grads = np.ones((n, nd, d))
    for a in range(nd):
        for ax in range(d):
            s = (a >> ax) & 1
            f = pts[:, ax] if s else 1.0 - pts[:, ax]
            vals[:, a] *= f
            for o in range(d):
                grads[:, a, o] *= (1.0 if s else -1.0) if o == ax else f
    return vals, grads


_OPP = {"tri": [(0.0, 1.0), (1.0, 0.0), (0.0, 0.0)],
        "tet": [(0.0, 0.0, 1.0), (0.0, 1.0, 0.0), (1.0, 0.0, 0.0), (0.0, 0.0, 0.0)]}


def flux_basis(kind, pts):
    """Facet-flux H(div) reference values (n, nf, dim) (elements.py:116-138)."""
    kind = _kind(kind)
    pts = np.atleast_2d(np.asarray(pts, dtype=float))
    if kind == "tri":
        return pts[:, None, :] - np.array(_OPP["tri"])[None]
    if kind == "tet":
        return 2.0 * (pts[:, None, :] - np.array(_OPP["tet"])[None])
    d = pts.shape[1]
    vals = np.zeros((len(pts), 2 * d, d))
    for ax in range(d):
        vals[:, 2 * ax, ax] = pts[:, ax] - 1.0
        vals[:, 2 * ax + 1, ax] = pts[:, ax]
    return vals


def eval_basis(kind, pts, hdiv=False):
    return flux_basis(kind, pts) if hdiv else scalar_basis(kind, pts)
