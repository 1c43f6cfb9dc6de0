"""Oracle: ten-block four-field assembly (H(div), CG-VMS, DG-VMS).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Restates reference assembly.py:
  :102-108  monolithic (u1,p1,u2,p2) CSR via sp.bmat
  :123-147  COO accumulation -> CSR (duplicates summed, explicit zeros kept, sorted)
  :161-189  facet quadrature and nodal traces
  :200-226  symmetric strong elimination
  :233-311  H(div) facet-flux / cellwise-constant assembly and boundary data
  :318-349  VMS cell blocks (uu, up, pu, pp, cross mass)
  :360-436  CG-VMS assembly and the -(w.n, p0) boundary functional
  :449-557  DG-VMS cell + interior facet consistency / penalty terms
The per-cell arithmetic uses the same numpy contractions as the reference so
that values are bitwise reproducible on the same host.
"""

from __future__ import annotations

import time
from dataclasses import dataclass

import numpy as np
import scipy.sparse as sp

from .geometry import CellKind, gauss01, quadrature_rule, scalar_basis, flux_basis

FIELDS = ("u1", "p1", "u2", "p2")
BLOCK_KEYS = (("u1", "u1"), ("u1", "p1"), ("p1", "u1"), ("p1", "p1"), ("u2", "u2"),
              ("u2", "p2"), ("p2", "u2"), ("p2", "p2"), ("p1", "p2"), ("p2", "p1"))
BLOCK_ATTR = ("k1_uu", "k1_up", "k1_pu", "k1_pp", "k2_uu", "k2_up", "k2_pu", "k2_pp",
              "k12_pp", "k21_pp")


@dataclass
class OBlockSystem:
    formulation: str
    mesh: object
    params: object
    blocks: dict          # attr name -> csr
    rhs: dict             # field -> ndarray
    wall_time_s: float = 0.0

    def __getattr__(self, k):
        b = self.__dict__.get("blocks", {})
        if k in b:
            return b[k]
        r = self.__dict__.get("rhs", {})
        m = {"f1_u": "u1", "f1_p": "p1", "f2_u": "u2", "f2_p": "p2"}
        if k in m:
            return r[m[k]]
        raise AttributeError(k)

    @property
    def field_sizes(self):
        return {"u1": self.blocks["k1_uu"].shape[0], "p1": self.blocks["k1_pp"].shape[0],
                "u2": self.blocks["k2_uu"].shape[0], "p2": self.blocks["k2_pp"].shape[0]}

    @property
    def size(self):
        return sum(self.field_sizes.values())

    def table(self):
        return {key: self.blocks[a] for key, a in zip(BLOCK_KEYS, BLOCK_ATTR)}

    def split_solution(self, x):
        out, s = {}, 0
        for f in FIELDS:
            n = self.field_sizes[f]
            out[f] = x[s:s + n]
            s += n
        return out


def monolithic_view(bs):
    t = bs.table()
    K = sp.bmat([[t.get((r, c)) for c in FIELDS] for r in FIELDS], format="csr")
    return K, np.concatenate([bs.rhs[f] for f in FIELDS])


class _Acc:
    def __init__(self, shape):
        self.shape, self.r, self.c, self.v = shape, [], [], []

    def add(self, loc, rows, cols):
        self.r.append(np.broadcast_to(rows[:, :, None], loc.shape).ravel())
        self.c.append(np.broadcast_to(cols[:, None, :], loc.shape).ravel())
        self.v.append(np.ascontiguousarray(loc).ravel())

    def csr(self):
        if not self.v:
            return sp.csr_matrix(self.shape)
        A = sp.csr_matrix((np.concatenate(self.v), (np.concatenate(self.r), np.concatenate(self.c))),
                          shape=self.shape)
        A.sum_duplicates()
        A.sort_indices()
        return A


def _blocks(nu, npr):
    shapes = {"uu": (nu, nu), "up": (nu, npr), "pu": (npr, nu), "pp": (npr, npr)}
    acc = {f"{b}{n}": _Acc(s) for n in (1, 2) for b, s in shapes.items()}
    acc["pp12"] = _Acc((npr, npr))
    acc["pp21"] = _Acc((npr, npr))
    return acc


def _table(acc):
    names = ("uu1", "up1", "pu1", "pp1", "uu2", "up2", "pu2", "pp2", "pp12", "pp21")
    return {key: acc[n].csr() for key, n in zip(BLOCK_KEYS, names)}


def _facet_points(mesh, fids, degree):
    """Physical facet quadrature points (F,nq,dim), weights (F,nq) (assembly.py:161-181)."""
    if mesh.dim == 2:
        t, w = gauss01(int(np.ceil((degree + 1) / 2)))
        ref, wref, rm = t[:, None], w, 1.0
    elif mesh.kind == "tet":
        ref, wref = quadrature_rule("tri", degree)
        rm = 0.5
    else:
        ref, wref = quadrature_rule("quad", degree)
        rm = 1.0
    verts = mesh.vertices[mesh.facet_vertex_ids[fids]]
    v0 = verts[:, 0]
    X = v0[:, None, :] + np.einsum("qk,fki->fqi", ref, verts[:, 1:1 + ref.shape[1]] - v0[:, None, :])
    W = wref[None, :] * (mesh.facet_measures[fids] / rm)[:, None]
    return X, W


def _trace(mesh, Jinv, origin, cells, X):
    Xh = np.einsum("fij,fqj->fqi", Jinv[cells], X - origin[cells][:, None, :])
    vals, _ = scalar_basis(mesh.kind, Xh.reshape(-1, mesh.dim))
    return vals.reshape(len(cells), X.shape[1], -1)


def _pressure_facets(mesh, bcs, net):
    return np.array([f for f in mesh.boundary_facets if not bcs.is_velocity_facet(net, int(f))],
                    dtype=np.int64)


def _eliminate(table, rhs, sizes, field, idx, values):
    """Strong elimination (assembly.py:200-226)."""
    if len(idx) == 0:
        return
    n = sizes[field]
    lift = np.zeros(n)
    lift[idx] = values
    keep = np.ones(n)
    keep[idx] = 0.0
    Dk, Dp = sp.diags(keep), sp.diags(1.0 - keep)
    for (r, c), B in list(table.items()):
        if B is None:
            continue
        if c == field:
            rhs[r] = rhs[r] - B @ lift
            B = B @ Dk
        if r == field:
            B = Dk @ B
        table[(r, c)] = B
    table[(field, field)] = table[(field, field)] + Dp
    rhs[field][idx] = values


def _vms_cells(mesh, p, cell_k=None):
    """Cell integrals of the stabilised forms (assembly.py:318-349).

    cell_k = (k1_cells, k2_cells): the config-3 extension (per-cell permeability; the reference
    has scalar k only) -- mu/k_c and k_c/mu per cell, in the scalar path's operation order, so
    constant arrays reproduce the reference bit for bit."""
    dim = mesh.dim
    q, w = quadrature_rule(mesh.kind, 2)
    N, G = scalar_basis(mesh.kind, q)
    nn = N.shape[1]
    J, det = mesh.J, mesh.det
    Jinv = np.linalg.inv(J)
    Gp = np.einsum("qaj,cji->cqai", G, Jinv)
    mass = det[:, None, None] * np.einsum("q,qa,qb->ab", w, N, N)[None]
    gg = det[:, None, None] * np.einsum("q,cqai,cqbi->cab", w, Gp, Gp)
    gn = det[:, None, None, None] * np.einsum("q,cqai,qb->cabi", w, Gp, N)
    C = len(det)
    out = {}
    for net, k in ((1, p.k1), (2, p.k2)):
        if cell_k is None:
            uu = 0.5 * p.mu / k * np.einsum("cab,ij->caibj", mass, np.eye(dim))
        else:
            kc = np.asarray(cell_k[net - 1], dtype=float)
            uu = (0.5 * p.mu / kc)[:, None, None, None, None] * np.einsum("cab,ij->caibj", mass, np.eye(dim))
        up = -(gn + 0.5 * gn.transpose(0, 2, 1, 3)).transpose(0, 1, 3, 2)
        pu = gn.transpose(0, 2, 1, 3) + 0.5 * gn
        if cell_k is None:
            pp = 0.5 * k / p.mu * gg + p.beta / p.mu * mass
        else:
            pp = (0.5 * kc / p.mu)[:, None, None] * gg + p.beta / p.mu * mass
        out[net] = (uu.reshape(C, nn * dim, nn * dim), up.reshape(C, nn * dim, nn),
                    pu.reshape(C, nn, nn * dim), pp)
    return out, mass, N, Gp, w, det, Jinv


def _body_force(p, k, N, Gp, w, det, gb):
    iN = np.einsum("q,qa->a", w, N)
    fu = 0.5 * det[:, None, None] * iN[None, :, None] * gb[None, None, :]
    kk = np.asarray(k, dtype=float)
    fp = ((0.5 * kk / p.mu * det)[:, None] if kk.ndim else 0.5 * k / p.mu * det[:, None]) * \
        np.einsum("q,cqai,i->ca", w, Gp, gb)
    return fu, fp


def _normal_velocity_dofs(mesh, bcs, net):
    """Config-3 extension (CG-VMS, velocity_dirichlet="strong"): component d = axis of the
    normal of every velocity-facet vertex, value g n_d (u.n = g from un_data, 0 = no flow)."""
    vel = np.array(sorted(bcs.velocity_facets[net - 1]), dtype=np.int64)
    if not len(vel):
        return np.empty(0, np.int64), np.empty(0)
    out = {}
    for f in vel:
        nrm = mesh.facet_normals[f]
        d = int(np.argmax(np.abs(nrm)))
        if abs(abs(nrm[d]) - 1.0) > 1e-12:
            raise ValueError("strong velocity conditions need axis-aligned boundary facets")
        vs = mesh.facet_vertex_ids[f]
        un = bcs.un_data[net - 1] if bcs.un_data is not None else None
        g = np.zeros(len(vs)) if un is None else np.asarray(un(mesh.vertices[vs], nrm), dtype=float) * nrm[d]
        for v, val in zip(vs, g):
            out.setdefault(int(v) * mesh.dim + d, float(val))
    idx = np.array(sorted(out), dtype=np.int64)
    return idx, np.array([out[i] for i in idx])


def _nodal_pressure_rhs(mesh, bcs, Jinv, origin, dm_u, rhs):
    for net in (1, 2):
        pf = _pressure_facets(mesh, bcs, net)
        if not len(pf):
            continue
        X, W = _facet_points(mesh, pf, 4)
        cells = mesh.facet_plus[pf]
        N = _trace(mesh, Jinv, origin, cells, X)
        p0 = bcs.p_data[net - 1](X.reshape(-1, mesh.dim)).reshape(W.shape)
        c = -np.einsum("fq,fq,fqa,fi->fai", W, p0, N, mesh.facet_normals[pf])
        np.add.at(rhs[f"u{net}"], dm_u[cells].ravel(), c.reshape(len(pf), -1).ravel())


def assemble(mesh, formulation, p, bcs, pressure_dirichlet="weak", cell_k=None, velocity_dirichlet="natural"):
    formulation = getattr(formulation, "value", formulation)
    t0 = time.perf_counter()
    gb = np.asarray(p.gamma_b, dtype=float)
    if gb.shape != (mesh.dim,):
        raise ValueError("gamma_b dimension does not match the mesh")
    if cell_k is not None and formulation == "dgvms":
        raise ValueError("per-cell permeability is implemented for H(div) and CG-VMS")
    if velocity_dirichlet == "strong" and formulation != "cgvms":
        raise ValueError("velocity_dirichlet='strong' is a CG-VMS option")
    if formulation == "hdiv":
        table, rhs = _hdiv(mesh, p, bcs, gb, cell_k)
    elif formulation == "cgvms":
        table, rhs = _cgvms(mesh, p, bcs, gb, pressure_dirichlet, cell_k, velocity_dirichlet)
    elif formulation == "dgvms":
        table, rhs = _dgvms(mesh, p, bcs, gb)
    else:
        raise ValueError(formulation)
    blocks = {}
    for key, a in zip(BLOCK_KEYS, BLOCK_ATTR):
        B = table[key].tocsr()
        B.sort_indices()
        blocks[a] = B
    return OBlockSystem(formulation, mesh, p, blocks, rhs, time.perf_counter() - t0)


def _hdiv(mesh, p, bcs, gb, cell_k=None):
    dim, C = mesh.dim, mesh.n_cells
    J, det = mesh.J, mesh.det
    nu, npr = mesh.n_facets, C
    q, w = quadrature_rule(mesh.kind, 2)
    Vref = flux_basis(mesh.kind, q)
    dm_u, sc = mesh.cell_facets, mesh.cell_facet_signs.astype(float)
    dm_p = np.arange(C, dtype=np.int64)[:, None]
    acc = _blocks(nu, npr)
    fu = {1: np.zeros(nu), 2: np.zeros(nu)}
    fp = {1: np.zeros(npr), 2: np.zeros(npr)}
    Vp = np.einsum("cij,qfj->cqfi", J, Vref) / det[:, None, None, None]
    mass = np.einsum("q,cqfi,cqgi->cfg", w, Vp, Vp) * det[:, None, None]
    mass = mass * sc[:, :, None] * sc[:, None, :]
    vol = det * w.sum()
    ones = np.ones((C, 1, 1))
    for net, k in ((1, p.k1), (2, p.k2)):
        if cell_k is None:
            acc[f"uu{net}"].add(p.mu / k * mass, dm_u, dm_u)
        else:
            acc[f"uu{net}"].add((p.mu / np.asarray(cell_k[net - 1], dtype=float))[:, None, None] * mass, dm_u, dm_u)
        acc[f"up{net}"].add(-sc[:, :, None], dm_u, dm_p)
        acc[f"pu{net}"].add(sc[:, None, :], dm_p, dm_u)
        acc[f"pp{net}"].add(p.beta / p.mu * vol[:, None, None] * ones, dm_p, dm_p)
        if np.any(gb):
            f = np.einsum("q,cqfi,i->cf", w, Vp, gb) * det[:, None] * sc
            np.add.at(fu[net], dm_u.ravel(), f.ravel())
    cross = -p.beta / p.mu * vol[:, None, None] * ones
    acc["pp12"].add(cross, dm_p, dm_p)
    acc["pp21"].add(cross, dm_p, dm_p)
    table = _table(acc)
    rhs = {"u1": fu[1], "p1": fp[1], "u2": fu[2], "p2": fp[2]}
    if bcs is not None:
        for net in (1, 2):
            pf = _pressure_facets(mesh, bcs, net)
            if len(pf):
                X, W = _facet_points(mesh, pf, 4)
                p0 = bcs.p_data[net - 1](X.reshape(-1, dim)).reshape(W.shape)
                np.add.at(rhs[f"u{net}"], pf, -np.einsum("fq,fq->f", W, p0) / mesh.facet_measures[pf])
            vel = np.array(sorted(bcs.velocity_facets[net - 1]), dtype=np.int64)
            if len(vel):
                X, W = _facet_points(mesh, vel, 4)
                g = np.array([W[i] @ bcs.un_data[net - 1](X[i], mesh.facet_normals[f])
                              for i, f in enumerate(vel)])
                _eliminate(table, rhs, {"u1": nu, "p1": npr, "u2": nu, "p2": npr}, f"u{net}", vel, g)
    return table, rhs


def _cgvms(mesh, p, bcs, gb, pressure_dirichlet, cell_k=None, velocity_dirichlet="natural"):
    dim, C, V = mesh.dim, mesh.n_cells, mesh.n_vertices
    nu, npr = V * dim, V
    dm_p = mesh.cells
    dm_u = (mesh.cells[:, :, None] * dim + np.arange(dim)).reshape(C, -1)
    acc = _blocks(nu, npr)
    fu = {1: np.zeros(nu), 2: np.zeros(nu)}
    fp = {1: np.zeros(npr), 2: np.zeros(npr)}
    nets, mass, N, Gp, w, det, Jinv = _vms_cells(mesh, p, cell_k)
    for net, k in ((1, p.k1), (2, p.k2)):
        uu, up, pu, pp = nets[net]
        acc[f"uu{net}"].add(uu, dm_u, dm_u)
        acc[f"up{net}"].add(up, dm_u, dm_p)
        acc[f"pu{net}"].add(pu, dm_p, dm_u)
        acc[f"pp{net}"].add(pp, dm_p, dm_p)
        if np.any(gb):
            a, b = _body_force(p, k if cell_k is None else cell_k[net - 1], N, Gp, w, det, gb)
            np.add.at(fu[net], dm_u.ravel(), a.ravel())
            np.add.at(fp[net], dm_p.ravel(), b.ravel())
    cross = -p.beta / p.mu * mass
    acc["pp12"].add(cross, dm_p, dm_p)
    acc["pp21"].add(cross, dm_p, dm_p)
    table = _table(acc)
    rhs = {"u1": fu[1], "p1": fp[1], "u2": fu[2], "p2": fp[2]}
    if bcs is not None:
        origin = mesh.vertices[mesh.cells[:, 0]]
        _nodal_pressure_rhs(mesh, bcs, Jinv, origin, dm_u, rhs)
        if pressure_dirichlet == "strong":
            sizes = {"u1": nu, "p1": npr, "u2": nu, "p2": npr}
            for net in (1, 2):
                ids = set()
                for f in mesh.boundary_facets:
                    if not bcs.is_velocity_facet(net, int(f)):
                        ids.update(int(v) for v in mesh.facet_vertex_ids[f])
                verts = np.array(sorted(ids), dtype=np.int64)
                _eliminate(table, rhs, sizes, f"p{net}", verts,
                           bcs.p_data[net - 1](mesh.vertices[verts]))
        elif pressure_dirichlet != "weak":
            raise ValueError("pressure_dirichlet must be 'weak' or 'strong'")
        if velocity_dirichlet == "strong":
            sizes = {"u1": nu, "p1": npr, "u2": nu, "p2": npr}
            for net in (1, 2):
                idx, vals = _normal_velocity_dofs(mesh, bcs, net)
                _eliminate(table, rhs, sizes, f"u{net}", idx, vals)
        elif velocity_dirichlet != "natural":
            raise ValueError("velocity_dirichlet must be 'natural' or 'strong'")
    return table, rhs


def _dgvms(mesh, p, bcs, gb):
    dim, C = mesh.dim, mesh.n_cells
    nn = CellKind.NODES[mesh.kind]
    npr = C * nn
    nu = npr * dim
    h = mesh.h
    dm_p = np.arange(C, dtype=np.int64)[:, None] * nn + np.arange(nn)
    dm_u = (dm_p[:, :, None] * dim + np.arange(dim)).reshape(C, -1)
    acc = _blocks(nu, npr)
    fu = {1: np.zeros(nu), 2: np.zeros(nu)}
    fp = {1: np.zeros(npr), 2: np.zeros(npr)}
    nets, mass, N, Gp, w, det, Jinv = _vms_cells(mesh, p)
    origin = mesh.vertices[mesh.cells[:, 0]]
    for net, k in ((1, p.k1), (2, p.k2)):
        uu, up, pu, pp = nets[net]
        acc[f"uu{net}"].add(uu, dm_u, dm_u)
        acc[f"up{net}"].add(up, dm_u, dm_p)
        acc[f"pu{net}"].add(pu, dm_p, dm_u)
        acc[f"pp{net}"].add(pp, dm_p, dm_p)
        if np.any(gb):
            a, b = _body_force(p, k, N, Gp, w, det, gb)
            np.add.at(fu[net], dm_u.ravel(), a.ravel())
            np.add.at(fp[net], dm_p.ravel(), b.ravel())
    cross = -p.beta / p.mu * mass
    acc["pp12"].add(cross, dm_p, dm_p)
    acc["pp21"].add(cross, dm_p, dm_p)
    ids = mesh.interior_facets
    if len(ids):
        X, W = _facet_points(mesh, ids, 2)
        nrm = mesh.facet_normals[ids]
        cp, cm = mesh.facet_plus[ids], mesh.facet_minus[ids]
        sides = {+1: (cp, _trace(mesh, Jinv, origin, cp, X)),
                 -1: (cm, _trace(mesh, Jinv, origin, cm, X))}
        F_ = len(ids)
        for ss, (cs, Ns) in sides.items():
            for st, (ct, Nt) in sides.items():
                F = np.einsum("fq,fqa,fqb->fab", W, Ns, Nt)
                Fs = np.einsum("fab,fi->faib", F, nrm).reshape(F_, nn * dim, nn)
                Ft = np.einsum("fab,fj->fabj", F, nrm).reshape(F_, nn, nn * dim)
                Fnn = np.einsum("fab,fi,fj->faibj", F, nrm, nrm).reshape(F_, nn * dim, nn * dim)
                for net, k in ((1, p.k1), (2, p.k2)):
                    acc[f"up{net}"].add(0.5 * ss * Fs, dm_u[cs], dm_p[ct])
                    acc[f"pu{net}"].add(-0.5 * st * Ft, dm_p[cs], dm_u[ct])
                    acc[f"uu{net}"].add(p.eta_u * h * p.mu / k * ss * st * Fnn, dm_u[cs], dm_u[ct])
                    acc[f"pp{net}"].add(p.eta_p / h * k / p.mu * ss * st * F, dm_p[cs], dm_p[ct])
    if bcs is not None:
        for net in (1, 2):
            vel = np.array(sorted(bcs.velocity_facets[net - 1]), dtype=np.int64)
            if not len(vel):
                continue
            Xv, Wv = _facet_points(mesh, vel, 2)
            cv = mesh.facet_plus[vel]
            Nv = _trace(mesh, Jinv, origin, cv, Xv)
            nv = mesh.facet_normals[vel]
            F = np.einsum("fq,fqa,fqb->fab", Wv, Nv, Nv)
            acc[f"up{net}"].add(np.einsum("fab,fi->faib", F, nv).reshape(len(vel), nn * dim, nn),
                                dm_u[cv], dm_p[cv])
            acc[f"pu{net}"].add(-np.einsum("fab,fj->fabj", F, nv).reshape(len(vel), nn, nn * dim),
                                dm_p[cv], dm_u[cv])
            Xd, Wd = _facet_points(mesh, vel, 4)
            Nd = _trace(mesh, Jinv, origin, cv, Xd)
            un = np.stack([bcs.un_data[net - 1](Xd[i], nv[i]) for i in range(len(vel))])
            np.add.at(fp[net], dm_p[cv].ravel(), (-np.einsum("fq,fq,fqa->fa", Wd, un, Nd)).ravel())
    table = _table(acc)
    rhs = {"u1": fu[1], "p1": fp[1], "u2": fu[2], "p2": fp[2]}
    if bcs is not None:
        _nodal_pressure_rhs(mesh, bcs, Jinv, origin, dm_u, rhs)
    return table, rhs
