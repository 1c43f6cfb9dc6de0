"""Ten-block four-field assembly on the device (drop-in for dppflow.assembly).

assemble() runs the sm_100a element kernels of csrc/assembly.cu (reference
assembly.py:233-557) and returns a BlockSystem whose blocks live in HBM; the
scipy views of the blocks (k1_uu, ...) are exported lazily on first access,
so code written against the reference keeps working unchanged.
"""

from __future__ import annotations

import ctypes as C
import time
from dataclasses import dataclass, field

import numpy as np
import scipy.sparse as sp

from . import _native as N
from .device import BLOCK_NAMES, DeviceSystem
from .elements import Formulation
from .mesh import Mesh
from .problem import BoundarySpec, DppParameters

FIELDS = ("u1", "p1", "u2", "p2")
FORM_QUAD_DEGREE = 2
DATA_QUAD_DEGREE = 4
_RHS_NAMES = ("f1_u", "f1_p", "f2_u", "f2_p")
_LAZY = frozenset(BLOCK_NAMES + _RHS_NAMES)


@dataclass
class AssemblyStats:
    wall_time_s: float
    nnz: dict


@dataclass
class BlockSystem:
    """Ten-block system with RHS segments (reference assembly.py:48-99).

    Built by assemble(): blocks are device-resident (`_dev`) and exported to
    scipy on first attribute access.  Built by the user from scipy blocks:
    uploaded to the device on first solve.
    """

    formulation: Formulation
    mesh: Mesh | None
    params: DppParameters | None
    k1_uu: sp.csr_matrix = None
    k1_up: sp.csr_matrix = None
    k1_pu: sp.csr_matrix = None
    k1_pp: sp.csr_matrix = None
    k2_uu: sp.csr_matrix = None
    k2_up: sp.csr_matrix = None
    k2_pu: sp.csr_matrix = None
    k2_pp: sp.csr_matrix = None
    k12_pp: sp.csr_matrix = None
    k21_pp: sp.csr_matrix = None
    f1_u: np.ndarray = None
    f1_p: np.ndarray = None
    f2_u: np.ndarray = None
    f2_p: np.ndarray = None
    stats: AssemblyStats | None = None
    _dev: DeviceSystem | None = field(default=None, init=False, repr=False, compare=False)

    def __getattribute__(self, name):
        v = object.__getattribute__(self, name)
        if v is None and name in _LAZY:
            dev = object.__getattribute__(self, "_dev")
            if dev is not None:
                if name in _RHS_NAMES:
                    v = dev.rhs(_RHS_NAMES.index(name))
                else:
                    v = dev.block(BLOCK_NAMES.index(name)).to_scipy()
                object.__setattr__(self, name, v)
        return v

    @property
    def field_sizes(self) -> dict:
        dev = object.__getattribute__(self, "_dev")
        if dev is not None and object.__getattribute__(self, "k1_uu") is None:
            return dict(zip(FIELDS, dev.sizes))
        return {"u1": self.k1_uu.shape[0], "p1": self.k1_pp.shape[0],
                "u2": self.k2_uu.shape[0], "p2": self.k2_pp.shape[0]}

    @property
    def size(self) -> int:
        return sum(self.field_sizes.values())

    def index_sets(self) -> dict:
        out, start = {}, 0
        for name, n in self.field_sizes.items():
            out[name] = np.arange(start, start + n)
            start += n
        return out

    def block_table(self) -> dict:
        return {("u1", "u1"): self.k1_uu, ("u1", "p1"): self.k1_up, ("p1", "u1"): self.k1_pu,
                ("p1", "p1"): self.k1_pp, ("p1", "p2"): self.k12_pp, ("p2", "p1"): self.k21_pp,
                ("u2", "u2"): self.k2_uu, ("u2", "p2"): self.k2_up, ("p2", "u2"): self.k2_pu,
                ("p2", "p2"): self.k2_pp}

    def rhs_segments(self) -> dict:
        return {"u1": self.f1_u, "p1": self.f1_p, "u2": self.f2_u, "p2": self.f2_p}

    def split_solution(self, x: np.ndarray) -> dict:
        # the index sets are contiguous ranges: copies of slices (the reference's x[idx] also copies)
        out, start = {}, 0
        for name, n in self.field_sizes.items():
            out[name] = np.array(x[start:start + n])
            start += n
        return out

    def device(self) -> DeviceSystem:
        """The HBM copy of this system (uploaded from the scipy blocks on first use)."""
        dev = object.__getattribute__(self, "_dev")
        if dev is None:
            blocks = [getattr(self, n) for n in BLOCK_NAMES]
            sizes = [self.k1_uu.shape[0], self.k1_pp.shape[0], self.k2_uu.shape[0], self.k2_pp.shape[0]]
            rhs = [getattr(self, n) for n in _RHS_NAMES]
            dev = DeviceSystem.from_blocks(blocks, rhs, sizes)
            object.__setattr__(self, "_dev", dev)
        return dev


def export_matrix_market(block_system: BlockSystem, path) -> None:
    """Monolithic K in MatrixMarket coordinate format (reference assembly.py:111-116)."""
    from .linalg import write_matrix_market
    K, _ = monolithic_view(block_system)
    write_matrix_market(path, K)


def monolithic_view(block_system: BlockSystem):
    """(K, f) in the (u1, p1, u2, p2) ordering (reference assembly.py:102-108).

    K is built on the device (sp.bmat semantics: sorted, explicit zeros kept)
    and returned as a scipy CSR matrix.
    """
    dev = block_system.device()
    K = dev.monolithic().to_scipy()
    f = np.concatenate([dev.rhs(i) for i in range(4)])
    return K, f


def _pressure_data(mesh: Mesh, bcs: BoundarySpec, net: int):
    """Pressure facets of one network and p0 at their degree-4 quadrature points.
    Returns (pf, p0, device) with device = (kind, coef) when the pressure closure is a
    package manufactured solution the device evaluates itself (p0 is then None)."""
    bf = mesh.boundary_facets
    vel = bcs.velocity_facets[net - 1]
    if vel:
        bf = bf[~np.isin(bf, np.fromiter(vel, dtype=np.int64))]
    pf = N.i64(bf)
    dev = getattr(bcs.p_data[net - 1], "_dpp_device", None)
    if dev is not None:
        return pf, None, dev
    nq = C.c_int()
    N.call("dpp_facet_rule_size", mesh.dim, N.KINDS[mesh.cell_kind.value], DATA_QUAD_DEGREE,
           C.byref(nq))
    X = np.empty((len(pf), nq.value, mesh.dim))
    if len(pf):
        N.call("dpp_facet_points", N.ctx(), mesh._h, DATA_QUAD_DEGREE, len(pf), N.ptr(pf),
               N.ptr(X), None)
    p0 = N.f64(np.asarray(bcs.p_data[net - 1](X.reshape(-1, mesh.dim)), dtype=float)
               .reshape(len(pf), nq.value))
    return pf, p0, None


def fill_bc_pressure(bc, net: int, pf, p0, dev):
    """Pressure-facet part of a dpp_bc (host p0 values or a device-evaluated MMS)."""
    bc.n_pfacets[net - 1] = len(pf)
    bc.pfacets[net - 1] = pf.ctypes.data
    if dev is not None:
        bc.p0_kind[net - 1] = dev[0]
        for i, v in enumerate(dev[1]):
            bc.p0_coef[net - 1][i] = v
    else:
        bc.p0[net - 1] = p0.ctypes.data


def _facet_points(mesh: Mesh, facets: np.ndarray, degree: int):
    """(X, W) of the facet rule on `facets` (reference assembly.py:173-181), from the device."""
    fids = N.i64(facets)
    nq = C.c_int()
    N.call("dpp_facet_rule_size", mesh.dim, N.KINDS[mesh.cell_kind.value], degree, C.byref(nq))
    X = np.empty((len(fids), nq.value, mesh.dim))
    W = np.empty((len(fids), nq.value))
    if len(fids):
        N.call("dpp_facet_points", N.ctx(), mesh._h, degree, len(fids), N.ptr(fids), N.ptr(X), N.ptr(W))
    return X, W


def _velocity_flux_data(mesh: Mesh, bcs: BoundarySpec, net: int):
    """Prescribed flux integrals g_f = sum_q W_fq (u.n)(X_fq) on the velocity facets of one
    network (reference assembly.py:301-309, one callable evaluation per facet)."""
    vel = np.array(sorted(bcs.velocity_facets[net - 1]), dtype=np.int64)
    X, W = _facet_points(mesh, vel, DATA_QUAD_DEGREE)
    g = np.empty(len(vel))
    for i, f in enumerate(vel):
        un = bcs.un_data[net - 1](X[i], mesh.facet_normals[f])
        g[i] = W[i] @ un
    return vel, g


def _pressure_dirichlet_vertices(mesh: Mesh, bcs: BoundarySpec, net: int) -> np.ndarray:
    """Vertices of the pressure facets (reference assembly.py:192-197), sorted."""
    bf = mesh.boundary_facets
    vel = bcs.velocity_facets[net - 1]
    if vel:
        bf = bf[~np.isin(bf, np.fromiter(vel, dtype=np.int64))]
    return np.unique(mesh.facet_vertex_ids[bf].ravel()).astype(np.int64)


def _normal_velocity_dofs(mesh: Mesh, bcs: BoundarySpec, net: int):
    """Config-3 extension: the nodal velocity components normal to the network's velocity
    facets and their prescribed values (u.n = g, bcs.un_data; 0 = no flow).  The structured
    unit meshes have axis-aligned boundary facets, so u.n = g pins component d of every facet
    vertex to g n_d (n = +-e_d)."""
    vel = np.array(sorted(bcs.velocity_facets[net - 1]), dtype=np.int64)
    if not len(vel):
        return np.empty(0, np.int64), np.empty(0)
    nrm = mesh.facet_normals[vel]
    axis = np.argmax(np.abs(nrm), axis=1)
    nd = nrm[np.arange(len(vel)), axis]
    if np.any(np.abs(np.abs(nd) - 1.0) > 1e-12):
        raise ValueError("strong velocity conditions need axis-aligned boundary facets")
    verts = mesh.facet_vertex_ids[vel]                     # (F, nvf)
    dofs = verts * mesh.dim + axis[:, None]
    un = bcs.un_data[net - 1] if bcs.un_data is not None else None
    if un is None:
        vals = np.zeros(verts.shape)
    else:
        vals = np.stack([np.asarray(un(mesh.vertices[verts[i]], nrm[i]), dtype=float) * nd[i]
                         for i in range(len(vel))])
    dofs, vals = dofs.ravel(), vals.ravel()
    order = np.argsort(dofs, kind="stable")
    dofs, vals = dofs[order], vals[order]
    first = np.ones(len(dofs), bool)
    first[1:] = dofs[1:] != dofs[:-1]
    u_d, u_v = dofs[first], vals[first]
    if np.any(np.abs(vals - np.repeat(u_v, np.diff(np.append(np.flatnonzero(first), len(dofs))))) > 1e-12):
        raise ValueError("inconsistent normal velocity data at a shared vertex")
    return u_d.astype(np.int64), u_v


def assemble(mesh: Mesh, formulation, params: DppParameters, bcs: BoundarySpec | None,
             workers: int = 1, pressure_dirichlet: str = "weak", *, cell_permeability=None,
             velocity_dirichlet: str = "natural") -> BlockSystem:
    """Device assembly (reference assembly.py:564-566).  `workers` is accepted
    for API compatibility; the device assembles all cells at once.

    Beyond the reference (BASELINE config 3; parity unpinned):
      cell_permeability=(k1_cells, k2_cells) -- per-cell permeabilities (H(div), CG-VMS)
        replacing params.k1 / k2 cell by cell (mu/k_c and k_c/mu in the cell integrals);
      velocity_dirichlet="strong" (CG-VMS) -- the velocity facets' normal velocity is imposed
        strongly (u.n = bcs.un_data, 0 = no flow) by the reference's symmetric elimination
        (assembly.py:200-226) of the normal components at those facets' vertices.  The
        reference's CG-VMS only drops the pressure functional there ("natural", the default).
    """
    t0 = time.perf_counter()
    form = Formulation(formulation)
    gb = np.asarray(params.gamma_b, dtype=float)
    if gb.shape != (mesh.dim,):
        raise ValueError("gamma_b dimension does not match the mesh")
    if pressure_dirichlet not in ("weak", "strong"):
        raise ValueError("pressure_dirichlet must be 'weak' or 'strong'")
    if pressure_dirichlet == "strong" and form != Formulation.CG_VMS:
        raise ValueError("pressure_dirichlet='strong' is a CG-VMS option (reference assemble_cgvms)")
    if velocity_dirichlet not in ("natural", "strong"):
        raise ValueError("velocity_dirichlet must be 'natural' or 'strong'")
    if velocity_dirichlet == "strong" and form != Formulation.CG_VMS:
        raise ValueError("velocity_dirichlet='strong' is a CG-VMS option (H(div) / DG-VMS impose the flux already)")
    ck = None
    if cell_permeability is not None:
        k1c, k2c = (N.f64(np.asarray(a, dtype=float).ravel()) for a in cell_permeability)
        if len(k1c) != mesh.n_cells or len(k2c) != mesh.n_cells:
            raise ValueError("cell_permeability needs one k1 and one k2 per cell")
        if not (np.all(k1c > 0) and np.all(k2c > 0)):
            raise ValueError("cell permeabilities must be positive")
        ck = (k1c, k2c)
    p = N.Params(params.mu, params.beta, params.k1, params.k2, params.eta_u, params.eta_p,
                 (C.c_double * 3)(*(list(gb) + [0.0] * (3 - len(gb)))))
    keep = []
    bcp = None
    if bcs is not None:
        bc = N.Bc()
        for net in (1, 2):
            pf, p0, dev = _pressure_data(mesh, bcs, net)
            keep += [pf, p0]
            fill_bc_pressure(bc, net, pf, p0, dev)
            if form == Formulation.HDIV and bcs.velocity_facets[net - 1]:
                vel, gflux = _velocity_flux_data(mesh, bcs, net)
                keep += [vel, gflux]
                bc.n_vfacets[net - 1] = len(vel)
                bc.vfacets[net - 1] = vel.ctypes.data
                bc.vdata[net - 1] = gflux.ctypes.data
            elif form == Formulation.DG_VMS and bcs.velocity_facets[net - 1]:
                # (u.n) at the degree-4 points, one callable evaluation per facet (assembly.py:532-534)
                vel = np.array(sorted(bcs.velocity_facets[net - 1]), dtype=np.int64)
                X, _ = _facet_points(mesh, vel, DATA_QUAD_DEGREE)
                un = N.f64(np.stack([np.asarray(bcs.un_data[net - 1](X[i], mesh.facet_normals[f]), dtype=float)
                                     for i, f in enumerate(vel)]) if len(vel) else np.empty((0, 1)))
                keep += [vel, un]
                bc.n_vfacets[net - 1] = len(vel)
                bc.vfacets[net - 1] = vel.ctypes.data
                bc.vdata[net - 1] = un.ctypes.data
        bcp = C.byref(bc)
    h = C.c_void_p()
    if ck is None:
        N.call("dpp_assemble", N.ctx(), mesh._h, N.FORMS[form.value], C.byref(p), bcp, C.byref(h))
    else:
        N.call("dpp_assemble_ext", N.ctx(), mesh._h, N.FORMS[form.value], C.byref(p), N.ptr(ck[0]),
               N.ptr(ck[1]), bcp, C.byref(h))
    dev = DeviceSystem(h)
    if bcs is not None and pressure_dirichlet == "strong":
        # strong boundary pressure: eliminate p1 then p2 (reference assembly.py:410-415)
        for net in (1, 2):
            verts = _pressure_dirichlet_vertices(mesh, bcs, net)
            vals = N.f64(np.asarray(bcs.p_data[net - 1](mesh.vertices[verts]), dtype=float))
            N.call("dpp_system_eliminate", h, 1 if net == 1 else 3, len(verts), N.ptr(verts), N.ptr(vals))
    if bcs is not None and velocity_dirichlet == "strong":
        for net in (1, 2):   # u1 then u2, after the pressure data (as the strong pressure route)
            dofs, vals = _normal_velocity_dofs(mesh, bcs, net)
            if len(dofs):
                dofs, vals = N.i64(dofs), N.f64(vals)
                N.call("dpp_system_eliminate", h, 0 if net == 1 else 2, len(dofs), N.ptr(dofs), N.ptr(vals))
    bs = BlockSystem(formulation=form, mesh=mesh, params=params)
    object.__setattr__(bs, "_dev", dev)
    wall = time.perf_counter() - t0
    bs.stats = AssemblyStats(wall_time_s=wall, nnz=_DeviceNnz(dev))
    return bs


def assemble_hdiv(mesh: Mesh, params: DppParameters, bcs: BoundarySpec | None, workers: int = 1,
                  **extension) -> BlockSystem:
    """Facet-flux velocities, cellwise-constant pressures (reference assembly.py:233)."""
    return assemble(mesh, Formulation.HDIV, params, bcs, workers=workers, **extension)


def assemble_cgvms(mesh: Mesh, params: DppParameters, bcs: BoundarySpec | None, workers: int = 1,
                   pressure_dirichlet: str = "weak", **extension) -> BlockSystem:
    """Continuous equal-order VMS (reference assembly.py:360)."""
    return assemble(mesh, Formulation.CG_VMS, params, bcs, workers=workers, pressure_dirichlet=pressure_dirichlet,
                    **extension)


def assemble_dgvms(mesh: Mesh, params: DppParameters, bcs: BoundarySpec | None, workers: int = 1) -> BlockSystem:
    """Discontinuous VMS with interior-facet couplings (reference assembly.py:449)."""
    return assemble(mesh, Formulation.DG_VMS, params, bcs, workers=workers)


class _DeviceNnz(dict):
    """nnz per block, read from the device lazily (AssemblyStats.nnz)."""

    def __init__(self, dev):
        super().__init__()
        self._dev = dev

    def _fill(self):
        if not super().__len__():
            for i, n in enumerate(BLOCK_NAMES):
                super().__setitem__(n, self._dev.block(i).nnz)

    def __getitem__(self, k):
        self._fill()
        return super().__getitem__(k)

    def items(self):
        self._fill()
        return super().items()

    def keys(self):
        self._fill()
        return super().keys()

    def values(self):
        self._fill()
        return super().values()

    def __iter__(self):
        self._fill()
        return super().__iter__()

    def __len__(self):
        self._fill()
        return super().__len__()


# ----------------------------------------------------------------------------- fields

@dataclass
class DiscreteField:
    """One solution field with per-cell evaluation (reference assembly.py:591-638).

    evaluate_all runs on the device (csrc/fields.cu): nodal P1/Q1 sums for pressures and
    CG/DG velocities, the contravariant Piola map of the RT facet-flux basis for H(div)
    velocities; (C, nq) for pressures, (C, nq, dim) for velocities.
    """

    mesh: Mesh
    formulation: Formulation
    name: str   # u1 | p1 | u2 | p2
    coeffs: np.ndarray

    @property
    def is_velocity(self) -> bool:
        return self.name.startswith("u")

    @property
    def field_index(self) -> int:
        return FIELDS.index(self.name)

    def evaluate_all(self, ref_points) -> np.ndarray:
        mesh = self.mesh
        pts = N.f64(np.atleast_2d(np.asarray(ref_points, dtype=float)))
        if pts.shape[1] != mesh.dim:
            raise ValueError("reference points do not match the mesh dimension")
        coef = N.f64(np.asarray(self.coeffs, dtype=float).ravel())
        nc = mesh.dim if self.is_velocity else 1
        out = np.empty((mesh.n_cells, len(pts), nc))
        N.call("dpp_field_evaluate", N.ctx(), mesh._h, N.FORMS[Formulation(self.formulation).value],
               self.field_index, N.ptr(coef), len(coef), len(pts), N.ptr(pts), N.ptr(out))
        return out if self.is_velocity else out[..., 0]

    def evaluate(self, cell: int, ref_points) -> np.ndarray:
        return self.evaluate_all(ref_points)[cell]


def solution_fields(block_system: BlockSystem, x: np.ndarray) -> dict:
    """{name: DiscreteField} (reference assembly.py:641-644)."""
    parts = block_system.split_solution(x)
    return {name: DiscreteField(block_system.mesh, block_system.formulation, name, parts[name])
            for name in FIELDS}
