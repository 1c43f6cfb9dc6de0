"""Device mesh generation (csrc/devmesh.cu) against the reference's numbering.

The reference numbers meshes in `mesh.generate_unit_mesh` / `Mesh._build_facets` /
`_facet_geometry` / `jacobians` (mesh.py:106-277).  The device generator must give the same
arrays bit for bit: against the golden fixtures generated from the unmodified reference, against
the oracle's restatement at larger sizes, and against the host builder (csrc/mesh.cpp) at the
BASELINE config sizes (every array, normals and measures included).
"""

import ctypes as C
import os
import time

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

dpp = pytest.importorskip("paper_1808_08328_b200")
from paper_1808_08328_b200 import _native as N  # noqa: E402
from paper_1808_08328_b200.mesh import Mesh  # noqa: E402

ARRAYS = ("vertices", "cells", "facet_vertex_ids", "cell_facets", "cell_facet_signs", "facet_plus",
          "facet_minus", "facet_normals", "facet_measures")


def device_mesh(dim, kind, n):
    h = C.c_void_p()
    N.call("dpp_mesh_generate_device", N.ctx(), dim, N.KINDS[kind], n, C.byref(h))
    return Mesh(dim, kind, n, None, None, _handle=h)


def host_mesh(dim, kind, n):
    h = C.c_void_p()
    N.call("dpp_mesh_generate", dim, N.KINDS[kind], n, C.byref(h))
    return Mesh(dim, kind, n, None, None, _handle=h)


@pytest.mark.parametrize("dim,kind,n", [(2, "tri", 3), (2, "quad", 3), (3, "tet", 2), (3, "hex", 2),
                                        (2, "tri", 7), (3, "tet", 3)])
def test_device_mesh_matches_reference_golden(golden, dim, kind, n):
    m = device_mesh(dim, kind, n)
    p = f"mesh/{kind}{n}/"
    for a in ("vertices", "cells", "facet_vertex_ids", "cell_facets", "cell_facet_signs",
              "facet_plus", "facet_minus"):
        assert np.array_equal(getattr(m, a), golden[p + a]), a
    J, det = m.jacobians()
    assert np.array_equal(J, golden[p + "J"])
    assert np.array_equal(det, golden[p + "det"])      # numpy's slogdet path, bitwise
    assert np.allclose(m.facet_normals, golden[p + "facet_normals"], rtol=0, atol=1e-15)
    assert np.allclose(m.facet_measures, golden[p + "facet_measures"], rtol=1e-15, atol=0)


@pytest.mark.parametrize("dim,kind,n", [(3, "tet", 12), (2, "tri", 33), (3, "hex", 9), (2, "quad", 17)])
def test_device_mesh_matches_oracle(dim, kind, n):
    m, o = device_mesh(dim, kind, n), oracle.generate_unit_mesh(dim, kind, n)
    for a in ("cells", "facet_vertex_ids", "cell_facets", "cell_facet_signs", "facet_plus",
              "facet_minus", "vertices"):
        assert np.array_equal(getattr(m, a), getattr(o, a)), a
    assert np.array_equal(m.jacobians()[1], o.det)


# n = 1 (every facet on the boundary), odd / prime sizes (many bit-distinct grid spacings), the
# BASELINE config sizes (C0 TRI 64, C1 TRI 256, C2 TET 40, C3 HEX 64: two-key sort, C4 TET 32)
@pytest.mark.parametrize("dim,kind,n", [(2, "tri", 1), (2, "quad", 1), (3, "tet", 1), (3, "hex", 1),
                                        (2, "quad", 49), (3, "tet", 7), (3, "hex", 13),
                                        (2, "tri", 64), (2, "tri", 256), (3, "tet", 40), (3, "hex", 64),
                                        (3, "tet", 32)])
def test_device_mesh_is_bitwise_the_host_builder(dim, kind, n):
    t0 = time.perf_counter()
    d = device_mesh(dim, kind, n)
    t1 = time.perf_counter()
    h = host_mesh(dim, kind, n)
    t2 = time.perf_counter()
    for a in ARRAYS:
        x, y = getattr(d, a), getattr(h, a)
        assert x.dtype == y.dtype and x.shape == y.shape, a
        assert np.array_equal(x, y), a
    assert np.array_equal(d.jacobians()[0], h.jacobians()[0])
    assert np.array_equal(d.jacobians()[1].view(np.int64), h.jacobians()[1].view(np.int64))
    assert np.array_equal(d.interior_facets, h.interior_facets)
    print(f"mesh {kind}{n}: device {1e3 * (t1 - t0):.1f} ms (incl. read-back + numpy export), "
          f"host {1e3 * (t2 - t1):.1f} ms")


@pytest.mark.parametrize("dim,kind,n", [(2, "tri", 300), (2, "quad", 257), (3, "tet", 48), (3, "hex", 72)])
def test_device_mesh_properties_beyond_the_config_sizes(dim, kind, n):
    """Size-independent checks where no reference answer is at hand: closed-form counts, facets in
    lexicographic order without duplicates, plus = lower cell, consistent cell <-> facet tables,
    closed cells (sum of outward measure-weighted normals = 0) and det J = dim! x cell volume."""
    m = device_mesh(dim, kind, n)
    F = {"tri": 3 * n * n + 2 * n, "quad": 2 * n * (n + 1), "tet": 12 * n ** 3 + 6 * n * n,
         "hex": 3 * n * n * (n + 1)}[kind]
    nb = {"tri": 4 * n, "quad": 4 * n, "tet": 12 * n * n, "hex": 6 * n * n}[kind]
    assert m.n_vertices == (n + 1) ** dim and m.n_facets == F and len(m.boundary_facets) == nb
    fv = m.facet_vertex_ids
    assert np.all(np.diff(fv, axis=1) > 0)                       # sorted tuples
    order = np.lexsort(fv.T[::-1])
    assert np.array_equal(order, np.arange(F))                   # lexicographic, hence unique ...
    assert np.all(np.any(fv[1:] != fv[:-1], axis=1))             # ... and no duplicates
    inner = m.facet_minus >= 0
    assert np.all(m.facet_plus[inner] < m.facet_minus[inner])
    nf = m.cell_facets.shape[1]
    cells = np.repeat(np.arange(m.n_cells), nf)
    cf, cs = m.cell_facets.ravel(), m.cell_facet_signs.ravel()
    assert np.array_equal(m.facet_plus[cf[cs > 0]], cells[cs > 0])
    assert np.array_equal(m.facet_minus[cf[cs < 0]], cells[cs < 0])
    assert np.count_nonzero(cs > 0) == F and np.count_nonzero(cs < 0) == F - nb
    flux = np.zeros((m.n_cells, dim))
    np.add.at(flux, cells, (cs * m.facet_measures[cf])[:, None] * m.facet_normals[cf])
    assert np.abs(flux).max() < 1e-14
    J, det = m.jacobians()
    ref = {"tri": 0.5, "quad": 1.0, "tet": 1.0 / 6.0, "hex": 1.0}[kind]
    assert np.all(det > 0) and abs(det.sum() * ref - 1.0) < 1e-12   # the cells tile the unit domain


def test_device_mesh_feeds_the_assembly_without_an_upload():
    """A device-generated mesh is already resident: the assembly uploads nothing for it and gives
    the blocks of the host-numbered mesh bit for bit (H(div) reads the facet arrays too)."""
    p = dpp.DppParameters()
    out = []
    for make in (device_mesh, host_mesh):
        m = make(2, "tri", 24)
        bcs = dpp.boundary_data(dpp.manufactured_solution(2, p), m)
        bs = dpp.assemble(m, "hdiv", p, bcs)
        mb = C.c_int64()
        N.call("dpp_mesh_upload_bytes", m._h, C.byref(mb))
        out.append((bs, mb.value))
    (a, ba), (b, bb) = out
    for name in ("k1_uu", "k1_up", "k1_pu", "k2_uu", "k12_pp"):
        A, B = getattr(a, name), getattr(b, name)
        assert np.array_equal(A.indptr, B.indptr) and np.array_equal(A.indices, B.indices), name
        assert np.array_equal(A.data, B.data), name
    assert bb > ba   # the host-numbered mesh paid for its vertices / cells / facet arrays
    # after a release the device image is rebuilt from the read-back arrays
    p = dpp.DppParameters(gamma_b=(0.0, 0.0, 0.0))
    m = device_mesh(3, "tet", 5)
    N.call("dpp_mesh_release_device", m._h)
    bcs = dpp.boundary_data(dpp.manufactured_solution(3, p), m)
    bs = dpp.assemble(m, "cgvms", p, bcs)
    m2 = host_mesh(3, "tet", 5)
    bs2 = dpp.assemble(m2, "cgvms", p, dpp.boundary_data(dpp.manufactured_solution(3, p), m2))
    assert np.array_equal(bs.k1_uu.data, bs2.k1_uu.data)


def test_generate_unit_mesh_uses_the_device(monkeypatch):
    n0 = N.launches()
    dpp.generate_unit_mesh(3, "hex", 6)
    assert N.launches() > n0
    monkeypatch.setenv("DPP_MESH", "host")
    n0 = N.launches()
    dpp.generate_unit_mesh(3, "hex", 6)
    assert N.launches() == n0
    monkeypatch.setenv("DPP_MESH", "nonsense")
    with pytest.raises(ValueError):
        dpp.generate_unit_mesh(3, "hex", 6)
    with pytest.raises(ValueError):
        device_mesh(2, "tet", 2)
    with pytest.raises(ValueError):
        device_mesh(2, "tri", 0)
