"""Pin the CPU oracle against the reference's own outputs (tests/golden).

The fixtures were produced by tests/golden/make_golden.py from the unmodified
reference (`dppflow`).  Integer data and sparsity patterns must match
bit-for-bit; floating-point values are held to 1e-13 relative (they are
bitwise on the generating host; other hosts may pick other BLAS kernels).
"""

import json
import os

import numpy as np
import pytest
import scipy.sparse as sp

import oracle
from oracle import solvers
from tests.conftest import GOLDEN, csr_from

MESHES = [(2, "tri", 3), (2, "quad", 3), (3, "tet", 2), (3, "hex", 2), (2, "tri", 7), (3, "tet", 3)]
BLOCKS = ("k1_uu", "k1_up", "k1_pu", "k1_pp", "k2_uu", "k2_up", "k2_pu", "k2_pp", "k12_pp", "k21_pp")


def close(a, b, tol=1e-13):
    a, b = np.asarray(a, float), np.asarray(b, float)
    assert a.shape == b.shape
    scale = max(1.0, float(np.max(np.abs(b)))) if b.size else 1.0
    assert np.max(np.abs(a - b), initial=0.0) <= tol * scale


def same_csr(A, B, tol=1e-13):
    A, B = sp.csr_matrix(A), sp.csr_matrix(B)
    assert A.shape == B.shape
    assert np.array_equal(A.indptr, B.indptr)
    assert np.array_equal(A.indices, B.indices)
    close(A.data, B.data, tol)


def system(form, dim, kind, n, **kw):
    p = oracle.Params(gamma_b=(0.0,) * dim, **kw)
    m = oracle.generate_unit_mesh(dim, kind, n)
    return oracle.assemble(m, form, p, oracle.boundary_data(oracle.mms(dim, p), m))


@pytest.mark.parametrize("dim,kind,n", MESHES)
def test_mesh_numbering_bit_exact(golden, dim, kind, n):
    m = oracle.generate_unit_mesh(dim, kind, n)
    p = f"mesh/{kind}{n}/"
    for a in ("cells", "facet_vertex_ids", "cell_facets", "cell_facet_signs", "facet_plus",
              "facet_minus"):
        assert np.array_equal(getattr(m, a), golden[p + a]), a
    assert np.array_equal(m.vertices, golden[p + "vertices"])
    assert np.array_equal(m.J, golden[p + "J"])
    assert np.array_equal(m.det, golden[p + "det"])
    close(m.facet_normals, golden[p + "facet_normals"], 1e-15)
    close(m.facet_measures, golden[p + "facet_measures"], 1e-15)


@pytest.mark.parametrize("form", ["hdiv", "cgvms", "dgvms"])
@pytest.mark.parametrize("dim,kind,n", MESHES[:4])
def test_assembly_matches_reference(golden, form, dim, kind, n):
    bs = system(form, dim, kind, n)
    p = f"asm/{form}/{kind}{n}/"
    for b in BLOCKS:
        same_csr(getattr(bs, b), csr_from(golden, p + b))
    for r in ("f1_u", "f1_p", "f2_u", "f2_p"):
        close(getattr(bs, r), golden[p + r])
    K, _ = oracle.monolithic_view(bs)
    same_csr(K, csr_from(golden, p + "K"))


@pytest.mark.parametrize("form", ["cgvms", "hdiv"])
def test_linalg_primitives_match_reference(golden, form):
    bs = system(form, 2, "tri", 4)
    p = f"lin/{form}/tri4/"
    f = oracle.ilu0(bs.k1_uu)
    same_csr(f.L, csr_from(golden, p + "L"))
    same_csr(f.U, csr_from(golden, p + "U"))
    close(oracle.apply_ilu0(f, golden[p + "ilu_r"]), golden[p + "ilu_z"], 1e-12)
    S = oracle.schur_selfp(bs.k1_pp, bs.k1_pu, oracle.diag_lump(bs.k1_uu), bs.k1_up)
    same_csr(S, csr_from(golden, p + "S"), 0.0)          # bitwise: AMG is ulp-sensitive
    h = oracle.amg_setup(S)
    assert h.level_count == int(golden[p + "amg_levels"])
    for li, lv in enumerate(h.levels):
        same_csr(lv.A, csr_from(golden, p + f"amg{li}.A"), 1e-12)
        if lv.P is not None:
            assert np.array_equal(lv.agg, golden[p + f"amg{li}.agg"])
            same_csr(lv.P, csr_from(golden, p + f"amg{li}.P"), 1e-12)
    close(oracle.amg_vcycle(h, golden[p + "vc_r"]), golden[p + "vc_z"], 1e-11)
    K, rhs = oracle.monolithic_view(bs)
    for meth in ("scale", "field"):
        pc = oracle.build_preconditioner(bs, oracle.method_config(meth))
        close(pc(golden[p + f"pc_{meth}_r"]), golden[p + f"pc_{meth}_z"], 1e-11)
        x, st = oracle.gmres(K, rhs, preconditioner=pc, rtol=1e-8)
        assert st.iterations == int(golden[p + f"gmres_{meth}_its"])
        close(st.history, golden[p + f"gmres_{meth}_hist"], 1e-10)
        close(x, golden[p + f"gmres_{meth}_x"], 1e-10)


def test_poisson_amg_matches_reference(golden):
    A = sp.diags([-np.ones(254), 2.0 * np.ones(255), -np.ones(254)], [-1, 0, 1], format="csr")
    h = oracle.amg_setup(A)
    for li, lv in enumerate(h.levels):
        same_csr(lv.A, csr_from(golden, f"lin/poisson255/amg{li}.A"), 1e-12)
        if lv.P is not None:
            same_csr(lv.P, csr_from(golden, f"lin/poisson255/amg{li}.P"), 1e-12)
    close(oracle.amg_vcycle(h, golden["lin/poisson255/vc_r"]), golden["lin/poisson255/vc_z"], 1e-11)


@pytest.mark.parametrize("form", ["hdiv", "cgvms", "dgvms"])
@pytest.mark.parametrize("dim,kind,n", MESHES[:4])
@pytest.mark.parametrize("meth", ["scale", "field"])
def test_solves_match_reference(golden, form, dim, kind, n, meth):
    bs = system(form, dim, kind, n)
    rep = oracle.solve(bs, oracle.method_config(meth, rtol=1e-8))
    p = f"solve/{form}/{kind}{n}/{meth}/"
    assert rep.stats.iterations == int(golden[p + "its"])
    xr = golden[p + "x"]
    assert np.linalg.norm(rep.x - xr) / np.linalg.norm(xr) < 1e-12


def _summary():
    with open(os.path.join(GOLDEN, "summary.json")) as fh:
        return json.load(fh)


@pytest.mark.parametrize("key", sorted(_summary()))
def test_medium_size_summaries(key):
    import hashlib
    s = _summary()[key]
    form, mk, meth, rtol, k2 = key.split("/")
    kind = mk.rstrip("0123456789")
    n = int(mk[len(kind):])
    dim = 2 if kind in ("tri", "quad") else 3
    bs = system(form, dim, kind, n, k2=float(k2.split("=")[1]))
    K, f = oracle.monolithic_view(bs)
    assert K.nnz == s["K_nnz"] and K.shape[0] == s["dof"]
    sha = lambda a: hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()  # noqa: E731
    assert sha(K.indptr.astype(np.int64)) == s["K_sha_indptr"]
    assert sha(K.indices.astype(np.int64)) == s["K_sha_indices"]
    S = oracle.schur_selfp(bs.k1_pp, bs.k1_pu, oracle.diag_lump(bs.k1_uu), bs.k1_up)
    assert S.nnz == s["S_nnz"]
    h = oracle.amg_setup(S)
    assert [lv.A.shape[0] for lv in h.levels] == s["amg_sizes"]
    assert [sha(lv.agg.astype(np.int64)) for lv in h.levels[:-1]] == s["agg_sha"]
    rep = oracle.solve(bs, oracle.method_config(meth, rtol=float(rtol)))
    assert rep.stats.iterations == s["its"]
    assert abs(np.linalg.norm(rep.x) - s["x_norm"]) <= 1e-9 * s["x_norm"]
