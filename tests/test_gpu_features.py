"""GPU parity of the assembly options beyond the benchmark path: body force
(gamma_b != 0, reference assembly.py:274-277 / :352-356), prescribed-flux boundary
facets (H(div) strong elimination :301-309, CG-VMS pressure-functional drop
:424-426) and strong boundary pressure for CG-VMS (:410-415, `_eliminate`
:200-226).  Same bars as test_gpu_parity: patterns bit-exact, entries and RHS
within 1e-12 relative, solutions within 1e-9 relative with iterations +-2.
"""

import numpy as np
import pytest

import oracle
import scipy.sparse as sp

from tests.test_gpu_parity import BLOCKS, entry_close, rel_close, same_pattern, union_close

pytestmark = pytest.mark.gpu

dpp = pytest.importorskip("paper_1808_08328_b200")


def pair(form, dim, kind, n, gamma=None, vel_side=None, strong=False, **kw):
    gb = tuple(gamma) if gamma is not None else (0.0,) * dim
    p = dpp.DppParameters(gamma_b=gb, **kw)
    op = oracle.Params(gamma_b=gb, **kw)
    m = dpp.generate_unit_mesh(dim, kind, n)
    om = oracle.generate_unit_mesh(dim, kind, n)
    vel = (frozenset(), frozenset())
    if vel_side is not None:
        # boundary facets with centroid on x = 0 carry prescribed flux in network 1
        # (and y = 0 in network 2)
        ctr = om.vertices[om.facet_vertex_ids].mean(axis=1)
        bf = np.flatnonzero(om.facet_minus < 0)
        v1 = frozenset(int(f) for f in bf if abs(ctr[f, 0]) < 1e-12)
        v2 = frozenset(int(f) for f in bf if abs(ctr[f, 1]) < 1e-12)
        vel = (v1, v2)
    bcs = dpp.boundary_data(dpp.manufactured_solution(dim, p), m, velocity_facets=vel)
    obcs = oracle.boundary_data(oracle.mms(dim, op), om, velocity_facets=vel)
    pd = "strong" if strong else "weak"
    bs = dpp.assemble(m, form, p, bcs, pressure_dirichlet=pd)
    obs = oracle.assemble(om, form, op, obcs, pressure_dirichlet=pd)
    return bs, obs


def negligible_pattern_diff(A, B, tol=1e-12):
    """Patterns equal except at entries negligible against their row (|v| <= tol row-max):
    CG/DG values are tolerance-equal to the reference, so a cancellation that gives an
    exact 0 on one side and ~1e-17 on the other flips an entry's presence once the
    elimination's products drop exact zeros (scipy csr_matmat)."""
    A, B = sp.csr_matrix(A), sp.csr_matrix(B)
    if A.shape != B.shape:
        return False
    pa, pb = A.copy(), B.copy()
    pa.data[:] = 1.0
    pb.data[:] = 1.0
    only = (pa - pb).tocoo()          # +1: only in A, -1: only in B
    rowmax = np.maximum(abs(A).max(axis=1).toarray().ravel(), abs(B).max(axis=1).toarray().ravel())
    for r, c, s in zip(only.row, only.col, only.data):
        if s == 0:
            continue
        v = A[r, c] if s > 0 else B[r, c]
        if abs(v) > tol * rowmax[r]:
            return False
    return True


def check_system(bs, obs, exact_pattern=True):
    for name in BLOCKS:
        A, B = getattr(bs, name), getattr(obs, name)
        if exact_pattern:
            assert same_pattern(A, B), name
            assert entry_close(A, B, 1e-12), name
        else:
            assert negligible_pattern_diff(A, B, 1e-12), name
            assert union_close(A, B, 1e-12), name
    for name in ("f1_u", "f1_p", "f2_u", "f2_p"):
        assert rel_close(getattr(bs, name), getattr(obs, name), 1e-12), name


def check_solve(bs, obs, method="scale"):
    rep = dpp.solve(bs, dpp.method_config(method, rtol=1e-8))
    orep = oracle.solve(obs, oracle.method_config(method, rtol=1e-8))
    x = rep.solution_vector()
    assert rep.converged and abs(rep.stats.iterations - orep.stats.iterations) <= 2
    assert np.linalg.norm(x - orep.x) / np.linalg.norm(orep.x) < 1e-9


@pytest.mark.parametrize("form,dim,kind,n", [("cgvms", 2, "tri", 8), ("hdiv", 2, "tri", 8), ("dgvms", 2, "tri", 4),
                                             ("cgvms", 3, "tet", 4), ("hdiv", 3, "hex", 3), ("dgvms", 2, "quad", 4)])
def test_body_force(form, dim, kind, n):
    gamma = (0.3, -1.1, 0.7)[:dim]
    bs, obs = pair(form, dim, kind, n, gamma=gamma)
    check_system(bs, obs)
    assert np.any(np.asarray(bs.f1_p) != 0.0) or form == "hdiv"
    check_solve(bs, obs)


@pytest.mark.parametrize("form,dim,kind,n", [("hdiv", 2, "tri", 8), ("cgvms", 2, "quad", 6), ("dgvms", 2, "tri", 4),
                                             ("dgvms", 3, "tet", 2)])
def test_velocity_facets(form, dim, kind, n):
    bs, obs = pair(form, dim, kind, n, vel_side=True)
    check_system(bs, obs)
    check_solve(bs, obs, "field")


def test_velocity_facets_hdiv_3d_system():
    # 3-D H(div) mass values are 1-ulp close, not bitwise (only 2-D H(div) is a config,
    # C1); after the elimination the pressure Schur complement's AMG aggregation hits
    # strength ties that 1-ulp changes flip, so only the assembled system is compared
    bs, obs = pair("hdiv", 3, "tet", 3, vel_side=True)
    check_system(bs, obs)


@pytest.mark.parametrize("dim,kind,n", [(2, "tri", 8), (3, "tet", 3)])
def test_strong_pressure(dim, kind, n):
    bs, obs = pair("cgvms", dim, kind, n, strong=True)
    check_system(bs, obs, exact_pattern=False)
    check_solve(bs, obs)


def test_strong_pressure_with_velocity_facets():
    bs, obs = pair("cgvms", 2, "tri", 6, vel_side=True, strong=True)
    check_system(bs, obs, exact_pattern=False)


def test_strong_is_cgvms_only():
    m = dpp.generate_unit_mesh(2, "tri", 3)
    p = dpp.DppParameters(gamma_b=(0.0, 0.0))
    with pytest.raises(ValueError):
        dpp.assemble(m, "hdiv", p, dpp.boundary_data(dpp.manufactured_solution(2, p), m),
                     pressure_dirichlet="strong")


@pytest.mark.parametrize("dim,kind,n,form", [(2, "tri", 8, "cgvms"), (3, "tet", 4, "cgvms"), (2, "quad", 6, "hdiv"),
                                             (3, "hex", 3, "dgvms")])
def test_device_mms_traces_match_host(dim, kind, n, form):
    """The package's manufactured pressures are evaluated on the device (dpp_bc.p0_kind);
    wrapping them in plain lambdas forces the host path: the RHS must agree."""
    p = dpp.DppParameters(gamma_b=(0.0,) * dim)
    m = dpp.generate_unit_mesh(dim, kind, n)
    mms = dpp.manufactured_solution(dim, p)
    assert hasattr(mms.p1, "_dpp_device") and hasattr(mms.p2, "_dpp_device")
    from paper_1808_08328_b200.problem import ManufacturedSolution
    host = ManufacturedSolution(dim, mms.u1, lambda x: mms.p1(x), mms.u2, lambda x: mms.p2(x))
    a = dpp.assemble(m, form, p, dpp.boundary_data(mms, m))
    b = dpp.assemble(m, form, p, dpp.boundary_data(host, m))
    for name in ("f1_u", "f1_p", "f2_u", "f2_p"):
        assert rel_close(getattr(a, name), getattr(b, name), 1e-13), name


@pytest.mark.gpu
def test_build_preconditioner_honours_monolithic():
    """build_preconditioner(bs, config, monolithic=K) builds the tree from the caller's matrix
    (reference blocksolve.py:288-294): the system's own K gives the same operator bit for bit,
    2K gives (up to rounding) half of it, a wrong shape is rejected."""
    import scipy.sparse as sp
    p = dpp.DppParameters(k2=0.01, gamma_b=(0.0, 0.0, 0.0))
    m = dpp.generate_unit_mesh(3, "tet", 4)
    bs = dpp.assemble(m, "cgvms", p, dpp.boundary_data(dpp.mms_3d(p), m))
    K, _ = dpp.monolithic_view(bs)
    r = np.random.default_rng(3).standard_normal(K.shape[0])
    for meth in ("scale", "field"):
        cfg = dpp.method_config(meth)
        z0 = dpp.build_preconditioner(bs, cfg)(r)
        z1 = dpp.build_preconditioner(bs, cfg, monolithic=K)(r)
        assert np.array_equal(z0, z1)
        z2 = dpp.build_preconditioner(bs, cfg, monolithic=(2.0 * K).tocsr())(r)
        assert np.linalg.norm(z2 - 0.5 * z0) <= 1e-12 * np.linalg.norm(z0)
    with pytest.raises(ValueError):
        dpp.build_preconditioner(bs, dpp.method_config("scale"), monolithic=sp.identity(5, format="csr"))
