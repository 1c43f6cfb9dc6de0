"""GPU parity: libdpp (through the C ABI / Python binding) vs the CPU oracle.

Bars (BASELINE north_star): mesh / DoF numbering / sparsity patterns bit-exact;
assembled values within 1e-12 relative (H(div) bitwise); solutions within
1e-9 relative L2 with iteration counts within +-2.  Tolerances are written in
each assertion.
"""

import numpy as np
import pytest
import scipy.sparse as sp

import oracle
import oracle.solvers as oracle_solvers
from tests.conftest import csr_from

pytestmark = pytest.mark.gpu

dpp = pytest.importorskip("paper_1808_08328_b200")

BLOCKS = ("k1_uu", "k1_up", "k1_pu", "k1_pp", "k2_uu", "k2_up", "k2_pu", "k2_pp", "k12_pp", "k21_pp")
MESHES = [(2, "tri", 3), (2, "quad", 3), (3, "tet", 2), (3, "hex", 2)]


def systems(form, dim, kind, n, **kw):
    p = dpp.DppParameters(gamma_b=(0.0,) * dim, **kw)
    m = dpp.generate_unit_mesh(dim, kind, n)
    bs = dpp.assemble(m, form, p, dpp.boundary_data(dpp.manufactured_solution(dim, p), m))
    op = oracle.Params(gamma_b=(0.0,) * dim, **kw)
    om = oracle.generate_unit_mesh(dim, kind, n)
    obs = oracle.assemble(om, form, op, oracle.boundary_data(oracle.mms(dim, op), om))
    return bs, obs


def rel_close(a, b, tol):
    a, b = np.asarray(a, float), np.asarray(b, float)
    scale = max(float(np.max(np.abs(b), initial=0.0)), 1e-300)
    return float(np.max(np.abs(a - b), initial=0.0)) <= tol * scale


def same_pattern(A, B):
    A, B = sp.csr_matrix(A), sp.csr_matrix(B)
    return A.shape == B.shape and np.array_equal(A.indptr, B.indptr) and np.array_equal(A.indices, B.indices)


def union_close(A, B, tol):
    """max |A - B| over the union pattern <= tol * max|B| (patterns may differ by exact-zero drops)."""
    D = (sp.csr_matrix(A) - sp.csr_matrix(B)).tocsr()
    return float(np.max(np.abs(D.data), initial=0.0)) <= tol * float(np.max(np.abs(sp.csr_matrix(B).data)))


def entry_close(A, B, tol=1e-12):
    """|a-b| <= tol * max(|b|, row-max |b|) entrywise."""
    A, B = sp.csr_matrix(A), sp.csr_matrix(B)
    if B.nnz == 0:
        return A.nnz == 0 or np.all(A.data == 0)
    rowmax = np.maximum.reduceat(np.abs(B.data), B.indptr[:-1][np.diff(B.indptr) > 0])
    rm = np.zeros(B.shape[0])
    rm[np.diff(B.indptr) > 0] = rowmax
    scale = np.maximum(np.abs(B.data), np.repeat(rm, np.diff(B.indptr)))
    return bool(np.all(np.abs(A.data - B.data) <= tol * np.maximum(scale, 1e-300)))


# ----------------------------------------------------------------------------- SpMV

def test_spmv_matches_scipy(rng):
    A = sp.random(300, 200, density=0.05, random_state=1, format="csr")
    x = rng.standard_normal(200)
    assert np.max(np.abs(dpp.spmv(A, x) - A @ x)) < 1e-14 * max(1, np.abs(A @ x).max())
    I7 = sp.identity(7, format="csr")
    assert np.allclose(dpp.spmv(I7, np.arange(7.0)), np.arange(7.0))
    assert np.allclose(dpp.spmv(sp.csr_matrix((7, 7)), np.ones(7)), 0.0)
    with pytest.raises(ValueError):
        dpp.spmv(sp.identity(3, format="csr"), np.ones(4))


def _spmv_cases(rng):
    """Row-length mixes the SpMV plans must handle: short / long / empty rows, a
    row longer than a CSR-stream block, rows not a multiple of the SELL slice."""
    yield "narrow", sp.random(1003, 900, density=0.004, random_state=2, format="csr")
    yield "wide", sp.random(517, 4000, density=0.03, random_state=3, format="csr")
    lens = rng.integers(0, 60, 2049)
    lens[::97] = 0
    lens[1000] = 5000                      # one row longer than a stream block (2048 entries)
    rows = np.repeat(np.arange(2049), lens)
    cols = np.concatenate([rng.choice(6000, l, replace=False) for l in lens])
    yield "ragged", sp.csr_matrix((rng.standard_normal(rows.size), (rows, cols)), shape=(2049, 6000))
    # a CG-VMS K (explicit zeros, the structured gathers SELL-32 is built for)
    bs, _ = systems("cgvms", 3, "tet", 3)
    yield "K", dpp.monolithic_view(bs)[0]
    # 16-bit SELL codes: four 2^14-column windows per slice exactly at their edges (coded),
    # and a fifth window (the whole matrix falls back to 32-bit columns)
    for name, starts in (("windows4", [0, 20000, 40000, 60000]), ("windows5", [0, 20000, 40000, 60000, 90000])):
        cols = np.concatenate([[s0, s0 + 16383] for s0 in starts])
        nr = 70
        rr = np.repeat(np.arange(nr), cols.size)
        cc = np.tile(cols, nr) + np.repeat(np.arange(nr) % 3, cols.size) * 0
        yield name, sp.csr_matrix((rng.standard_normal(rr.size), (rr, cc)), shape=(nr, 120000))


@pytest.mark.parametrize("sell16", ["1", "0"])
@pytest.mark.parametrize("kind", [0, 1, 2, 3])
def test_spmv_plans_match_scipy(kind, sell16, rng, monkeypatch):
    """Every SpMV kernel (row / CSR-stream / SELL-32 / auto) against scipy's csr_matvec
    (linalg.py:27-32): 1e-14 relative per row; SELL-32 with one warp per slice sums each
    row sequentially in column order and is bitwise equal."""
    import ctypes as C
    from paper_1808_08328_b200 import _native as N
    from paper_1808_08328_b200.device import DeviceCsr
    monkeypatch.setenv("DPP_SELL16", sell16)   # 16-bit SELL column codes (default) / 32-bit
    for name, A in _spmv_cases(rng):
        A = sp.csr_matrix(A)
        A.sort_indices()
        D = DeviceCsr.from_scipy(A)
        N.call("dpp_csr_plan", D.h, kind)
        x = rng.standard_normal(A.shape[1])
        y, ref = D @ x, A @ x
        scale = np.maximum(np.abs(A).dot(np.abs(x)), 1e-300)
        assert np.all(np.abs(y - ref) <= 1e-14 * scale), (name, kind)
        if kind == 2 and A.nnz / A.shape[0] <= 8:
            assert np.array_equal(y, ref), name


# ----------------------------------------------------------------------------- assembly

@pytest.mark.parametrize("form", ["hdiv", "cgvms", "dgvms"])
@pytest.mark.parametrize("dim,kind,n", MESHES)
def test_assembly_matches_oracle(form, dim, kind, n):
    bs, obs = systems(form, dim, kind, n)
    for b in BLOCKS:
        A, B = getattr(bs, b), getattr(obs, b)
        assert same_pattern(A, B), b                     # pattern bit-exact (incl. explicit zeros)
        if form == "hdiv" and dim == 2:
            assert np.array_equal(A.data, B.data), b     # 2D H(div): bitwise (config 1 needs it)
        else:
            assert entry_close(A, B, 1e-12), b
    for r in ("f1_u", "f1_p", "f2_u", "f2_p"):
        assert rel_close(getattr(bs, r), getattr(obs, r), 1e-12), r
    K, f = dpp.monolithic_view(bs)
    Ko, fo = oracle.monolithic_view(obs)
    assert same_pattern(K, Ko)
    assert entry_close(K, Ko, 1e-12)


@pytest.mark.parametrize("form", ["hdiv", "cgvms", "dgvms"])
def test_assembly_matches_reference_golden(golden, form):
    for dim, kind, n in MESHES:
        p = dpp.DppParameters(gamma_b=(0.0,) * dim)
        m = dpp.generate_unit_mesh(dim, kind, n)
        bs = dpp.assemble(m, form, p, dpp.boundary_data(dpp.manufactured_solution(dim, p), m))
        for b in BLOCKS:
            G = csr_from(golden, f"asm/{form}/{kind}{n}/{b}")
            A = getattr(bs, b)
            assert same_pattern(A, G), (kind, b)
            assert entry_close(A, G, 1e-12), (kind, b)


def test_rt0_reference_triangle_known_answer():
    # reference tests/test_assembly.py:43-53
    m = dpp.Mesh(2, dpp.CellKind.TRI, 1, np.array([[0.0, 0.0], [1.0, 0.0], [0.0, 1.0]]),
                 np.array([[0, 1, 2]]))
    bs = dpp.assemble(m, "hdiv", dpp.DppParameters(mu=1.0, k1=1.0, k2=1.0), None)
    expected = np.array([[1 / 3, -1 / 6, 0.0], [-1 / 6, 1 / 3, 0.0], [0.0, 0.0, 1 / 6]])
    assert np.allclose(bs.k1_uu.toarray(), expected, atol=1e-14)
    assert np.allclose(bs.k1_up.toarray().ravel(), [-1.0, -1.0, -1.0], atol=1e-14)


def test_hdiv_tri256_bitwise_diag_and_schur():
    # config 1 (H(div) TRI 256^2) needs bitwise level-0 S_p: its blocks and
    # S_p at the config's own size, bit for bit
    bs, obs = systems("hdiv", 2, "tri", 256)
    for b in BLOCKS:
        assert np.array_equal(getattr(bs, b).data, getattr(obs, b).data), b
    S = dpp.schur_selfp(bs.k1_pp, bs.k1_pu, dpp.diag_lump(bs.k1_uu), bs.k1_up)
    So = oracle.schur_selfp(obs.k1_pp, obs.k1_pu, oracle.diag_lump(obs.k1_uu), obs.k1_up)
    assert same_pattern(S, So) and np.array_equal(S.data, So.data)


# ----------------------------------------------------------------------------- ILU(0)

def poisson_1d(n):
    return sp.diags([-np.ones(n - 1), 2.0 * np.ones(n), -np.ones(n - 1)], [-1, 0, 1], format="csr")


def test_ilu0_exact_on_tridiagonal(rng):
    A = poisson_1d(25)
    f = dpp.ilu0(A)
    b = rng.standard_normal(25)
    assert np.linalg.norm(A @ dpp.apply_ilu0(f, b) - b) < 1e-12


def test_ilu0_errors():
    with pytest.raises(dpp.ZeroPivotError):
        dpp.ilu0(sp.csr_matrix(np.array([[0.0, 1.0], [1.0, 1.0]])))
    A = sp.csr_matrix(np.array([[1.0, 1.0], [1.0, 0.0]]))
    A.eliminate_zeros()
    with pytest.raises(dpp.ZeroPivotError):
        dpp.ilu0(A)


@pytest.mark.parametrize("form,dim,kind,n", [("cgvms", 2, "tri", 6), ("hdiv", 2, "tri", 6),
                                             ("dgvms", 2, "tri", 3), ("cgvms", 3, "tet", 3),
                                             ("cgvms", 3, "hex", 3), ("dgvms", 3, "tet", 2),
                                             # >= 16384 velocity rows: Kronecker factorization
                                             # and component-parallel sweeps (M (x) I_dim)
                                             ("cgvms", 3, "tet", 18), ("cgvms", 2, "tri", 95),
                                             ("dgvms", 3, "tet", 7)])
def test_ilu0_factors_bitwise_and_apply(form, dim, kind, n, rng):
    bs, obs = systems(form, dim, kind, n)
    # same input -> bitwise factors (same IKJ order, separate mul/sub)
    f, fo = dpp.ilu0(obs.k1_uu), oracle.ilu0(obs.k1_uu)
    for X, Xo in ((f.L, fo.L), (f.U, fo.U)):
        assert same_pattern(X, Xo)
        assert np.array_equal(X.data, Xo.data)
    r = rng.standard_normal(bs.k1_uu.shape[0])
    assert rel_close(dpp.apply_ilu0(f, r), oracle.apply_ilu0(fo, r), 1e-11)
    # product's own assembly (entries within 1e-12) -> factors within rounding
    fd = dpp.ilu0(bs.k1_uu)
    assert union_close(fd.U, fo.U, 1e-11) and union_close(fd.L, fo.L, 1e-11)
    assert rel_close(dpp.apply_ilu0(fd, r), oracle.apply_ilu0(fo, r), 1e-10)


# ----------------------------------------------------------------------------- selfp + AMG

@pytest.mark.parametrize("form,dim,kind,n", [("cgvms", 2, "tri", 8), ("hdiv", 2, "tri", 8),
                                             ("dgvms", 2, "tri", 4), ("cgvms", 3, "tet", 4),
                                             ("cgvms", 3, "hex", 4), ("hdiv", 3, "tet", 2)])
def test_selfp_and_amg_match_oracle(form, dim, kind, n, rng):
    bs, obs = systems(form, dim, kind, n)
    # same inputs -> bitwise S_p (scipy csr_matmat order reproduced)
    Sx = dpp.schur_selfp(obs.k1_pp, obs.k1_pu, oracle.diag_lump(obs.k1_uu), obs.k1_up)
    So = oracle.schur_selfp(obs.k1_pp, obs.k1_pu, oracle.diag_lump(obs.k1_uu), obs.k1_up)
    assert same_pattern(Sx, So) and np.array_equal(Sx.data, So.data)
    # product's own blocks
    S = dpp.schur_selfp(bs.k1_pp, bs.k1_pu, dpp.diag_lump(bs.k1_uu), bs.k1_up)
    if form == "hdiv" and dim == 2:
        assert same_pattern(S, So) and np.array_equal(S.data, So.data)
    else:
        assert union_close(S, So, 1e-12)
    h, ho = dpp.amg_setup(S), oracle.amg_setup(So)
    assert h.level_count == ho.level_count
    for lv, lo in zip(h.levels, ho.levels):
        assert lv.A.shape == lo.A.shape
        if lo.P is not None:
            assert np.array_equal(lv.aggregates, lo.agg)  # aggregates identical level by level
            assert lv.P.shape == lo.P.shape
            assert np.max(np.abs((lv.P - lo.P).toarray())) < 1e-12
        assert np.max(np.abs((lv.A - lo.A).toarray())) < 1e-11 * max(1.0, abs(lo.A).max())
    r = rng.standard_normal(S.shape[0])
    assert rel_close(dpp.amg_vcycle(h, r), oracle.amg_vcycle(ho, r), 1e-10)


@pytest.mark.parametrize("form,dim,kind,n", [("hdiv", 2, "tri", 16), ("cgvms", 3, "tet", 6), ("dgvms", 2, "tri", 6)])
def test_amg_prolongator_bitwise(form, dim, kind, n):
    """P = P0 - (2 w / rho) Dinv (A P0) (linalg.py:369-371) with scipy's own rounding, rebuilt
    here from the device's operator, aggregates and rho: the device forms P without A @ P0
    (warp-per-row key extraction) and must agree bit for bit, pattern and order included."""
    bs, obs = systems(form, dim, kind, n)
    S = dpp.schur_selfp(obs.k1_pp, obs.k1_pu, oracle.diag_lump(obs.k1_uu), obs.k1_up)
    h = dpp.amg_setup(S)
    for lv in h.levels[:-1]:
        A = lv.A.tocsr()
        nr, nc = A.shape[0], lv.P.shape[1]
        P0 = sp.csr_matrix((np.ones(nr), (np.arange(nr), lv.aggregates)), shape=(nr, nc))
        Dinv = sp.diags(1.0 / A.diagonal(), format="csr")
        P = (P0 - (2.0 * (2.0 / 3.0) / lv.rho) * (Dinv @ (A @ P0))).tocsr()
        P.sort_indices()
        assert same_pattern(lv.P, P) and np.array_equal(lv.P.data, P.data)
    # Galerkin products A_c = R (A P), R = P^T (the device transpose is a stable sort of
    # column ids); coarse rows may be split-k summed, so entries agree to rounding
    for lv, nx in zip(h.levels[:-1], h.levels[1:]):
        A, P = lv.A.tocsr(), lv.P.tocsr()
        Ac = (P.T.tocsr() @ (A @ P)).tocsr()
        Ac.sort_indices()
        assert abs(nx.A - Ac).max() <= 1e-14 * abs(Ac).max()


def _agg_case(kind, n, rng):
    """Strength graphs the mesh operators do not produce: asymmetric patterns, rows with
    no off-diagonal entries, ties at the threshold, long chains, dense hubs."""
    if kind == "random_asym":
        A = sp.random(n, n, density=6.0 / n, random_state=int(rng.integers(1 << 30)), format="csr")
        A = A + sp.diags(np.full(n, 10.0))
    elif kind == "chain":   # a path in reverse order plus a few long-range ties
        i = np.arange(n - 1)
        A = sp.coo_matrix((-np.ones(n - 1), (i + 1, i)), shape=(n, n)) + sp.diags(np.full(n, 2.0))
        A = A + sp.coo_matrix((-np.ones(20), (rng.integers(0, n, 20), rng.integers(0, n, 20))), shape=(n, n))
    elif kind == "ties":    # integer magnitudes: many |a_ij| == theta * max exactly
        A = sp.random(n, n, density=8.0 / n, random_state=int(rng.integers(1 << 30)), format="csr")
        A.data = np.round(A.data * 4.0) + 1.0
        A = A + sp.diags(np.full(n, 50.0))
    elif kind == "hubs":    # a few rows / columns strongly tied to everything
        A = sp.random(n, n, density=3.0 / n, random_state=int(rng.integers(1 << 30)), format="lil")
        for h in rng.integers(0, n, 4):
            A[h, :] = 0.5
            A[:, h] = 0.5
        A = sp.csr_matrix(A) + sp.diags(np.full(n, 20.0))
    A = sp.csr_matrix(A)
    A.sum_duplicates()
    A.sort_indices()
    # isolated rows: diagonal only
    iso = rng.integers(0, n, max(1, n // 50))
    A = sp.lil_matrix(A)
    for r in iso:
        d = A[r, r]
        A[r, :] = 0.0
        A[r, r] = d
    A = sp.csr_matrix(A)
    A.eliminate_zeros()
    A.sort_indices()
    return A


@pytest.mark.parametrize("kind", ["random_asym", "chain", "ties", "hubs"])
@pytest.mark.parametrize("n", [300, 20000])
def test_device_aggregation_bitwise(kind, n, rng):
    """Device aggregation (three passes: seeds by owner waits, first-taken neighbour,
    singletons) == the reference's sequential greedy (linalg.py:279-324) via the oracle,
    on patterns chosen to stress its order dependence (device passes forced at every size)."""
    A = _agg_case(kind, n, rng)
    ref = oracle_solvers.aggregate(A, 0.5)
    for path in ("device", "host"):
        assert np.array_equal(dpp.strength_aggregates(A, 0.5, path=path), ref)


def test_amg_known_answers(rng):
    # reference tests/test_linalg.py:234-305
    A = poisson_1d(63)
    h = dpp.amg_setup(A)
    assert h.level_count == 1
    b = np.ones(63)
    assert np.linalg.norm(b - A @ dpp.amg_vcycle(h, b)) / np.linalg.norm(b) < 0.2
    A = poisson_1d(255)
    h = dpp.amg_setup(A)
    assert h.level_count >= 2
    b = rng.standard_normal(255)
    x = dpp.amg_vcycle(h, b)
    first = np.linalg.norm(b - A @ x) / np.linalg.norm(b)
    assert first < 0.5
    prev = first
    for _ in range(3):
        x = x + dpp.amg_vcycle(h, b - A @ x)
        cur = np.linalg.norm(b - A @ x) / np.linalg.norm(b)
        assert cur < 0.35 * prev
        prev = cur
    for lvl in range(h.level_count - 1):
        L = h.levels[lvl]
        assert np.max(np.abs(h.levels[lvl + 1].A.toarray() - (L.P.T @ L.A @ L.P).toarray())) < 1e-12
    hi = dpp.amg_setup(sp.identity(50, format="csr"))
    r = rng.standard_normal(50)
    assert np.allclose(dpp.amg_vcycle(hi, r), r, atol=1e-14)
    with pytest.raises(dpp.ZeroPivotError):
        dpp.amg_setup(sp.csr_matrix(np.array([[1.0, 1.0], [1.0, 0.0]])))
    A = poisson_1d(200)
    h = dpp.amg_setup(A)
    for _ in range(4):
        r1, r2 = rng.standard_normal(200), rng.standard_normal(200)
        z1, z2 = dpp.amg_vcycle(h, r1), dpp.amg_vcycle(h, r2)
        assert abs(z2 @ r1 - z1 @ r2) < 1e-8 * max(1.0, abs(z1 @ r2))


def test_poisson_amg_matches_golden(golden):
    A = poisson_1d(255)
    h = dpp.amg_setup(A)
    for li, lv in enumerate(h.levels):
        G = csr_from(golden, f"lin/poisson255/amg{li}.A")
        assert np.max(np.abs((lv.A - G).toarray())) < 1e-12
    z = dpp.amg_vcycle(h, golden["lin/poisson255/vc_r"])
    assert rel_close(z, golden["lin/poisson255/vc_z"], 1e-10)


# ----------------------------------------------------------------------------- GMRES

def test_gmres_reference_contract(rng):
    # reference tests/test_linalg.py:60-130
    b = rng.standard_normal(12)
    x, st = dpp.gmres(sp.identity(12, format="csr"), b, rtol=1e-12)
    assert st.converged and st.iterations == 1 and np.allclose(x, b, atol=1e-12)
    A = rng.standard_normal((10, 10)) + 10.0 * np.eye(10)
    b = rng.standard_normal(10)
    x, st = dpp.gmres(sp.csr_matrix(A), b, rtol=1e-10)
    assert st.converged and np.linalg.norm(x - np.linalg.solve(A, b)) / np.linalg.norm(x) < 1e-8
    R = sp.csr_matrix(np.array([[1.0, -1, 0, 0], [1, 1, -1, 0], [0, 1, 1, -1], [0, 0, 1, 1]]))
    bb = np.array([1.0, 0.0, 0.0, 0.5])
    xf, full = dpp.gmres(R, bb, rtol=1e-12, restart=30)
    x2, two = dpp.gmres(R, bb, rtol=1e-12, restart=2, max_iter=200)
    assert full.converged and two.converged and two.iterations > full.iterations
    assert np.allclose(xf, x2, atol=1e-9)
    x, st = dpp.gmres(sp.identity(4, format="csr"), np.zeros(4))
    assert st.converged and st.iterations == 0 and np.all(x == 0)
    _, st = dpp.gmres(sp.csr_matrix(np.diag([1.0, 1.0, 0.0])), np.array([0.0, 0.0, 1.0]),
                      rtol=1e-12, restart=3, max_iter=50)
    assert not st.converged and st.reason == "stagnation"
    A = sp.csr_matrix(rng.standard_normal((40, 40)) + 2 * np.eye(40))
    _, st = dpp.gmres(A, rng.standard_normal(40), rtol=1e-14, max_iter=3)
    assert not st.converged and st.reason in ("max_iter", "stagnation") and st.iterations <= 3


def test_gmres_matches_oracle_history(rng):
    A = sp.csr_matrix(rng.standard_normal((30, 30)) + 6 * np.eye(30))
    b = rng.standard_normal(30)
    x, st = dpp.gmres(A, b, rtol=1e-12, restart=10)
    xo, so = oracle.gmres(A, b, rtol=1e-12, restart=10)
    assert st.iterations == so.iterations
    assert rel_close(st.history, so.history, 1e-8)
    assert np.linalg.norm(x - xo) / np.linalg.norm(xo) < 1e-10


def test_gmres_with_host_callables(rng):
    A = sp.csr_matrix(rng.standard_normal((20, 20)) + 8 * np.eye(20))
    b = rng.standard_normal(20)
    D = A.diagonal()
    x, st = dpp.gmres(lambda v: A @ v, b, preconditioner=lambda r: r / D, rtol=1e-10)
    xo, so = oracle.gmres(lambda v: A @ v, b, preconditioner=lambda r: r / D, rtol=1e-10)
    assert st.converged and st.iterations == so.iterations
    assert np.linalg.norm(x - xo) / np.linalg.norm(xo) < 1e-9


# ----------------------------------------------------------------------------- preconditioner + solve

@pytest.mark.parametrize("form,dim,kind,n", [("hdiv", 2, "tri", 4), ("cgvms", 2, "tri", 4),
                                             ("dgvms", 2, "tri", 3), ("cgvms", 3, "tet", 2),
                                             ("hdiv", 3, "hex", 2)])
@pytest.mark.parametrize("meth", ["scale", "field"])
def test_pc_apply_matches_oracle(form, dim, kind, n, meth, rng):
    bs, obs = systems(form, dim, kind, n)
    pc = dpp.build_preconditioner(bs, dpp.method_config(meth))
    pco = oracle.build_preconditioner(obs, oracle.method_config(meth))
    assert pc.description == pco.description
    r = rng.standard_normal(bs.size)
    assert rel_close(pc(r), pco(r), 1e-10)


@pytest.mark.parametrize("form", ["hdiv", "cgvms", "dgvms"])
@pytest.mark.parametrize("dim,kind,n", MESHES)
@pytest.mark.parametrize("meth", ["scale", "field"])
def test_solve_matches_oracle(form, dim, kind, n, meth, golden):
    bs, obs = systems(form, dim, kind, n)
    rep = dpp.solve(bs, dpp.method_config(meth, rtol=1e-8))
    orep = oracle.solve(obs, oracle.method_config(meth, rtol=1e-8))
    x = rep.solution_vector()
    assert rep.converged
    assert abs(rep.stats.iterations - orep.stats.iterations) <= 2
    assert np.linalg.norm(x - orep.x) / np.linalg.norm(orep.x) < 1e-9
    p = f"solve/{form}/{kind}{n}/{meth}/"
    assert abs(rep.stats.iterations - int(golden[p + "its"])) <= 2
    assert np.linalg.norm(x - golden[p + "x"]) / np.linalg.norm(golden[p + "x"]) < 1e-9


def test_identity_like_system_and_user_blocks():
    # reference tests/test_blocksolve.py:43-51, :163-169
    n = 6
    eye, zero = sp.identity(n, format="csr"), sp.csr_matrix((n, n))
    bs = dpp.BlockSystem(formulation=dpp.Formulation.HDIV, mesh=None, params=None,
                         k1_uu=eye, k1_up=zero, k1_pu=zero, k1_pp=eye, k2_uu=eye, k2_up=zero,
                         k2_pu=zero, k2_pp=eye, k12_pp=zero, k21_pp=zero,
                         f1_u=np.ones(n), f1_p=np.ones(n), f2_u=np.ones(n), f2_p=np.ones(n))
    for cfg in (dpp.method_config("scale", rtol=1e-12), dpp.method_config("field", rtol=1e-12)):
        rep = dpp.solve(bs, cfg)
        assert rep.converged and rep.stats.iterations == 1


@pytest.mark.parametrize("form", ["hdiv", "cgvms", "dgvms"])
def test_patch_test_recovers_constants(form):
    # reference tests/test_blocksolve.py:206-230
    m = dpp.generate_unit_mesh(2, "tri", 2)
    bs = dpp.assemble(m, form, dpp.DppParameters(), dpp.boundary_data(dpp.constant_mms(2, 3.25), m))
    for meth in ("scale", "field"):
        rep = dpp.solve(bs, dpp.method_config(meth, rtol=1e-12))
        assert rep.converged
        assert np.max(np.abs(rep.fields["u1"])) < 1e-10 and np.max(np.abs(rep.fields["p1"] - 3.25)) < 1e-10


def test_solve_matches_dense_direct():
    for form, kind in (("hdiv", "tri"), ("cgvms", "quad")):
        p = dpp.DppParameters(gamma_b=(0.0, 0.0))
        m = dpp.generate_unit_mesh(2, kind, 4)
        bs = dpp.assemble(m, form, p, dpp.boundary_data(dpp.mms_2d(p), m))
        K, f = dpp.monolithic_view(bs)
        x_ref = np.linalg.solve(K.toarray(), f)
        rep = dpp.solve(bs, dpp.method_config("field", rtol=1e-10))
        assert rep.converged
        assert np.linalg.norm(rep.solution_vector() - x_ref) / np.linalg.norm(x_ref) < 1e-6


# ----------------------------------------------------------------------------- config sizes

CONFIGS = {
    "C0": ("cgvms", 2, "tri", 64, {}, "scale"),
    "C1": ("hdiv", 2, "tri", 256, {}, "field"),
    "C2": ("cgvms", 3, "tet", 40, {"k2": 0.01}, "scale"),
    "C2s": ("cgvms", 3, "tet", 16, {"k2": 0.01}, "field"),
    "C3s": ("cgvms", 3, "hex", 16, {"k2": 0.01}, "field"),
    "C4s": ("dgvms", 3, "tet", 6, {}, "scale"),
}


@pytest.mark.slow
@pytest.mark.parametrize("name", ["C0", "C1", "C2s", "C3s", "C4s", "C2"])
def test_config_parity(name):
    form, dim, kind, n, kw, meth = CONFIGS[name]
    bs, obs = systems(form, dim, kind, n, **kw)
    K, _ = dpp.monolithic_view(bs)
    Ko, _ = oracle.monolithic_view(obs)
    assert same_pattern(K, Ko)
    assert entry_close(K, Ko, 1e-12)
    rep = dpp.solve(bs, dpp.method_config(meth, rtol=1e-8))
    orep = oracle.solve(obs, oracle.method_config(meth, rtol=1e-8))
    x = rep.solution_vector()
    rel = np.linalg.norm(x - orep.x) / np.linalg.norm(orep.x)
    print(f"{name}: ksp {rep.stats.iterations} vs {orep.stats.iterations}, rel {rel:.2e}, "
          f"solve {rep.solve_s:.3f}s vs {orep.solve_s:.3f}s")
    assert rep.converged and abs(rep.stats.iterations - orep.stats.iterations) <= 2
    assert rel < 1e-9
