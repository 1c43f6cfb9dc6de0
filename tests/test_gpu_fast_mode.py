"""NON-PARITY fast mode: triangular solves as k Jacobi sweeps.

Not the reference's algorithm (its substitution is exact), so nothing here is a parity
claim.  Checked instead: the sweeps are exactly the stated iteration (numpy restatement
below), k >= the triangle's depth reproduces the exact solve (the strict part is
nilpotent), solves in this mode still reach rtol on the true residual, and the mode is
off unless asked for.
"""

import numpy as np
import pytest
import scipy.sparse as sp

import paper_1808_08328_b200 as dpp
from paper_1808_08328_b200 import _native as N

pytestmark = pytest.mark.gpu


def jacobi_ref(T, b, k, unit):
    """x0 = D^-1 b, x <- D^-1 (b - S x), k times (S = strict part of the triangle T)."""
    T = sp.csr_matrix(T)
    d = np.ones(T.shape[0]) if unit else T.diagonal()
    S = T - sp.diags(T.diagonal())
    x = b / d
    for _ in range(k):
        x = (b - S @ x) / d
    return x


def ilu_mats(n):
    m = dpp.generate_unit_mesh(3, "tet", n)
    p = dpp.DppParameters(k2=0.01, gamma_b=(0.0, 0.0, 0.0))
    bs = dpp.assemble(m, "cgvms", p, dpp.boundary_data(dpp.mms_3d(p), m))
    return bs


@pytest.mark.parametrize("k", [1, 2, 3])
def test_jacobi_sweeps_match_restatement(k, rng):
    bs = ilu_mats(4)
    A = bs.k1_uu.tocsr()
    exact = dpp.ilu0(A)             # exact mode first: the factors (bitwise the oracle's)
    L = sp.tril(exact.L, -1) + sp.identity(A.shape[0])
    U = sp.triu(exact.U)
    N.call("dpp_ctx_set_tri_jacobi", N.ctx(), k)
    try:
        f = dpp.ilu0(A)
    finally:
        N.call("dpp_ctx_set_tri_jacobi", N.ctx(), 0)
    r = rng.standard_normal(A.shape[0])
    y = jacobi_ref(L, r, k, unit=True)
    z = jacobi_ref(U, y, k, unit=False)
    got = dpp.apply_ilu0(f, r)
    assert np.max(np.abs(got - z)) <= 1e-12 * np.max(np.abs(z))


def test_deep_jacobi_equals_exact_solve(rng):
    bs = ilu_mats(3)
    A = bs.k1_uu.tocsr()
    exact = dpp.ilu0(A)
    N.call("dpp_ctx_set_tri_jacobi", N.ctx(), 64)   # >= the factors' dependency depth here
    try:
        f = dpp.ilu0(A)
    finally:
        N.call("dpp_ctx_set_tri_jacobi", N.ctx(), 0)
    r = rng.standard_normal(A.shape[0])
    a, b = dpp.apply_ilu0(f, r), dpp.apply_ilu0(exact, r)
    assert np.max(np.abs(a - b)) <= 1e-10 * np.max(np.abs(b))


@pytest.mark.parametrize("method", ["scale", "field"])
def test_fast_mode_solve_converges(method):
    bs = ilu_mats(12)
    cfg = dpp.method_config(method, rtol=1e-8, triangular="jacobi2")
    pc = dpp.build_preconditioner(bs, cfg)
    assert "NON-PARITY" in pc.description
    del pc
    rep = dpp.solve(bs, cfg)
    assert rep.stats.converged
    K, f = dpp.monolithic_view(bs)
    x = rep.solution_vector()
    assert np.linalg.norm(f - K @ x) <= 1.01e-8 * np.linalg.norm(f)
    # the default is the reference's exact substitution
    ex = dpp.solve(bs, dpp.method_config(method, rtol=1e-8))
    assert dpp.method_config(method).triangular == "exact"
    assert ex.stats.converged


def test_option_validation():
    for bad in ("jacobi", "jacobi0", "jacobi65", "gauss"):
        with pytest.raises(ValueError):
            dpp.method_config("scale", triangular=bad)
