"""Config-size parity pinned to the UNMODIFIED reference (tests/golden/configs.json, written by
tests/golden/make_golden_configs.py in the build container): BASELINE configs 1 and 2 at full
size, and the survey's reduced parity sizes of configs 3 (HEX 32^3, homogeneous-k MMS variant,
field split) and 4 (DG-VMS TET 16^3, scale split).

CPU (oracle): C1 / C2 bit-for-bit -- K pattern, S_p pattern and values, aggregates of every AMG
level, iteration count and the solution sample.
GPU (device path): every case -- K pattern bit-exact, S_p pattern and values bitwise the
reference's for H(div) (C1: its AMG setup is ulp-sensitive) and bitwise scipy's selfp of the
device blocks otherwise (CG / DG entries agree to rounding only, so exact cancellations can
differ), AMG aggregates identical to the reference's on every level, iterations within +-2 and
the solution within 1e-9 relative (north_star bars) on the strided sample the reference stored.
"""

import hashlib
import json
import os

import numpy as np
import pytest

from tests.conftest import GOLDEN

with open(os.path.join(GOLDEN, "configs.json")) as _fh:
    CFG = json.load(_fh)


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def _sample_rel(x, g):
    s = np.asarray(g["x_sample"])
    xs = x[::g["x_sample_stride"]]
    return np.linalg.norm(xs - s) / np.linalg.norm(s)


@pytest.mark.parametrize("name", ["C1", "C2"])
def test_oracle_matches_reference_at_config_size(name):
    import oracle
    from oracle import solvers
    g = CFG[name]
    op = oracle.Params(k2=g["k2"], gamma_b=(0.0,) * g["dim"])
    m = oracle.generate_unit_mesh(g["dim"], g["kind"], g["n"])
    obs = oracle.assemble(m, g["form"], op, oracle.boundary_data(oracle.mms(g["dim"], op), m))
    K, _ = oracle.monolithic_view(obs)
    assert K.nnz == g["K_nnz"]
    assert sha(K.indptr.astype(np.int64)) == g["K_sha_indptr"] and sha(K.indices.astype(np.int64)) == g["K_sha_indices"]
    for net in (1, 2):
        blk = {b: getattr(obs, f"k{net}_{b}") for b in ("uu", "pp", "pu", "up")}
        S = solvers.schur_selfp(blk["pp"], blk["pu"], solvers.diag_lump(blk["uu"]), blk["up"])
        gs = g[f"S{net}"]
        assert sha(S.indptr.astype(np.int64)) == gs["sha_indptr"] and sha(S.indices.astype(np.int64)) == gs["sha_indices"]
        assert sha(S.data) == gs["sha_data"]
        h = solvers.amg_setup(S)
        assert [lv.A.shape[0] for lv in h.levels] == gs["amg_sizes"]
        assert [sha(lv.agg.astype(np.int64)) for lv in h.levels[:-1]] == gs["agg_sha"]
    rep = oracle.solve(obs, oracle.method_config(g["method"], rtol=1e-8))
    assert rep.stats.iterations == g["its"]
    assert _sample_rel(rep.x, g) == 0.0   # bitwise


@pytest.mark.gpu
@pytest.mark.slow
@pytest.mark.timeout(900)
@pytest.mark.parametrize("name", ["C1", "C2", "C3p", "C4pp"])
def test_device_matches_reference_at_config_size(name):
    import paper_1808_08328_b200 as dpp
    from paper_1808_08328_b200 import linalg
    g = CFG[name]
    p = dpp.DppParameters(k2=g["k2"], gamma_b=(0.0,) * g["dim"])
    m = dpp.generate_unit_mesh(g["dim"], g["kind"], g["n"])
    bs = dpp.assemble(m, g["form"], p, dpp.boundary_data(dpp.manufactured_solution(g["dim"], p), m))
    K, f = dpp.monolithic_view(bs)
    assert K.nnz == g["K_nnz"] and K.shape[0] == g["dof"]
    assert sha(K.indptr.astype(np.int64)) == g["K_sha_indptr"] and sha(K.indices.astype(np.int64)) == g["K_sha_indices"]
    assert abs(np.linalg.norm(f) - g["f_norm"]) <= 1e-12 * g["f_norm"]
    for net in (1, 2):
        blk = {b: getattr(bs, f"k{net}_{b}") for b in ("uu", "pp", "pu", "up")}
        S = linalg.schur_selfp(blk["pp"], blk["pu"], linalg.diag_lump(blk["uu"]), blk["up"])
        gs = g[f"S{net}"]
        if g["form"] == "hdiv":
            # H(div) blocks are bitwise the reference's, so S_p is too (pattern and values)
            assert sha(S.indptr.astype(np.int64)) == gs["sha_indptr"]
            assert sha(S.indices.astype(np.int64)) == gs["sha_indices"] and sha(S.data) == gs["sha_data"]
        else:
            # CG / DG blocks agree to rounding, so entries that cancel to exactly zero in one
            # S_p (and are dropped, as scipy drops them) may survive as ~1e-17 in the other:
            # the device S_p must equal scipy's selfp on the same blocks bit for bit
            from oracle import solvers
            So = solvers.schur_selfp(blk["pp"], blk["pu"], solvers.diag_lump(blk["uu"]), blk["up"])
            assert np.array_equal(S.indptr, So.indptr) and np.array_equal(S.indices, So.indices)
            assert np.array_equal(S.data, So.data)
            assert abs(S.nnz - gs["nnz"]) <= 1e-3 * gs["nnz"]
        h = linalg.amg_setup(S)
        assert [lv.A.shape[0] for lv in h.levels] == gs["amg_sizes"]
        assert [sha(lv.aggregates.astype(np.int64)) for lv in h.levels[:-1]] == gs["agg_sha"]
        del h
    rep = dpp.solve(bs, dpp.method_config(g["method"], rtol=1e-8))
    x = rep.solution_vector()
    rel = _sample_rel(x, g)
    print(f"{name}: ksp {rep.stats.iterations} (reference {g['its']}), sample rel {rel:.2e}, "
          f"x_norm rel {abs(np.linalg.norm(x) - g['x_norm']) / g['x_norm']:.2e}")
    assert rep.converged and abs(rep.stats.iterations - g["its"]) <= 2
    assert rel < 1e-9
    assert abs(np.linalg.norm(x) - g["x_norm"]) <= 1e-9 * g["x_norm"]
