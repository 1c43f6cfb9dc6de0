"""Every triangular-sweep strategy stays correct (the default path picks one per
triangle; these force the others).  Each variant runs in a fresh process (the
switches are read once per process) and must match the CPU oracle to the usual
bars: solution within 1e-9 relative, iterations within +-2.

  default                     global-stream dataflow sweeps for thin rows (k_trsv_gs, lane per row, entries
                              streamed from global memory), lane-group dataflow sweeps otherwise
                              (k_trsv_flow) + block-dense / dense smoothers + collapsed AMG tail
  DPP_PU_MODE=flow            lane-group dataflow sweeps everywhere (k_trsv_flow, polled x slots)
  DPP_PU_MODE=gs              global-stream sweeps everywhere
  DPP_GS_MIN_CLUSTERS=2       global-stream sweeps spread over two clusters of 16 CTAs (the form triangles too
                              large for one cluster's shared memory take): cross-cluster sources imported from
                              global memory by an extra warp
  DPP_PU_MODE=ws              warp-stream sweeps (lane per row, per-warp TMA rings) everywhere
  DPP_AMG_TAIL=0              launch-by-launch V-cycle on the small tail levels (no dense collapse)
  DPP_SGS_PLAIN=1             Gauss-Seidel half-sweeps with the literal residual b - A x (four SpMVs per level)
  DPP_BD_MAX=0 DPP_GBD_ROW=1  global block-dense sweeps (two launches per 512-row block) on the first AMG level
  DPP_BD_INV=sparse           diagonal-block / dense-level inverses by sparse substitution (not the blocked GEMMs)
  DPP_PU_MODE=lvl             level-mbarrier cluster sweeps (k_trsv_lvl: level teams, SELL chunks)
  DPP_PU_FLOW=0               level-synchronous push-exchange cluster sweeps (k_trsv_push)
  DPP_NO_PUSH=1               barrier-per-level cluster sweeps (tricluster.cu)
  DPP_BD_MAX=0                no block-dense smoothers (level sweeps on every AMG level)
  DPP_BD_MAX=0 DPP_NO_PUSH=1 DPP_NO_CLUSTER=1
                              block-sequential (triblock.cu) / sync-free warp-per-row sweeps
"""

import json
import os
import subprocess
import sys

import numpy as np
import pytest

from tests.conftest import ROOT

pytestmark = pytest.mark.gpu

SCRIPT = r"""
import json, sys
import numpy as np
sys.path.insert(0, {root!r})
import paper_1808_08328_b200 as dpp
p = dpp.DppParameters(k2=0.01, gamma_b=(0.0, 0.0, 0.0))
m = dpp.generate_unit_mesh(3, "tet", 16)
bs = dpp.assemble(m, "cgvms", p, dpp.boundary_data(dpp.mms_3d(p), m))
r = dpp.solve(bs, dpp.method_config("scale", rtol=1e-8))
np.save({out!r}, r.solution_vector())
print(json.dumps({{"its": r.stats.iterations, "converged": bool(r.stats.converged)}}))
"""

VARIANTS = {
    "default": {},
    "lane_group_flow": {"DPP_PU_MODE": "flow"},
    "global_stream": {"DPP_PU_MODE": "gs"},
    "multi_cluster_stream": {"DPP_GS_MIN_CLUSTERS": "2"},
    "warp_stream": {"DPP_PU_MODE": "ws"},
    "no_tail_collapse": {"DPP_AMG_TAIL": "0"},
    "plain_sgs_residuals": {"DPP_SGS_PLAIN": "1"},
    "global_block_dense": {"DPP_BD_MAX": "0", "DPP_GBD_ROW": "1"},
    "sparse_block_inverses": {"DPP_BD_INV": "sparse"},
    "level_mbarrier": {"DPP_PU_MODE": "lvl"},
    "level_sync_push": {"DPP_PU_FLOW": "0"},
    "pull_cluster": {"DPP_NO_PUSH": "1"},
    "no_block_dense": {"DPP_BD_MAX": "0"},
    "sync_free_and_block": {"DPP_BD_MAX": "0", "DPP_NO_PUSH": "1", "DPP_NO_CLUSTER": "1"},
}


@pytest.fixture(scope="module")
def oracle_ref():
    import oracle
    op = oracle.Params(k2=0.01, gamma_b=(0.0, 0.0, 0.0))
    om = oracle.generate_unit_mesh(3, "tet", 16)
    obs = oracle.assemble(om, "cgvms", op, oracle.boundary_data(oracle.mms(3, op), om))
    rep = oracle.solve(obs, oracle.method_config("scale", rtol=1e-8))
    return rep.x, rep.stats.iterations


@pytest.mark.timeout(600)
@pytest.mark.parametrize("name", list(VARIANTS))
def test_sweep_strategy(name, oracle_ref, tmp_path):
    out = str(tmp_path / "x.npy")
    env = dict(os.environ, **VARIANTS[name])
    res = subprocess.run([sys.executable, "-c", SCRIPT.format(root=ROOT, out=out)], env=env,
                         capture_output=True, text=True, timeout=500)
    assert res.returncode == 0, res.stderr[-2000:]
    info = json.loads(res.stdout.strip().splitlines()[-1])
    x_ref, its_ref = oracle_ref
    x = np.load(out)
    rel = np.linalg.norm(x - x_ref) / np.linalg.norm(x_ref)
    assert info["converged"] and abs(info["its"] - its_ref) <= 2, (info, its_ref)
    assert rel < 1e-9, rel


@pytest.mark.timeout(600)
def test_cluster_sweeps_bitwise(tmp_path):
    """The lane-group dataflow and level-synchronous push sweeps only change when a row is
    computed, not how: per-lane products in entry order, the same xor-shuffle reduction,
    (b - sum) * (1/t_ii) -- so the whole solve is bit-for-bit the same.  (The warp-stream and
    level-mbarrier sweeps regroup the row sums into partial sums: tolerance-checked in
    test_sweep_strategy.)"""
    xs = []
    for k, extra in enumerate(({"DPP_PU_MODE": "flow"}, {"DPP_PU_MODE": "push"})):
        out = str(tmp_path / f"x{k}.npy")
        res = subprocess.run([sys.executable, "-c", SCRIPT.format(root=ROOT, out=out)],
                             env=dict(os.environ, **extra), capture_output=True, text=True, timeout=500)
        assert res.returncode == 0, res.stderr[-2000:]
        xs.append(np.load(out))
    assert np.array_equal(xs[0], xs[1])


@pytest.mark.timeout(600)
def test_gmres_lookahead_bitwise(tmp_path):
    """Enqueueing the next Arnoldi column's SpMV + PC apply while the host reads H[:, j]
    (DPP_GMRES_AHEAD, default on) changes only when work is issued: same iterates bit for bit."""
    xs = []
    for k, extra in enumerate(({}, {"DPP_GMRES_AHEAD": "0"})):
        out = str(tmp_path / f"x{k}.npy")
        res = subprocess.run([sys.executable, "-c", SCRIPT.format(root=ROOT, out=out)],
                             env=dict(os.environ, **extra), capture_output=True, text=True, timeout=500)
        assert res.returncode == 0, res.stderr[-2000:]
        xs.append(np.load(out))
    assert np.array_equal(xs[0], xs[1])
