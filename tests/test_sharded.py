"""Row-sharded SpMV (paper_1808_08328_b200/sharded.py, csrc/shard.cu).

CPU part: the host logic -- entry-balanced row partition, owner-coded columns, per-rank plans --
alone and under a world_size-2 gloo group (x slices exchanged with all_gather_object, the plan
evaluated by a numpy decode in this file: the package itself has no CPU SpMV).
GPU part: the device kernel against scipy's csr_matvec (the reference's SpMV, linalg.py:27-32;
tolerance 1e-13 relative to |K||x| -- lane-parallel row sums, a non-parity extension): all shards
of one operator in one process, and two processes on the one GPU that map each other's x slice
over CUDA IPC (the kernels only read the mapped slices; no launch waits on another).
"""

import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest
import scipy.sparse as sp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

from paper_1808_08328_b200 import sharded as S  # noqa: E402


def operator(n=300, seed=3, density=0.02):
    rng = np.random.default_rng(seed)
    A = sp.random(n, n, density=density, random_state=rng, format="csr") + sp.eye(n, format="csr")
    A = sp.csr_matrix(A)
    A.sort_indices()
    return A


def decode_apply(plan, xsegs):
    """numpy evaluation of a plan: y[r] = sum_j values[j] * xsegs[owner(j)][offset(j)]."""
    owner = plan.codes >> S.OFF_BITS
    off = plan.codes & ((1 << S.OFF_BITS) - 1)
    xv = np.empty(len(plan.codes))
    for p in range(plan.world):
        m = owner == p
        xv[m] = xsegs[p][off[m]]
    y = np.zeros(plan.rows)
    rows = np.repeat(np.arange(plan.rows), np.diff(plan.indptr))
    np.add.at(y, rows, plan.values * xv)
    return y


@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_partition_is_balanced_and_covers_rows(world):
    A = operator()
    st = S.partition_rows(A.indptr, world)
    assert st[0] == 0 and st[-1] == A.shape[0] and np.all(np.diff(st) > 0)
    per = np.diff(A.indptr[st])
    assert per.sum() == A.nnz
    assert per.max() - per.min() <= 2 * np.diff(A.indptr).max()   # within one (long) row of the mean


def test_partition_keeps_blocks_nonempty_for_skewed_rows():
    A = sp.lil_matrix((6, 6))
    A[0, :] = 1.0                      # all entries in the first row
    A.setdiag(1.0)
    st = S.partition_rows(sp.csr_matrix(A).indptr, 4)
    assert np.all(np.diff(st) > 0) and st[-1] == 6
    with pytest.raises(ValueError):
        S.partition_rows(sp.csr_matrix(A).indptr, 7)
    with pytest.raises(ValueError):
        S.partition_rows(sp.csr_matrix(A).indptr, 9)


def test_codes_round_trip_and_reject_bad_columns():
    st = np.array([0, 5, 5, 12])      # an empty middle slice is legal for the coding
    idx = np.array([0, 4, 5, 11, 7])
    c = S.encode_columns(idx, st)
    owner, off = c >> S.OFF_BITS, c & ((1 << S.OFF_BITS) - 1)
    assert owner.tolist() == [0, 0, 2, 2, 2] and off.tolist() == [0, 4, 0, 6, 2]
    assert np.array_equal(st[owner] + off, idx)
    with pytest.raises(ValueError):
        S.encode_columns([12], st)
    with pytest.raises(ValueError):
        S.encode_columns([-1], st)


@pytest.mark.parametrize("world", [1, 2, 5])
def test_plans_reassemble_the_product(world):
    A = operator(seed=world)
    x = np.random.default_rng(0).standard_normal(A.shape[0])
    plans = [S.ShardPlan.from_global(A, p, world) for p in range(world)]
    st = plans[0].starts
    xsegs = [x[st[p]:st[p + 1]] for p in range(world)]
    y = np.concatenate([decode_apply(pl, xsegs) for pl in plans])
    assert np.allclose(y, A @ x, rtol=0, atol=1e-13 * np.abs(A).dot(np.abs(x)).max())
    assert (sum(pl.halo_entries for pl in plans) == 0) == (world == 1)
    with pytest.raises(ValueError):
        S.ShardPlan.from_global(A[:, :10], 0, 1)
    with pytest.raises(ValueError):
        S.ShardPlan.from_global(A, 2, 2)


def test_node_interleaved_order_groups_a_nodes_dofs():
    perm = S.node_interleaved_order([6, 3, 6, 3], (2, 1, 2, 1))     # 3 nodes, dim 2
    assert sorted(perm.tolist()) == list(range(18))
    assert perm[:6].tolist() == [0, 1, 6, 9, 10, 15]                # node 0: u1x u1y p1 u2x u2y p2
    assert perm[6:12].tolist() == [2, 3, 7, 11, 12, 16]
    with pytest.raises(ValueError):
        S.node_interleaved_order([6, 4, 6, 3], (2, 1, 2, 1))
    with pytest.raises(ValueError):
        S.node_interleaved_order([6, 3], (2, 1, 2))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _run_world2(script, tmp_path, timeout=240):
    path = tmp_path / "w.py"
    path.write_text(script)
    port = _free_port()
    procs = []
    for r in range(2):
        env = dict(os.environ, RANK=str(r), LOCAL_RANK="0", WORLD_SIZE="2", DPP_DEVICE="0",
                   MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        procs.append(subprocess.Popen([sys.executable, str(path)], env=env, stdout=subprocess.PIPE,
                                      stderr=subprocess.PIPE, text=True))
    outs = [p.communicate(timeout=timeout) for p in procs]
    for p, (o, e) in zip(procs, outs):
        if p.returncode != 0 and "cudaIpc" in e:
            # legacy CUDA IPC can be closed to a container (no shared IPC namespace); the kernel
            # and the plans are covered by the single-process tests either way
            pytest.skip("CUDA IPC is not available between processes here: " + e.strip().splitlines()[-1][:200])
        assert p.returncode == 0, e[-3000:]
    return [json.loads(o.strip().splitlines()[-1]) for o, _ in outs]


GLOO_WORKER = r"""
import json, os, sys
sys.path.insert(0, {root!r})
import numpy as np
import torch.distributed as dist
from paper_1808_08328_b200 import sharded as S
from tests.test_sharded import operator, decode_apply
dist.init_process_group("gloo", rank=int(os.environ["RANK"]), world_size=int(os.environ["WORLD_SIZE"]))
rank, world = S._rank_world(None)
A = operator(seed=11)
x = np.random.default_rng(5).standard_normal(A.shape[0])
plan = S.ShardPlan.from_global(A, rank, world)
r0, r1 = int(plan.starts[rank]), int(plan.starts[rank + 1])
slices = [None] * world
dist.all_gather_object(slices, x[r0:r1])          # what the IPC mappings give the kernel
y = decode_apply(plan, slices)
ref = (A @ x)[r0:r1]
parts = [None] * world
dist.all_gather_object(parts, y)
full = np.concatenate(parts)
print(json.dumps({{"rank": rank, "rows": [r0, r1], "err": float(np.abs(y - ref).max()),
                  "full_err": float(np.abs(full - A @ x).max()), "halo": plan.halo_entries}}))
dist.destroy_process_group()
"""


@pytest.mark.timeout(300)
def test_plans_under_gloo_world2(tmp_path):
    res = _run_world2(GLOO_WORKER.format(root=ROOT), tmp_path)
    res.sort(key=lambda r: r["rank"])
    assert res[0]["rows"][0] == 0 and res[0]["rows"][1] == res[1]["rows"][0] and res[1]["rows"][1] == 300
    assert all(r["err"] < 1e-13 and r["full_err"] < 1e-13 for r in res)
    assert all(r["halo"] > 0 for r in res)


def test_device_objects_fail_loudly_without_a_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(Exception) as ei:
        S.LocalShards(operator(), 2)
    assert "DeviceUnavailable" in type(ei.value).__name__ or "CUDA" in str(ei.value) or "device" in str(ei.value).lower()


# ------------------------------------------------------------------------------- GPU

def _bound(A, x):
    return 1e-13 * max(np.abs(A).dot(np.abs(x)).max(), 1e-300)


@pytest.mark.gpu
@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_local_shards_match_csr_matvec(world):
    A = operator(n=2000, seed=world, density=0.01)
    x = np.random.default_rng(1).standard_normal(A.shape[0])
    op = S.LocalShards(A, world)
    y = op.matvec(x)
    assert np.abs(y - A @ x).max() <= _bound(A, x)
    # ragged rows: empty rows, one dense row, a 1-row shard
    B = sp.lil_matrix((64, 64))
    B[3, :] = np.arange(1, 65)
    B[10, 5] = 2.0
    B[63, 0] = -1.0
    B = sp.csr_matrix(B)
    xb = np.random.default_rng(2).standard_normal(64)
    st = np.array([0, 3, 4, 64]) if world == 3 else None
    if world in (1, 3):
        assert np.abs(S.LocalShards(B, world, st).matvec(xb) - B @ xb).max() <= _bound(B, xb)


@pytest.mark.gpu
def test_sharded_k_of_an_assembled_system():
    """The four-field K of a CG-VMS system (the operator GMRES multiplies by) in 4 shards."""
    import paper_1808_08328_b200 as dpp
    p = dpp.DppParameters(k2=0.01, gamma_b=(0.0, 0.0, 0.0))
    m = dpp.generate_unit_mesh(3, "tet", 10)
    bs = dpp.assemble(m, "cgvms", p, dpp.boundary_data(dpp.manufactured_solution(3, p), m))
    K = sp.csr_matrix(dpp.monolithic_view(bs)[0])
    x = np.random.default_rng(4).standard_normal(K.shape[0])
    op = S.LocalShards(K, 4)
    assert np.abs(op.matvec(x) - K @ x).max() <= _bound(K, x)
    for ms, by in op.profile(reps=5):
        assert ms > 0 and by > 0
    # node-interleaved ordering: row blocks become slabs of the mesh, far fewer off-rank entries
    sizes = bs.device().sizes
    opi = S.LocalShards(K, 4, perm=S.node_interleaved_order(sizes, (3, 1, 3, 1)))
    assert np.abs(opi.matvec(x) - K @ x).max() <= _bound(K, x)
    off = sum(pl.halo_entries for pl in op.plans) / K.nnz
    offi = sum(pl.halo_entries for pl in opi.plans) / K.nnz
    assert offi < 0.6 * off, (off, offi)      # 11 node planes over 4 ranks: 34 % -> 17 % (C2: 57 % -> 4 %)


@pytest.mark.gpu
def test_shard_abi_rejects_bad_plans():
    A = operator(n=100)
    pl = S.ShardPlan.from_global(A, 0, 2)
    bad = S.ShardPlan(pl.rank, pl.world, pl.starts, pl.indptr, pl.codes.copy(), pl.values, pl.halo_entries)
    bad.codes[0] = (1 << S.OFF_BITS) | (1 << 20)       # offset beyond the owner's slice
    with pytest.raises(ValueError):
        S._DeviceShard(bad)
    sh = S._DeviceShard(pl)
    short = [S.PeerBuffer(3), S.PeerBuffer(3)]
    with pytest.raises(ValueError):
        sh.spmv(short)


IPC_WORKER = r"""
import json, os, sys
sys.path.insert(0, {root!r})
import numpy as np
import torch.distributed as dist
from paper_1808_08328_b200 import sharded as S
from tests.test_sharded import operator
dist.init_process_group("gloo", rank=int(os.environ["RANK"]), world_size=int(os.environ["WORLD_SIZE"]))
A = operator(n=5000, seed=21, density=0.004)
op = S.ShardedOperator(A)
r0, r1 = op.local_rows
errs = []
for k in range(3):                                   # repeated products: slices are rewritten
    x = np.random.default_rng(100 + k).standard_normal(A.shape[0])
    y = op.matvec(x[r0:r1])
    errs.append(float(np.abs(y - (A @ x)[r0:r1]).max() / np.abs(A).dot(np.abs(x)).max()))
ms, by = op.profile(reps=5)
print(json.dumps({{"rank": op.rank, "rows": [r0, r1], "err": max(errs), "halo": op.plan.halo_entries, "ms": ms}}))
dist.destroy_process_group()
"""


@pytest.mark.gpu
@pytest.mark.timeout(600)
def test_two_processes_read_each_others_slice_over_ipc(tmp_path):
    res = _run_world2(IPC_WORKER.format(root=ROOT), tmp_path, timeout=500)
    res.sort(key=lambda r: r["rank"])
    assert res[0]["rows"][1] == res[1]["rows"][0] and res[1]["rows"][1] == 5000
    assert all(r["err"] <= 1e-13 for r in res), res
    assert all(r["halo"] > 0 for r in res)
