"""Sharded SpMV kernel (csrc/shard.cu) on the C2 operator, all shards on one GPU (LocalShards):
ms per launch and algorithmic GB/s per shard for world = 1, 2, 4, 8, next to the SELL SpMV of
the unsharded K.  Peer loads are local here (one GPU); across GPUs the off-rank share of the
entries (printed) travels over NVLink instead.  usage: python tools/shard_timing.py [n]"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, scipy.sparse as sp
import paper_1808_08328_b200 as dpp
from paper_1808_08328_b200 import sharded as S

n = int(sys.argv[1]) if len(sys.argv) > 1 else 40
p = dpp.DppParameters(k2=0.01, gamma_b=(0.0, 0.0, 0.0))
m = dpp.generate_unit_mesh(3, "tet", n)
bs = dpp.assemble(m, "cgvms", p, dpp.boundary_data(dpp.manufactured_solution(3, p), m))
K = sp.csr_matrix(dpp.monolithic_view(bs)[0])
K.eliminate_zeros()            # the zero-free K the SELL plan stores too
x = np.random.default_rng(0).standard_normal(K.shape[0])
ref = K @ x
print(f"K: {K.shape[0]} rows, {K.nnz} entries")
perm = S.node_interleaved_order(bs.device().sizes, (3, 1, 3, 1))
for world, pm in [(w, q) for q in (None, perm) for w in (1, 2, 4, 8)]:
    op = S.LocalShards(K, world, perm=pm)
    err = np.abs(op.matvec(x) - ref).max() / np.abs(K).dot(np.abs(x)).max()
    prof = op.profile(reps=50)
    halo = [pl.halo_entries / max(len(pl.values), 1) for pl in op.plans]
    ms = [a for a, _ in prof]
    gbs = [b / a / 1e6 for a, b in prof]
    print(f"{'field-major' if pm is None else 'node-interleaved'} world {world}: err {err:.1e}  ms/launch max {max(ms):.4f}  GB/s per shard {min(gbs):.0f}-{max(gbs):.0f}"
          f"  off-rank entries {100 * min(halo):.1f}-{100 * max(halo):.1f} %  rows {np.diff(op.starts).tolist()}")
