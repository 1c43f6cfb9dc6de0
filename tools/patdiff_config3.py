import sys, numpy as np
sys.path.insert(0, '/root/repo')
import paper_1808_08328_b200 as dpp, oracle
from tests.test_config3 import _oracle_channel
for vd in ("natural", "strong"):
    m = dpp.generate_unit_mesh(3, "hex", 8)
    params, bcs, ck = dpp.problem.heterogeneous_channel(m)
    bs = dpp.assemble(m, "cgvms", params, bcs, cell_permeability=ck, velocity_dirichlet=vd)
    om, op, obcs, ock = _oracle_channel(3, "hex", 8)
    obs = oracle.assemble(om, "cgvms", op, obcs, cell_k=ock, velocity_dirichlet=vd)
    for name in ("k1_uu", "k1_up", "k1_pu", "k1_pp"):
        A = getattr(bs, name).tocsr(); B = obs.blocks[name].tocsr()
        A.sort_indices(); B.sort_indices()
        a = set(zip(*A.nonzero())) if False else None
        Ac = A.tocoo(); Bc = B.tocoo()
        sa = set(zip(Ac.row.tolist(), Ac.col.tolist())); sb = set(zip(Bc.row.tolist(), Bc.col.tolist()))
        only_a, only_b = sa - sb, sb - sa
        da = {(r, c): v for r, c, v in zip(Ac.row, Ac.col, Ac.data)}
        db = {(r, c): v for r, c, v in zip(Bc.row, Bc.col, Bc.data)}
        print(vd, name, A.nnz, B.nnz, "only device", len(only_a), "only oracle", len(only_b),
              "max |dev val| on only-device", max([abs(da[k]) for k in only_a], default=0),
              "max |oracle val| on only-oracle", max([abs(db[k]) for k in only_b], default=0),
              "explicit zeros dev/oracle", int((A.data == 0).sum()), int((B.data == 0).sum()))
