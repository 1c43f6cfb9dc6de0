"""Diagnostics for the assembly-option parity tests (bitwise block / RHS / PC comparison)."""
import numpy as np, scipy.sparse as sp, sys, os
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
from tests.test_gpu_features import pair
import oracle, paper_1808_08328_b200 as dpp
bs, obs = pair("hdiv", 3, "tet", 3, vel_side=True)
for name in ("k1_uu", "k1_up", "k1_pu", "k1_pp", "k2_uu", "k12_pp"):
    A, B = sp.csr_matrix(getattr(bs, name)), sp.csr_matrix(getattr(obs, name))
    D = (A - B)
    print(name, A.nnz, B.nnz, "max|diff|", abs(D).max() if D.nnz else 0.0)
for name in ("f1_u", "f1_p", "f2_u", "f2_p"):
    a, b = np.asarray(getattr(bs, name)), np.asarray(getattr(obs, name))
    i = np.argmax(np.abs(a - b))
    print(name, "max|diff|", np.max(np.abs(a - b)), "at", i, a[i], b[i])
cfg = dpp.method_config("field", rtol=1e-8)
pc = dpp.build_preconditioner(bs, cfg)
opc = oracle.build_preconditioner(obs, oracle.method_config("field", rtol=1e-8))
r = np.random.default_rng(0).standard_normal(pc.size if hasattr(pc, "size") else len(np.concatenate([bs.f1_u, bs.f1_p, bs.f2_u, bs.f2_p])))
z, oz = pc(r), opc(r)
print("pc rel diff", np.linalg.norm(z - oz) / np.linalg.norm(oz))
