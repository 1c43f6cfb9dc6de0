import sys, os
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import numpy as np, scipy.sparse as sp
import oracle, paper_1808_08328_b200 as dpp
np.set_printoptions(linewidth=200, precision=6, suppress=True)
n = 12
A = sp.diags([-np.ones(n-1), 2.0*np.ones(n), -np.ones(n-1)], [-1,0,1], format="csr")
h = dpp.amg_setup(A, max_coarse=2); ho = oracle.amg_setup(A, max_coarse=2)
lv, lo = h.levels[0], ho.levels[0]
print("agg", lv.aggregates, lo.agg, "rho", lv.rho, lo.rho)
print("P dev\n", lv.P.toarray()); print("P ora\n", lo.P.toarray())
print("P dev csr", lv.P.indptr, lv.P.indices, lv.P.data)
print("Ac dev\n", h.levels[1].A.toarray()); print("Ac ora\n", ho.levels[1].A.toarray())
