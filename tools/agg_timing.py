"""Aggregation alone on C2's S_p (network 1): device passes vs host greedy, medians."""
import os, sys, time
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import numpy as np
import paper_1808_08328_b200 as dpp
n = int(os.environ.get("AB_N", "40"))
p = dpp.DppParameters(k2=0.01, gamma_b=(0.0, 0.0, 0.0))
m = dpp.generate_unit_mesh(3, "tet", n)
bs = dpp.assemble(m, "cgvms", p, dpp.boundary_data(dpp.mms_3d(p), m))
S = dpp.schur_selfp(bs.k1_pp, bs.k1_pu, dpp.diag_lump(bs.k1_uu), bs.k1_up)
from paper_1808_08328_b200.device import as_device
dS = as_device(S)
for path in ("device", "host", "device", "host"):
    ts = []
    for _ in range(10):
        t0 = time.perf_counter()
        a = dpp.strength_aggregates(dS, 0.5, path=path)
        ts.append(1e3 * (time.perf_counter() - t0))
    print(f"{path:7s} median {np.median(ts):.3f} ms min {min(ts):.3f} (n={S.shape[0]}, naggs={a.max() + 1})")
