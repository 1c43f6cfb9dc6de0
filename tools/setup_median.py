"""Median PC-setup and solve time over REPS steps of C2 (after one warm-up)."""
import os, sys, time
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import numpy as np
import paper_1808_08328_b200 as dpp
p = dpp.DppParameters(k2=0.01, gamma_b=(0.0, 0.0, 0.0))
m = dpp.generate_unit_mesh(3, "tet", 40)
bcs = dpp.boundary_data(dpp.mms_3d(p), m)
cfg = dpp.method_config("scale", rtol=1e-8)
su, so = [], []
for rep in range(int(os.environ.get("REPS", "9")) + 1):
    bs = dpp.assemble(m, "cgvms", p, bcs)
    t0 = time.perf_counter()
    r = dpp.solve(bs, cfg, want_solution=False)
    t1 = time.perf_counter()
    if rep:
        su.append(1e3 * r.pc_setup_s)
        so.append(1e3 * (t1 - t0))
    del bs, r
print(f"setup median {np.median(su):.1f} ms (min {min(su):.1f}, max {max(su):.1f}); solve median {np.median(so):.1f} ms")
