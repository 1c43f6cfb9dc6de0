"""C2 in the NON-PARITY fast mode: iterations, setup and solve time per Jacobi sweep count."""
import os, sys, time
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import numpy as np
import paper_1808_08328_b200 as dpp
n = int(os.environ.get("FM_N", "40"))
p = dpp.DppParameters(k2=0.01, gamma_b=(0.0, 0.0, 0.0))
m = dpp.generate_unit_mesh(3, "tet", n)
bcs = dpp.boundary_data(dpp.mms_3d(p), m)
bs = dpp.assemble(m, "cgvms", p, bcs)
K, f = dpp.monolithic_view(bs)
for tri in ["exact"] + [f"jacobi{k}" for k in (1, 2, 3, 4, 6)]:
    for method in os.environ.get("FM_METHODS", "scale").split(","):
        cfg = dpp.method_config(method, rtol=1e-8, triangular=tri)
        ts, su = [], []
        for rep in range(4):
            t0 = time.perf_counter()
            r = dpp.solve(bs, cfg)
            ts.append(1e3 * (time.perf_counter() - t0))
            su.append(1e3 * r.pc_setup_s)
        x = r.solution_vector()
        res = np.linalg.norm(f - K @ x) / np.linalg.norm(f)
        print(f"{method:5s} {tri:8s} its {r.stats.iterations:4d} conv {r.stats.converged} true relres {res:.2e} "
              f"solve {np.median(ts[1:]):8.2f} ms (setup {np.median(su[1:]):6.2f})", flush=True)
