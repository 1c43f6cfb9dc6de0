"""Where the end-to-end C2 step spends its time (public API, mesh re-uploaded each step)."""
import os, sys, time
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import numpy as np
import paper_1808_08328_b200 as dpp
from paper_1808_08328_b200 import _native as N
from paper_1808_08328_b200.assembly import _pressure_data
p = dpp.DppParameters(k2=0.01, gamma_b=(0.0, 0.0, 0.0))
m = dpp.generate_unit_mesh(3, "tet", 40)
bcs = dpp.boundary_data(dpp.mms_3d(p), m)
cfg = dpp.method_config("scale", rtol=1e-8)
for rep in range(4):
    N.call("dpp_mesh_release_device", m._h)
    t0 = time.perf_counter()
    pd = [_pressure_data(m, bcs, net) for net in (1, 2)]
    t1 = time.perf_counter()
    N.call("dpp_mesh_release_device", m._h)
    t2 = time.perf_counter()
    bs = dpp.assemble(m, "cgvms", p, bcs)
    N.sync()
    t3 = time.perf_counter()
    r = dpp.solve(bs, cfg)
    t4 = time.perf_counter()
    x = r.solution_vector()
    t5 = time.perf_counter()
    print(f"rep {rep}: pressure traces {1e3*(t1-t0):.1f} ms (incl. mesh upload), assemble() {1e3*(t3-t2):.1f} ms, "
          f"solve {1e3*(t4-t3):.1f} ms (setup {1e3*r.pc_setup_s:.1f}), x download {1e3*(t5-t4):.1f} ms", flush=True)
    del bs, r
