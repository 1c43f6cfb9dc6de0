"""Full-size runs of BASELINE configs on the device (no oracle): assemble + solve, twice.

  python tools/run_config.py C3 | C3h | C4 [n]
C3  = config 3 as BASELINE.json states it (HEX 64^3 CG-VMS, per-cell log-normal k1, k2 = 1e-2 k1,
      p = 1 / 0 on x = 0 / 1, no flow elsewhere; field split) -- the extension, parity unpinned;
C3h = its parity-pinned variant (homogeneous k1=1, k2=0.01, MMS BCs, field split);
C4  = DG-VMS TET 32^3, paper_3d_parameters, scale split, plus the 100x SpMV / PC-apply sweep.
"""
import ctypes as C
import os
import sys
import time
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import paper_1808_08328_b200 as dpp
from paper_1808_08328_b200 import _native as N

name = sys.argv[1]
ext = {}
if name in ("C3", "C3h"):
    form, dim, kind, n, meth = "cgvms", 3, "hex", 64, "field"
    p = dpp.DppParameters(k2=0.01, gamma_b=(0.0, 0.0, 0.0))
else:
    form, dim, kind, n, meth = "dgvms", 3, "tet", 32, "scale"
    p = dpp.paper_3d_parameters()
if len(sys.argv) > 2:
    n = int(sys.argv[2])
t0 = time.perf_counter()
m = dpp.generate_unit_mesh(dim, kind, n)
bcs = dpp.boundary_data(dpp.manufactured_solution(dim, p), m)
if name == "C3":
    p, bcs, ck = dpp.problem.heterogeneous_channel(m)
    ext = dict(cell_permeability=ck, velocity_dirichlet="strong")
print(f"{name} n={n}: mesh {time.perf_counter() - t0:.2f} s", flush=True)
for rep in range(int(os.environ.get("REPS", "2"))):
    t0 = time.perf_counter()
    bs = dpp.assemble(m, form, p, bcs, **ext)
    N.sync()
    t1 = time.perf_counter()
    r = dpp.solve(bs, dpp.method_config(meth, rtol=1e-8), want_solution=False)
    t2 = time.perf_counter()
    dof = int(sum(bs.device().sizes))
    print(f"  rep {rep}: assemble {1e3 * (t1 - t0):.1f} ms, solve {1e3 * (t2 - t1):.1f} ms "
          f"(pc setup {1e3 * r.pc_setup_s:.1f}), its {r.stats.iterations}, converged {r.stats.converged}, "
          f"relres {r.stats.relative_residual:.2e}, {dof} DoF -> {dof / (t2 - t0) / 1e6:.2f} M DoF/s", flush=True)
    if rep == 0 and name == "C4":
        pc = dpp.build_preconditioner(bs, dpp.method_config(meth, rtol=1e-8))
        prof = N.StepProfile()
        N.call("dpp_profile_step", N.ctx(), bs.device().h, pc.handle(), 100, 0, C.byref(prof))
        print(f"  100x sweep: spmv {prof.spmv_ms:.3f} ms ({prof.spmv_bytes / prof.spmv_ms / 1e6:.0f} GB/s), "
              f"pc {prof.pc_ms:.3f} ms ({prof.pc_bytes / prof.pc_ms / 1e6:.0f} GB/s), "
              f"{prof.pc_launches} kernels/apply", flush=True)
        del pc
    del bs, r
