"""Build the C2 system + scale-split PC and run a few PC applies (profiling target)."""
import ctypes as C
import os
import sys
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import numpy as np
import paper_1808_08328_b200 as dpp
from paper_1808_08328_b200 import _native as N

n = int(os.environ.get("PROF_N", "40"))
meth = os.environ.get("PROF_METHOD", "scale")
p = dpp.DppParameters(k2=0.01, gamma_b=(0.0, 0.0, 0.0))
m = dpp.generate_unit_mesh(3, "tet", n)
bs = dpp.assemble(m, "cgvms", p, dpp.boundary_data(dpp.mms_3d(p), m))
pc = dpp.build_preconditioner(bs, dpp.method_config(meth))
prof = N.StepProfile()
N.call("dpp_profile_step", N.ctx(), bs.device().h, pc.handle(), int(os.environ.get("PROF_REPS", "3")), 0, C.byref(prof))
print("spmv_ms", prof.spmv_ms, "pc_ms", prof.pc_ms, "kernels/apply", prof.pc_launches)
