"""Build a system + PC and run a few PC applies (profiling target).

PROF_CFG = C2 (default, CG-VMS TET 40 scale) | C3 (CG-VMS HEX 64 field) | C4 (DG-VMS TET 32 scale)."""
import ctypes as C
import os
import sys
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import numpy as np
import paper_1808_08328_b200 as dpp
from paper_1808_08328_b200 import _native as N

cfg = os.environ.get("PROF_CFG", "C2")
form, kind, n, meth, p = {
    "C2": ("cgvms", "tet", 40, "scale", dpp.DppParameters(k2=0.01, gamma_b=(0.0, 0.0, 0.0))),
    "C3": ("cgvms", "hex", 64, "field", dpp.DppParameters(k2=0.01, gamma_b=(0.0, 0.0, 0.0))),
    "C4": ("dgvms", "tet", 32, "scale", dpp.paper_3d_parameters()),
}[cfg]
n = int(os.environ.get("PROF_N", n))
meth = os.environ.get("PROF_METHOD", meth)
m = dpp.generate_unit_mesh(3, kind, n)
bs = dpp.assemble(m, form, p, dpp.boundary_data(dpp.mms_3d(p), m))
pc = dpp.build_preconditioner(bs, dpp.method_config(meth))
prof = N.StepProfile()
if os.environ.get("PROF_RANGE") == "1":   # ncu --profile-from-start off: only the profiled step
    C.CDLL("libcudart.so.12").cudaProfilerStart()
N.call("dpp_profile_step", N.ctx(), bs.device().h, pc.handle(), int(os.environ.get("PROF_REPS", "3")), int(os.environ.get("PROF_FLUSH", "0")), C.byref(prof))
print("spmv_ms", prof.spmv_ms, "pc_ms", prof.pc_ms, "kernels/apply", prof.pc_launches)
