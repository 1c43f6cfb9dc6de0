"""PC apply of C2 per triangular mode (exact / jacobi<k>): dpp_profile_step device times,
algorithmic bytes and launches (L2 flushed between applies)."""
import ctypes as C, os, sys
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import paper_1808_08328_b200 as dpp
from paper_1808_08328_b200 import _native as N
p = dpp.DppParameters(k2=0.01, gamma_b=(0.0, 0.0, 0.0))
m = dpp.generate_unit_mesh(3, "tet", int(os.environ.get("FM_N", "40")))
bs = dpp.assemble(m, "cgvms", p, dpp.boundary_data(dpp.mms_3d(p), m))
dev = bs.device()
for tri in os.environ.get("FM_TRI", "exact,jacobi2,jacobi3").split(","):
    pc = dpp.build_preconditioner(bs, dpp.method_config("scale", rtol=1e-8, triangular=tri))
    prof = N.StepProfile()
    N.call("dpp_profile_step", N.ctx(), dev.h, pc.handle(), 10, 1, C.byref(prof))
    print(f"{tri:8s} pc {prof.pc_ms:.4f} ms  {prof.pc_bytes / 1e6:8.1f} MB  {prof.pc_bytes / prof.pc_ms / 1e6:7.1f} GB/s  "
          f"spmv {prof.spmv_ms:.4f} ms  launches/apply {prof.pc_launches}", flush=True)
    del pc
