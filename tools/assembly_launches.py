"""One C2 assembly between cudaProfilerStart/Stop (ncu --profile-from-start off target)."""
import ctypes as C, os, sys, time
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import paper_1808_08328_b200 as dpp
from paper_1808_08328_b200 import _native as N
p = dpp.DppParameters(k2=0.01, gamma_b=(0.0, 0.0, 0.0))
m = dpp.generate_unit_mesh(3, "tet", 40)
bcs = dpp.boundary_data(dpp.mms_3d(p), m)
rt = C.CDLL("libcudart.so.12")
for rep in range(4):
    if rep == 3:
        rt.cudaDeviceSynchronize(); rt.cudaProfilerStart()
    t0 = time.perf_counter()
    bs = dpp.assemble(m, "cgvms", p, bcs)
    bs.device()
    N.sync()
    t1 = time.perf_counter()
    if rep == 3:
        rt.cudaProfilerStop()
    print(f"assemble {1e3 * (t1 - t0):.2f} ms", file=sys.stderr)
    del bs
