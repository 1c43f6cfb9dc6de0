"""One C2 PC setup between cudaProfilerStart/Stop (ncu --profile-from-start off target)."""
import ctypes as C, os, sys, time
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import paper_1808_08328_b200 as dpp
p = dpp.DppParameters(k2=0.01, gamma_b=(0.0, 0.0, 0.0))
m = dpp.generate_unit_mesh(3, "tet", 40)
bcs = dpp.boundary_data(dpp.mms_3d(p), m)
cfg = dpp.method_config("scale", rtol=1e-8)
rt = C.CDLL("libcudart.so.12")
for rep in range(3):
    bs = dpp.assemble(m, "cgvms", p, bcs)
    bs.device()
    if rep == 2:
        rt.cudaDeviceSynchronize(); rt.cudaProfilerStart()
    t0 = time.perf_counter()
    pc = dpp.build_preconditioner(bs, cfg)
    rt.cudaDeviceSynchronize()
    t1 = time.perf_counter()
    if rep == 2:
        rt.cudaProfilerStop()
    print(f"setup {1e3 * (t1 - t0):.1f} ms", file=sys.stderr)
    del pc, bs
