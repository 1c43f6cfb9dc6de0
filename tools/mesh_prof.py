"""One device mesh generation at C2 size (for an ncu launch list of csrc/devmesh.cu's kernels)."""
import ctypes as C, os, sys
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_1808_08328_b200 import _native as N
kind, n = sys.argv[1] if len(sys.argv) > 1 else "tet", int(sys.argv[2]) if len(sys.argv) > 2 else 40
for _ in range(2):
    h = C.c_void_p()
    N.call("dpp_mesh_generate_device", N.ctx(), 2 if kind in ("tri", "quad") else 3, N.KINDS[kind], n, C.byref(h))
    nv, nc, nf = C.c_int64(), C.c_int64(), C.c_int64()
    N.call("dpp_mesh_counts", h, C.byref(nv), C.byref(nc), C.byref(nf))
    N.call("dpp_mesh_destroy", h)
print(kind, n, nv.value, nc.value, nf.value)
