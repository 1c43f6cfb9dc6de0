"""One assemble + PC setup (+ solve) on C2 through the public API (profiling target)."""
import os, sys
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import paper_1808_08328_b200 as dpp
p = dpp.DppParameters(k2=0.01, gamma_b=(0.0, 0.0, 0.0))
m = dpp.generate_unit_mesh(3, "tet", int(os.environ.get("TRACE_N", "40")))
bcs = dpp.boundary_data(dpp.mms_3d(p), m)
cfg = dpp.method_config("scale", rtol=1e-8)
for _ in range(int(os.environ.get("REPS", "2"))):
    bs = dpp.assemble(m, "cgvms", p, bcs)
    r = dpp.solve(bs, cfg, want_solution=False)
    print("its", r.stats.iterations, "setup ms", 1e3 * r.pc_setup_s, flush=True)
    del bs, r
