"""One C2 step (assemble + PC setup + GMRES) through the public API with DPP_TRACE=1."""
import os, sys, time
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
os.environ.setdefault("DPP_TRACE", "1")
import paper_1808_08328_b200 as dpp
n = int(os.environ.get("TRACE_N", "40"))
p = dpp.DppParameters(k2=0.01, gamma_b=(0.0, 0.0, 0.0))
m = dpp.generate_unit_mesh(3, "tet", n)
bcs = dpp.boundary_data(dpp.mms_3d(p), m)
cfg = dpp.method_config(os.environ.get("TRACE_METHOD", "scale"), rtol=1e-8)
for rep in range(int(os.environ.get("TRACE_STEPS", "3"))):
    print(f"---- step {rep}", file=sys.stderr, flush=True)
    t0 = time.perf_counter()
    bs = dpp.assemble(m, "cgvms", p, bcs)
    t1 = time.perf_counter()
    r = dpp.solve(bs, cfg, want_solution=False)
    t2 = time.perf_counter()
    print(f"step {rep}: assemble {1e3*(t1-t0):.1f} ms, solve {1e3*(t2-t1):.1f} ms "
          f"(pc setup {1e3*r.pc_setup_s:.1f}), its {r.stats.iterations}", file=sys.stderr, flush=True)
    del bs, r
