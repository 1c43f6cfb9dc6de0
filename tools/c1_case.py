import os, sys
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import paper_1808_08328_b200 as dpp
n = int(sys.argv[1])
p = dpp.DppParameters(gamma_b=(0.0, 0.0))
m = dpp.generate_unit_mesh(2, "tri", n)
bs = dpp.assemble(m, "hdiv", p, dpp.boundary_data(dpp.mms_2d(p), m))
r = dpp.solve(bs, dpp.method_config("field", rtol=1e-8))
print("its", r.stats.iterations)
