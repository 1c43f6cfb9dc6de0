"""Dataflow sweep timeline (DPP_FLOW_DEBUG=<file>): ILU apply + one V-cycle outside capture."""
import os, sys
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import numpy as np
import paper_1808_08328_b200 as dpp
p = dpp.DppParameters(k2=0.01, gamma_b=(0.0, 0.0, 0.0))
m = dpp.generate_unit_mesh(3, "tet", 40)
bs = dpp.assemble(m, "cgvms", p, dpp.boundary_data(dpp.mms_3d(p), m))
S = dpp.schur_selfp(bs.k1_pp, bs.k1_pu, dpp.diag_lump(bs.k1_uu), bs.k1_up)
f = dpp.ilu0(bs.k1_uu)
h = dpp.amg_setup(S)
for _ in range(2):
    z = dpp.apply_ilu0(f, np.ones(bs.k1_uu.shape[0]))
    z = dpp.amg_vcycle(h, np.ones(S.shape[0]))
