"""Alternate the config-size solves in one process (pool memory reuse between systems);
prints iterations / solution norms so run-to-run differences show up."""
import os, sys
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import numpy as np
import paper_1808_08328_b200 as dpp

CASES = [("cgvms", 2, "tri", 64, {}, "scale"), ("hdiv", 2, "tri", 256, {}, "field"),
         ("cgvms", 3, "tet", 16, {"k2": 0.01}, "field"), ("cgvms", 3, "hex", 16, {"k2": 0.01}, "field"),
         ("dgvms", 3, "tet", 6, {}, "scale"), ("cgvms", 3, "tet", 40, {"k2": 0.01}, "scale")]
ref = {}
for rep in range(int(os.environ.get("REPS", "4"))):
    for i, (form, dim, kind, n, kw, meth) in enumerate(CASES):
        p = dpp.DppParameters(gamma_b=(0.0,) * dim, **kw)
        m = dpp.generate_unit_mesh(dim, kind, n)
        mms = dpp.mms_2d(p) if dim == 2 else dpp.mms_3d(p)
        bs = dpp.assemble(m, form, p, dpp.boundary_data(mms, m))
        r = dpp.solve(bs, dpp.method_config(meth, rtol=1e-8))
        x = r.solution_vector()
        key = (r.stats.iterations, float(np.linalg.norm(x)))
        if i in ref and ref[i] != key:
            print(f"MISMATCH case {i} rep {rep}: {key} vs {ref[i]}", flush=True)
        ref.setdefault(i, key)
        print(rep, i, key, flush=True)
        del bs, r, x
print("done")
