"""Known answers for discrete-field evaluation, L2 errors and run_case from the UNMODIFIED
reference (dppflow), read-only, in the build container:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_fields.py

Writes tests/golden/fields.npz: per case the reference solution x, DiscreteField.evaluate_all
of every field at three reference points, field_errors (spectrum.py:172-176), and for two cases
the run_case record (its, l2, DoF) plus a write_csv file (schema check).
"""

import json
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
import dppflow  # noqa: E402
from dppflow import problem, spectrum  # noqa: E402
from dppflow.assembly import solution_fields  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
CASES = [("hdiv", 2, "tri", 6), ("hdiv", 2, "quad", 5), ("hdiv", 3, "tet", 3), ("hdiv", 3, "hex", 3),
         ("cgvms", 2, "tri", 6), ("cgvms", 2, "quad", 5), ("cgvms", 3, "tet", 3), ("cgvms", 3, "hex", 3),
         ("dgvms", 2, "tri", 4), ("dgvms", 3, "tet", 2)]
REF_PTS = {2: np.array([[0.2, 0.3], [0.1, 0.1], [0.25, 0.5]]),
           3: np.array([[0.2, 0.3, 0.1], [0.1, 0.1, 0.1], [0.25, 0.2, 0.3]])}


def main():
    d = {}
    for form, dim, kind, n in CASES:
        params = problem.DppParameters(gamma_b=(0.0,) * dim)
        mms = problem.manufactured_solution(dim, params)
        mesh = dppflow.generate_unit_mesh(dim, kind, n)
        bs = dppflow.assemble(mesh, form, params, problem.boundary_data(mms, mesh))
        rep = dppflow.solve(bs, dppflow.method_config("field", rtol=1e-10))
        x = rep.solution_vector()
        p = f"{form}/{kind}{n}/"
        d[p + "x"] = x
        fields = solution_fields(bs, x)
        for name, fld in fields.items():
            d[p + "eval/" + name] = fld.evaluate_all(REF_PTS[dim])
        errs = spectrum.field_errors(bs, x, mms)
        d[p + "l2"] = np.array([errs[f] for f in ("u1", "p1", "u2", "p2")])
        print(form, kind, n, rep.stats.iterations, errs, flush=True)
    runs = {}
    for form, kind, n, meth in (("cgvms", "tri", 8, "scale"), ("hdiv", "tri", 8, "field")):
        rec = spectrum.run_case(form, kind, n, method=meth, rtol=1e-8)
        runs[f"{form}/{kind}{n}/{meth}"] = {"ksp": rec.ksp, "dof": rec.dof, "l2": rec.l2,
                                            "doa": rec.doa, "dos": rec.dos}
        spectrum.write_csv([rec], os.path.join(OUT, f"run_case_{form}_{kind}{n}.csv"))
    np.savez_compressed(os.path.join(OUT, "fields.npz"), **d)
    with open(os.path.join(OUT, "run_case.json"), "w") as fh:
        json.dump(runs, fh, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
