"""Config-size known answers from the UNMODIFIED reference (dppflow), read-only.

Run in the build container (the only place /root/reference exists):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_configs.py [C1 C2 C3p C4pp]

Writes tests/golden/configs.json: per case the iteration count, relative residual, solution
norm / sum, a strided sample of the solution (every 997th entry), SHA-256 of the monolithic
pattern (indptr, indices), of S_p's pattern and values for both networks, the AMG level sizes
and the SHA-256 of every level's aggregates.  tests/test_config_golden.py checks the oracle
(CPU, C1) and the device path (GPU, all cases) against it.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
import dppflow  # noqa: E402
from dppflow import linalg, problem  # noqa: E402
from dppflow.linalg import _strength_aggregates  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "configs.json")
STRIDE = 997

# name: formulation, dim, cell, n, k2, method  (BASELINE.json configs; C3' / C4'' are the survey's
# reduced parity sizes of configs 3 (homogeneous-k MMS variant) and 4)
CASES = {
    "C1": ("hdiv", 2, "tri", 256, 0.1, "field"),
    "C2": ("cgvms", 3, "tet", 40, 0.01, "scale"),
    "C3p": ("cgvms", 3, "hex", 32, 0.01, "field"),
    "C4pp": ("dgvms", 3, "tet", 16, 0.1, "scale"),
}


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def case(name):
    form, dim, kind, n, k2, meth = CASES[name]
    t0 = time.perf_counter()
    params = problem.DppParameters(k2=k2, gamma_b=(0.0,) * dim)
    mesh = dppflow.generate_unit_mesh(dim, kind, n)
    bcs = problem.boundary_data(problem.manufactured_solution(dim, params), mesh)
    t1 = time.perf_counter()
    bs = dppflow.assemble(mesh, form, params, bcs)
    K, f = dppflow.monolithic_view(bs)
    rep = dppflow.solve(bs, dppflow.method_config(meth, rtol=1e-8))
    t2 = time.perf_counter()
    x = rep.solution_vector()
    out = {"form": form, "dim": dim, "kind": kind, "n": n, "k2": k2, "method": meth,
           "dof": int(K.shape[0]), "its": int(rep.stats.iterations),
           "relres": float(rep.stats.relative_residual), "converged": bool(rep.stats.converged),
           "x_norm": float(np.linalg.norm(x)), "x_sum": float(x.sum()),
           "x_sample_stride": STRIDE, "x_sample": [float(v) for v in x[::STRIDE]],
           "f_norm": float(np.linalg.norm(f)), "K_nnz": int(K.nnz),
           "K_sha_indptr": sha(K.indptr.astype(np.int64)), "K_sha_indices": sha(K.indices.astype(np.int64)),
           "reference_s": {"mesh": t1 - t0, "assemble_solve": t2 - t1,
                           "assembly_s": bs.stats.wall_time_s, "solve_s": rep.solve_s}}
    for net in (1, 2):
        uu, pp, pu, up = (getattr(bs, f"k{net}_{b}") for b in ("uu", "pp", "pu", "up"))
        S = linalg.schur_selfp(pp, pu, linalg.diag_lump(uu), up)
        h = linalg.amg_setup(S)
        out[f"S{net}"] = {"nnz": int(S.nnz), "sha_indptr": sha(S.indptr.astype(np.int64)),
                          "sha_indices": sha(S.indices.astype(np.int64)), "sha_data": sha(S.data),
                          "amg_sizes": [int(lv.A.shape[0]) for lv in h.levels],
                          "agg_sha": [sha(_strength_aggregates(lv.A, 0.5).astype(np.int64)) for lv in h.levels[:-1]]}
    print(f"{name}: {form} {kind} n={n} dof={out['dof']} its={out['its']} "
          f"({t2 - t1:.0f} s assemble+solve, {t1 - t0:.0f} s mesh)", flush=True)
    return out


def main():
    names = sys.argv[1:] or list(CASES)
    data = {}
    if os.path.exists(OUT):
        with open(OUT) as fh:
            data = json.load(fh)
    for name in names:
        data[name] = case(name)
        with open(OUT, "w") as fh:
            json.dump(data, fh, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
