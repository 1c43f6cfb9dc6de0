"""Generate the golden fixtures that pin the oracle to the real reference.

Run in the build container (the only place /root/reference exists):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

It imports the UNMODIFIED reference package `dppflow` read-only and dumps
small-size known answers into tests/golden/*.npz.  Nothing in the GPU tests,
smoke() or bench.py reads /root/reference; they read these fixtures.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np
import scipy.sparse as sp

sys.path.insert(0, "/root/reference/pkg/src")
import dppflow  # noqa: E402
from dppflow import blocksolve, linalg, problem  # noqa: E402
from dppflow.linalg import _strength_aggregates  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
BLOCKS = ("k1_uu", "k1_up", "k1_pu", "k1_pp", "k2_uu", "k2_up", "k2_pu", "k2_pp", "k12_pp", "k21_pp")
RHS = ("f1_u", "f1_p", "f2_u", "f2_p")
MESHES = [(2, "tri", 3), (2, "quad", 3), (3, "tet", 2), (3, "hex", 2)]


def put_csr(d, key, A):
    A = sp.csr_matrix(A)
    d[key + ".indptr"] = A.indptr.astype(np.int64)
    d[key + ".indices"] = A.indices.astype(np.int64)
    d[key + ".data"] = A.data
    d[key + ".shape"] = np.array(A.shape, dtype=np.int64)


def system(form, dim, kind, n, params=None):
    params = params or problem.DppParameters(gamma_b=(0.0,) * dim)
    mesh = dppflow.generate_unit_mesh(dim, kind, n)
    bcs = problem.boundary_data(problem.manufactured_solution(dim, params), mesh)
    return dppflow.assemble(mesh, form, params, bcs)


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def main():
    d = {}
    # -- meshes ---------------------------------------------------------------
    for dim, kind, n in MESHES + [(2, "tri", 7), (3, "tet", 3)]:
        m = dppflow.generate_unit_mesh(dim, kind, n)
        J, det = m.jacobians()
        p = f"mesh/{kind}{n}/"
        for a in ("vertices", "cells", "facet_vertex_ids", "cell_facets", "cell_facet_signs",
                  "facet_plus", "facet_minus", "facet_normals", "facet_measures"):
            d[p + a] = np.asarray(getattr(m, a))
        d[p + "J"], d[p + "det"] = J, det
    np.savez_compressed(os.path.join(OUT, "mesh.npz"), **d)

    # -- assembly: 3 formulations x 4 cell kinds -----------------------------
    d = {}
    for form in ("hdiv", "cgvms", "dgvms"):
        for dim, kind, n in MESHES:
            bs = system(form, dim, kind, n)
            p = f"asm/{form}/{kind}{n}/"
            for b in BLOCKS:
                put_csr(d, p + b, getattr(bs, b))
            for r in RHS:
                d[p + r] = getattr(bs, r)
            K, f = dppflow.monolithic_view(bs)
            put_csr(d, p + "K", K)
    np.savez_compressed(os.path.join(OUT, "assembly.npz"), **d)

    # -- linear algebra primitives on assembled blocks ------------------------
    d = {}
    rng = np.random.default_rng(20240817)
    for form, n in (("cgvms", 4), ("hdiv", 4)):
        bs = system(form, 2, "tri", n)
        p = f"lin/{form}/tri{n}/"
        fact = linalg.ilu0(bs.k1_uu)
        put_csr(d, p + "L", fact.L)
        put_csr(d, p + "U", fact.U)
        r = rng.standard_normal(bs.k1_uu.shape[0])
        d[p + "ilu_r"], d[p + "ilu_z"] = r, linalg.apply_ilu0(fact, r)
        S = linalg.schur_selfp(bs.k1_pp, bs.k1_pu, linalg.diag_lump(bs.k1_uu), bs.k1_up)
        put_csr(d, p + "S", S)
        h = linalg.amg_setup(S)
        d[p + "amg_levels"] = np.array(h.level_count)
        for li, lv in enumerate(h.levels):
            put_csr(d, p + f"amg{li}.A", lv.A)
            if lv.P is not None:
                put_csr(d, p + f"amg{li}.P", lv.P)
                d[p + f"amg{li}.agg"] = _strength_aggregates(lv.A, 0.5)
        r = rng.standard_normal(S.shape[0])
        d[p + "vc_r"], d[p + "vc_z"] = r, linalg.amg_vcycle(h, r)
        K, f = dppflow.monolithic_view(bs)
        for meth in ("scale", "field"):
            pc = blocksolve.build_preconditioner(bs, dppflow.method_config(meth))
            r = rng.standard_normal(K.shape[0])
            d[p + f"pc_{meth}_r"], d[p + f"pc_{meth}_z"] = r, pc(r)
            x, st = linalg.gmres(K, f, preconditioner=pc, rtol=1e-8)
            d[p + f"gmres_{meth}_x"] = x
            d[p + f"gmres_{meth}_its"] = np.array(st.iterations)
            d[p + f"gmres_{meth}_hist"] = np.array(st.history)
    A = sp.diags([-np.ones(254), 2.0 * np.ones(255), -np.ones(254)], [-1, 0, 1], format="csr")
    h = linalg.amg_setup(A)
    for li, lv in enumerate(h.levels):
        put_csr(d, f"lin/poisson255/amg{li}.A", lv.A)
        if lv.P is not None:
            put_csr(d, f"lin/poisson255/amg{li}.P", lv.P)
    r = rng.standard_normal(255)
    d["lin/poisson255/vc_r"], d["lin/poisson255/vc_z"] = r, linalg.amg_vcycle(h, r)
    np.savez_compressed(os.path.join(OUT, "linalg.npz"), **d)

    # -- full solves: iteration counts + solutions (small) ---------------------
    d = {}
    for form in ("hdiv", "cgvms", "dgvms"):
        for dim, kind, n in MESHES:
            bs = system(form, dim, kind, n)
            for meth in ("scale", "field"):
                rep = dppflow.solve(bs, dppflow.method_config(meth, rtol=1e-8))
                p = f"solve/{form}/{kind}{n}/{meth}/"
                d[p + "x"] = rep.solution_vector()
                d[p + "its"] = np.array(rep.stats.iterations)
                d[p + "relres"] = np.array(rep.stats.relative_residual)
                d[p + "hist"] = np.array(rep.stats.history)
    np.savez_compressed(os.path.join(OUT, "solve.npz"), **d)

    # -- medium / config-size summaries (hashes, counts, norms) ---------------
    summ = {}
    cases = [("cgvms", 2, "tri", 8, "field", 1e-9), ("cgvms", 2, "tri", 16, "scale", 1e-8),
             ("hdiv", 2, "tri", 16, "field", 1e-8), ("hdiv", 2, "tri", 5, "field", 1e-8),
             ("cgvms", 2, "tri", 64, "scale", 1e-8), ("hdiv", 2, "tri", 64, "field", 1e-8),
             ("cgvms", 3, "tet", 8, "scale", 1e-8), ("dgvms", 3, "tet", 4, "scale", 1e-8)]
    for form, dim, kind, n, meth, rtol in cases:
        params = problem.DppParameters(gamma_b=(0.0,) * dim)
        if dim == 3 and form == "cgvms":
            params = problem.DppParameters(k2=0.01, gamma_b=(0.0,) * dim)
        bs = system(form, dim, kind, n, params)
        K, f = dppflow.monolithic_view(bs)
        rep = dppflow.solve(bs, dppflow.method_config(meth, rtol=rtol))
        x = rep.solution_vector()
        S = linalg.schur_selfp(bs.k1_pp, bs.k1_pu, linalg.diag_lump(bs.k1_uu), bs.k1_up)
        aggs = []
        A = S
        h = linalg.amg_setup(S)
        for lv in h.levels[:-1]:
            aggs.append(sha(_strength_aggregates(lv.A, 0.5).astype(np.int64)))
        summ[f"{form}/{kind}{n}/{meth}/{rtol:g}/k2={params.k2}"] = {
            "its": rep.stats.iterations, "relres": rep.stats.relative_residual,
            "x_norm": float(np.linalg.norm(x)), "x_sum": float(x.sum()),
            "K_nnz": int(K.nnz), "K_sha_indptr": sha(K.indptr.astype(np.int64)),
            "K_sha_indices": sha(K.indices.astype(np.int64)),
            "S_nnz": int(S.nnz), "S_sha_data": sha(S.data),
            "amg_sizes": [int(lv.A.shape[0]) for lv in h.levels], "agg_sha": aggs,
            "f_norm": float(np.linalg.norm(f)), "dof": int(K.shape[0]),
        }
        del A
        print(form, kind, n, meth, rep.stats.iterations, flush=True)
    with open(os.path.join(OUT, "summary.json"), "w") as fh:
        json.dump(summ, fh, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
