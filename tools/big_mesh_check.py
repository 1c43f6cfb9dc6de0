"""Device mesh generation at sizes far beyond the configs (2-9 M cells): closed-form facet count,
strictly increasing facet tuples, plus < minus, volumes (run on a B200: python tools/big_mesh_check.py)."""
import sys, time
import os
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
from tests.test_gpu_mesh import device_mesh
for dim, kind, n in [(3, "hex", 128), (3, "tet", 100), (2, "tri", 2048), (2, "quad", 3000)]:
    t0 = time.perf_counter()
    m = device_mesh(dim, kind, n)
    dt = time.perf_counter() - t0
    F = {"tri": 3 * n * n + 2 * n, "quad": 2 * n * (n + 1), "tet": 12 * n ** 3 + 6 * n * n, "hex": 3 * n * n * (n + 1)}[kind]
    assert m.n_facets == F, (m.n_facets, F)
    fv = m.facet_vertex_ids
    d = fv[1:] - fv[:-1]
    first = np.argmax(d != 0, axis=1)
    assert np.all(d[np.arange(len(d)), first] > 0)       # strictly increasing lexicographically
    inner = m.facet_minus >= 0
    assert np.all(m.facet_plus[inner] < m.facet_minus[inner])
    J, det = m.jacobians()
    ref = {"tri": 0.5, "quad": 1.0, "tet": 1.0 / 6.0, "hex": 1.0}[kind]
    assert abs(det.sum() * ref - 1.0) < 1e-10
    print(f"{kind} {n}: {m.n_cells} cells, {F} facets, {dt:.2f} s ok", flush=True)
    del m
