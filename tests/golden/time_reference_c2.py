"""Time the UNMODIFIED reference on config 2 through its own harness, run_case(repeats=3)
(reference spectrum.py:211-255: min over repeats of assembly_s and solve_s; mesh generation
excluded), in the build container.  Writes tests/golden/reference_c2_timing.json, which
bench.py quotes in its cpu_baseline sample (the GPU box has no /root/reference).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/time_reference_c2.py
"""
import json
import os
import platform
import sys
import time

sys.path.insert(0, "/root/reference/pkg/src")
from dppflow import problem, spectrum  # noqa: E402

t0 = time.perf_counter()
params = problem.DppParameters(k2=0.01, gamma_b=(0.0, 0.0, 0.0))
rec = spectrum.run_case("cgvms", "tet", 40, method="scale", rtol=1e-8, params=params, repeats=3)
out = {"config": "C2: cgvms tet 40^3, k2=0.01, scale, rtol 1e-8", "dof": rec.dof, "ksp": rec.ksp,
       "assembly_s": rec.assembly_s, "solve_s": rec.solve_s, "total_s": rec.total_s,
       "dof_per_s": rec.rates["total"], "repeats": 3, "wall_s": time.perf_counter() - t0,
       "host": platform.processor() or platform.machine(), "cpu_count": os.cpu_count(),
       "note": "reference spectrum.run_case, single-threaded numpy/scipy + pure-Python ILU(0)"}
with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "reference_c2_timing.json"), "w") as fh:
    json.dump(out, fh, indent=1)
print(json.dumps(out))
