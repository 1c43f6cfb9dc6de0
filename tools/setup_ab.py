"""A/B of per-call setup switches in ONE process (C2 PC setup, interleaved, medians).

    python tools/setup_ab.py "base:" "hostagg:DPP_AGG_HOST=1" "oldinv:DPP_BD_INV_OLD=1"

Each argument is  label:VAR=VAL,VAR=VAL  (empty = defaults); only switches the library
reads per call can be compared this way.
"""
import os
import sys
import time

sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import numpy as np  # noqa: E402

import paper_1808_08328_b200 as dpp  # noqa: E402

arms = []
for a in sys.argv[1:] or ["base:"]:
    label, _, kv = a.partition(":")
    env = dict(x.split("=", 1) for x in kv.split(",") if x)
    arms.append((label, env))
p = dpp.DppParameters(k2=0.01, gamma_b=(0.0, 0.0, 0.0))
m = dpp.generate_unit_mesh(3, "tet", int(os.environ.get("AB_N", "40")))
bcs = dpp.boundary_data(dpp.mms_3d(p), m)
cfg = dpp.method_config("scale", rtol=1e-8)
bs = dpp.assemble(m, "cgvms", p, bcs)
res = {label: [] for label, _ in arms}
reps = int(os.environ.get("REPS", "12"))
for rep in range(reps + 1):
    for label, env in arms:
        saved = {k: os.environ.get(k) for k in env}
        os.environ.update(env)
        pc = dpp.build_preconditioner(bs, cfg)
        if rep:
            res[label].append(1e3 * pc.setup_time_s)
        del pc
        for k, v in saved.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
for label, v in res.items():
    v = np.array(v)
    print(f"{label:12s} setup median {np.median(v):6.2f} ms  p25 {np.percentile(v, 25):6.2f}  "
          f"p75 {np.percentile(v, 75):6.2f}  min {v.min():6.2f}")
