"""Warp-stream sweep check: solve a small C2-like case under DPP_PU_MODE=<modes> in fresh
processes and compare the solutions / iteration counts (first mode = reference)."""
import json, os, subprocess, sys
import numpy as np
ROOT = os.environ.get("GRAFT_REPO_ROOT", "/root/repo")
SCRIPT = r"""
import json, sys
import numpy as np
sys.path.insert(0, %r)
import paper_1808_08328_b200 as dpp
p = dpp.DppParameters(k2=0.01, gamma_b=(0.0, 0.0, 0.0))
m = dpp.generate_unit_mesh(3, "tet", int(sys.argv[2]))
bs = dpp.assemble(m, "cgvms", p, dpp.boundary_data(dpp.mms_3d(p), m))
r = dpp.solve(bs, dpp.method_config("scale", rtol=1e-8))
np.save(sys.argv[1], r.solution_vector())
print(json.dumps({"its": r.stats.iterations, "converged": bool(r.stats.converged)}))
""" % ROOT
n = sys.argv[1] if len(sys.argv) > 1 else "16"
ref = None
for k, envs in enumerate(sys.argv[2:] or ["", "DPP_PU_MODE=ws"]):
    env = dict(os.environ)
    for kv in envs.split():
        a, b = kv.split("=", 1)
        env[a] = b
    out = f"/tmp/ws_x{k}.npy"
    res = subprocess.run([sys.executable, "-c", SCRIPT, out, n], env=env, capture_output=True, text=True, timeout=400)
    if res.returncode != 0:
        print(f"[{envs}] FAILED rc={res.returncode}\n{res.stderr[-3000:]}")
        continue
    info = json.loads(res.stdout.strip().splitlines()[-1])
    x = np.load(out)
    if ref is None:
        ref = x
    print(f"[{envs}] {info} rel diff to first {np.linalg.norm(x - ref) / np.linalg.norm(ref):.3e}", flush=True)
