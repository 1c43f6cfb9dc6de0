"""C2 PC setup timeline from device events (DPP_TRACE=ev: every trace scope records a
CUDA event pair on its own stream, no synchronisation added), last of REPS setups.

    python tools/setup_timeline.py            # on the GPU box
prints every scope as  start end duration(ms) host-thread name, sorted by start.
"""
import os
import subprocess
import sys

root = os.environ.get("GRAFT_REPO_ROOT", "/root/repo")
env = dict(os.environ, DPP_TRACE="ev", REPS=os.environ.get("REPS", "3"))
p = subprocess.run([sys.executable, os.path.join(root, "tools/setup_once.py")], env=env,
                   capture_output=True, text=True)
print(p.stdout)
blocks, cur = [], None
for line in p.stderr.splitlines():
    if not line.startswith("[dpp-evtrace]"):
        continue
    if "==" in line:
        cur = []
        blocks.append(cur)
        continue
    f = line.split()
    cur.append((float(f[1]), float(f[2]), float(f[3]), f[4], " ".join(f[5:])))
if not blocks:
    print(p.stderr[-3000:])
    sys.exit(1)
rows = sorted(blocks[-1])
for a, b, d, t, name in rows:
    print(f"{a:9.3f} {b:9.3f} {d:8.3f} {t} {name}")
