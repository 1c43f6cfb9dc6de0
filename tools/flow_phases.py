"""Summarise DPP_FLOW_PHASES output (phase-instrumented build, tools/flow_phases.sh):
per sweep launch, cycles per row-group iteration by phase, averaged over the warps with rows."""
import sys
import numpy as np
secs, cur = [], None
for line in open(sys.argv[1]):
    if line.startswith("#"):
        cur = {"hdr": line[2:].strip(), "rows": []}
        secs.append(cur)
    elif cur is not None:
        cur["rows"].append([int(v) for v in line.split()])
names = ["ring", "hdr", "ld+poll+fma", "reduce", "store", "idle"]
names_lvl = ["arrive", "earlywait", "early", "midwait+mid", "late", "latewait"]
for s in secs:
    a = np.array(s["rows"], dtype=np.float64)
    if a.size == 0:
        continue
    it = a[:, 8]
    tot = a[:, 2:8].sum(0)
    per = tot / it.sum()
    lvl = s["hdr"].startswith("lvl")
    hdr = dict(kv.split("=") for kv in s["hdr"].split() if "=" in kv)
    L = int(hdr["L"]); us = float(hdr["us"])
    print(f"{s['hdr']}: {us * 1e3 / L:.0f} ns/level | iters {int(it.sum())} over {len(a)} warps | "
          + " ".join(f"{n} {v:.0f}" for n, v in zip(names_lvl if lvl else names, per))
          + (f" | store+push" if lvl else " | spins/iter") + f" {a[:, 9].sum() / it.sum():.2f}")
