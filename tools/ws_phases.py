"""Summarise a DPP_WS_PH dump (tools/variant_build.sh wsph "-DDPP_WS_PH"; DPP_PC_NOGRAPH=1): per sweep
launch of the global-stream kernel, cycles per chunk by phase, averaged over the warps of a CTA (first
launch of every triangle)."""
import sys
import numpy as np
secs, cur = [], None
for line in open(sys.argv[1]):
    if line.startswith("#"):
        cur = {"hdr": line[2:].strip(), "rows": []}
        secs.append(cur)
    elif cur is not None:
        cur["rows"].append([int(v) for v in line.split()])
names = ["head", "loads+groups", "tail"]
seen = set()
for s in secs:
    hdr = dict(kv.split("=") for kv in s["hdr"].split() if "=" in kv)
    key = (hdr["n"], hdr["L"])
    if key in seen:
        continue
    seen.add(key)
    a = np.array(s["rows"], dtype=np.float64)
    print("==", s["hdr"], f"({float(hdr['us']) * 1e3 / int(hdr['L']):.0f} ns/level)")
    C = int(hdr["C"])
    for cta in sorted(set([0, 1, 15, 16, 17, C // 2, C - 17, C - 16, C - 1])):
        if cta < 0 or cta >= C:
            continue
        c = a[a[:, 0] == cta]
        ch = c[:, 8].sum()
        if ch == 0:
            continue
        tot = c[:, 2:5].sum()
        print(f"  cta {cta:2d}: chunks {int(ch):5d} | per chunk per warp: total {tot / ch:6.0f} cyc = "
              + " + ".join(f"{n} {c[:, 2 + i].sum() / ch:5.0f}" for i, n in enumerate(names))
              + f" | polls inside groups {c[:, 7].sum() / ch:5.0f}")
