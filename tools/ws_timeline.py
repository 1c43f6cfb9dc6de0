"""Summarise a DPP_WS_TL dump (tools/variant_build.sh wstl "-DDPP_WS_TL"; DPP_PC_NOGRAPH=1):
per sweep launch and CTA, cycles between consecutive chunk completions, time spent polling in the
last group (inputs of level l-1), tail (ready -> stored) and slack (landed -> last group)."""
import sys
import numpy as np
secs, cur = [], None
for line in open(sys.argv[1]):
    if line.startswith("#"):
        cur = {"hdr": line[2:].strip(), "rows": []}
        secs.append(cur)
    elif cur is not None:
        cur["rows"].append([int(v) for v in line.split()])
seen = set()
for s in secs:
    hdr = dict(kv.split("=") for kv in s["hdr"].split() if "=" in kv)
    key = (hdr["n"], hdr["L"])
    if key in seen and "-a" not in sys.argv:
        continue
    seen.add(key)
    a = np.array(s["rows"], dtype=np.int64)
    if a.size == 0:
        continue
    nw = int(hdr["warps"])
    print(f"== {s['hdr']}  ({float(hdr['us']) * 1e3 / int(hdr['L']):.0f} ns/level)")
    for cta in sorted(set(a[:, 0]))[: int(hdr["C"])]:
        c = a[a[:, 0] == cta]
        g = c[:, 2] * nw + c[:, 1]
        o = np.argsort(g)
        c = c[o]
        t0, t1, t2, t3 = (c[:, k].astype(np.float64) for k in (3, 4, 5, 6))
        dd = np.diff(t3)
        print(f" cta {cta:2d}: chunks {len(c):4d} span {t3[-1] - t0[0]:9.0f} cyc | done-to-done med {np.median(dd):6.0f} "
              f"p90 {np.percentile(dd, 90):6.0f} | lastpoll med {np.median(t2 - t1):6.0f} mean {np.mean(t2 - t1):6.0f} | "
              f"tail med {np.median(t3 - t2):5.0f} | slack(land->last) med {np.median(t1 - t0):6.0f} | "
              f"ready->next ready med {np.median(np.diff(t2)):6.0f}"
              + (f" | early-poll med {np.median(c[:, 7]):6.0f} mbar-wait med {np.median(c[:, 8]):6.0f}" if c.shape[1] > 8 else ""))
        if c.shape[1] > 8:   # per warp: period between consecutive chunks of one warp
            per = []
            for w in range(nw):
                cw = c[c[:, 1] == w]
                cw = cw[np.argsort(cw[:, 2])]
                per.extend(np.diff(cw[:, 3]))
            print(f"          per-warp chunk period med {np.median(per):6.0f} = proc {np.median(t1 - t0):6.0f} (of which early polls "
                  f"{np.median(c[:, 7]):6.0f}) + last poll {np.median(t2 - t1):5.0f} + tail {np.median(t3 - t2):5.0f} + rest")
    if "-v" in sys.argv:
        cta = int(sys.argv[sys.argv.index("-v") + 1])
        c = a[a[:, 0] == cta]
        g = c[:, 2] * nw + c[:, 1]
        c = c[np.argsort(g)]
        base = c[0, 3]
        for r in c[:200]:
            print("   ", r[1], r[2], r[3] - base, r[4] - base, r[5] - base, r[6] - base)
