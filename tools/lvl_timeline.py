"""Per-CTA level timeline of k_trsv_lvl (phase build, DPP_FLOW_PHASES=<f> writes <f>.tl):
cycles between consecutive level completions inside each CTA (SM clock), and the late-part
span (last wait passed -> arrival) per level."""
import sys
import numpy as np
secs, cur = [], None
for line in open(sys.argv[1]):
    if line.startswith("#"):
        cur = {"hdr": line[2:].strip(), "rows": []}
        secs.append(cur)
    elif cur is not None:
        cur["rows"].append([int(v) for v in line.split()])
for s in secs[: int(sys.argv[2]) if len(sys.argv) > 2 else 4]:
    a = np.array(s["rows"], dtype=np.int64)
    if a.size == 0:
        continue
    cta, step, lvl, tfirst, tlate, tdone = a.T
    out = []
    for c in np.unique(cta):
        m = cta == c
        lv, d, tl, tf = lvl[m], tdone[m], tlate[m], tfirst[m]
        o = np.argsort(lv)
        lv, d, tl, tf = lv[o], d[o], tl[o], tf[o]
        dd = np.diff(d)
        out.append((c, len(lv), np.median(dd) if len(dd) else 0, np.median(d - tl), np.median(d - tf), (d[-1] - d[0]) / max(len(lv) - 1, 1)))
    print(s["hdr"])
    for c, nl, med, late, whole, avg in out[:16]:
        print(f"  cta {c:3d}: {nl:4d} levels, level-to-level median {med:6.0f} mean {avg:6.0f} cyc | late->arrive {late:5.0f} | first->arrive {whole:6.0f}")
