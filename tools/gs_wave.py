"""Wavefront of a DPP_WS_PH dump of k_trsv_gs: per CTA, when its first / last chunk was solved (us after
the launch's earliest chunk), for the first launch of every triangle."""
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
    if key in seen:
        continue
    seen.add(key)
    a = np.array(s["rows"], dtype=np.float64)
    a = a[a[:, 8] > 0]
    t0 = a[:, 5].min()
    print("==", s["hdr"])
    C = int(hdr["C"])
    step = max(1, C // 24)
    for cta in list(range(0, C, step)) + [C - 1]:
        c = a[a[:, 0] == cta]
        if len(c) == 0:
            continue
        print(f"  cta {cta:3d}: chunks {int(c[:, 8].sum()):5d} first solved {(c[:, 5].min() - t0) / 1e3:8.1f} us, last {(c[:, 6].max() - t0) / 1e3:8.1f} us, "
              f"polls/chunk {c[:, 7].sum() / c[:, 8].sum():8.0f} cyc")
