"""k_trsv_lvl timeline (phase build, <f>.tl): per CTA and level team, median cycles from the
previous level's completion to this level's completion, and percentiles over all levels."""
import sys
import numpy as np
secs, cur = [], None
for line in open(sys.argv[1]):
    if line.startswith("#"):
        cur = {"hdr": line.strip(), "rows": []}
        secs.append(cur)
    elif cur is not None:
        cur["rows"].append([int(v) for v in line.split()])
want = sys.argv[2] if len(sys.argv) > 2 else "L=281"
for s in secs:
    if want not in s["hdr"]:
        continue
    a = np.array(s["rows"])
    print(s["hdr"])
    for c in (0, 5, 10, 15):
        b = a[a[:, 0] == c]
        if not len(b):
            continue
        # level completion = max over the level's steps
        lv = np.unique(b[:, 2])
        done = np.array([b[b[:, 2] == l][:, 5].max() for l in lv])
        d = np.diff(done)
        teams = lv[1:] % 4
        print(f"  cta {c}: levels {len(lv)}, delta pct10/50/90/99 {np.percentile(d, [10, 50, 90, 99]).astype(int)} | per team median "
              + " ".join(str(int(np.median(d[teams == t]))) for t in range(4)) + f" | mean {int(d.mean())}")
    break
