"""Level hand-off inside CTA 0 from a DPP_WS_PH dump (<path>.hop): per chunk {level, t last group
entered, t inputs there, t x stored}; prints, per triangle (first launch), the cycles from the
previous level's last store to this level's inputs being seen (hand-off), the solve tail (inputs
seen -> x stored), and the level period."""
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
    if key in seen or not s["rows"]:
        continue
    seen.add(key)
    a = np.array(s["rows"], dtype=np.int64)
    lev = a[:, 2]
    by = {}
    for l in np.unique(lev):
        c = a[lev == l]
        by[int(l)] = (c[:, 3].min(), c[:, 4].max(), c[:, 5].max(), c[:, 4] - c[:, 3])   # enter, ready(max), stored(max), waits
    ls = sorted(by)
    hand, tail, per, waited = [], [], [], []
    for l0, l1 in zip(ls[:-1], ls[1:]):
        if l1 != l0 + 1:
            continue
        hand.append(by[l1][1] - by[l0][2])
        tail.append(by[l1][2] - by[l1][1])
        per.append(by[l1][2] - by[l0][2])
        waited.append(by[l1][3].max())
    hand, tail, per, waited = map(np.array, (hand, tail, per, waited))
    w = waited > 50   # levels whose last group really waited
    print("==", s["hdr"], f"levels seen {len(ls)}")
    print(f"   level period med {np.median(per):6.0f} cyc | hand-off (prev level stored -> inputs seen) med {np.median(hand[w]) if w.any() else float('nan'):6.0f} "
          f"p25 {np.percentile(hand[w], 25) if w.any() else float('nan'):6.0f} | tail (inputs seen -> stored) med {np.median(tail):5.0f} | "
          f"levels that waited {w.sum()} of {len(w)}")
