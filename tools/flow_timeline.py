"""Per-launch view of a dataflow sweep timeline (DPP_FLOW_DEBUG=<file>):
span, ns per level, mean step time of the warps with rows (landed -> rows done),
ring gaps (previous step done -> this block landed; > 0 means the ring starved)."""
import sys
import numpy as np
secs, cur = [], None
for line in open(sys.argv[1]):
    if line.startswith("#"):
        cur = {"hdr": line[2:].strip(), "rows": []}
        secs.append(cur)
    else:
        cur["rows"].append([int(v) for v in line.split()])
for s in secs:
    a = np.array(s["rows"], dtype=np.int64)
    if a.size == 0:
        continue
    cta, step, lvl, nr, t0, t1 = a.T
    L = lvl.max() + 1
    span = (t1.max() - t0.min()) / 1e3
    work = (t1 - t0).mean()
    gaps = []
    for c in np.unique(cta):
        m = cta == c
        tt0, tt1 = t0[m], t1[m]
        gaps.extend(tt0[1:] - tt1[:-1])
    gaps = np.array(gaps)
    # level completion times
    lend = np.zeros(L); 
    for i in range(len(a)):
        lend[lvl[i]] = max(lend[lvl[i]], t1[i])
    dl = np.diff(lend[lend > 0])
    print(f"{s['hdr']}: span {span:.1f} us / {L} levels = {span / L * 1e3:.0f} ns/level | step (land->done) mean {work:.0f} ns "
          f"| ring gap mean {gaps.mean():.0f} ns, >0 in {100 * (gaps > 0).mean():.0f}% | level-end delta median {np.median(dl):.0f} ns")
