"""Critical-path view of a push-sweep timeline written by DPP_PU_DEBUG (tools/push_debug.py).

Per section (one sweep launch): per level, when its rows started (first CTA past the
barrier with a block of that level) and finished (last push), and the average gaps."""
import sys
import numpy as np

secs, cur = [], None
for line in open(sys.argv[1]):
    if line.startswith("#"):
        cur = {"hdr": line[2:].strip(), "rows": []}
        secs.append(cur)
    else:
        cur["rows"].append([int(v) for v in line.split()])
for s in secs[-int(sys.argv[2]) if len(sys.argv) > 2 else 0:]:
    a = np.array(s["rows"], dtype=np.int64)
    if a.size == 0:
        continue
    cta, step, lvl, nr, t_ring, t_lev, t_sync, t_done = a.T
    t0 = t_sync.min()
    L = lvl.max() + 1
    start = np.full(L, np.iinfo(np.int64).max); end = np.zeros(L, np.int64); ncta = np.zeros(L, int)
    for i in range(len(a)):
        start[lvl[i]] = min(start[lvl[i]], t_sync[i]); end[lvl[i]] = max(end[lvl[i]], t_done[i]); ncta[lvl[i]] += 1
    span = (end.max() - t0) / 1e3
    comp = np.mean(t_done - t_sync) / 1e3
    wait_ring = np.mean(t_ring - np.r_[t_done[:1], t_done[:-1]]) / 1e3
    gap = np.mean(t_sync - t_lev) / 1e3
    # level-to-level: next level's first start minus this level's end
    hand = np.median(start[1:] - end[:-1]) / 1e3
    print(f"{s['hdr']}: span {span:.1f} us over {L} levels = {span / L * 1e3:.0f} ns/level; per step: "
          f"compute+push {comp * 1e3:.0f} ns, barrier {gap * 1e3:.0f} ns; median end(l)->start(l+1) {hand * 1e3:.0f} ns; "
          f"CTAs per level {ncta.mean():.1f}")
