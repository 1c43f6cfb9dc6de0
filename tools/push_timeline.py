"""Critical-path view of a push-sweep timeline written by DPP_PU_DEBUG (tools/push_debug.py).

Per sweep launch: ns per level, and the average per-step phases of a CTA:
  ring   previous step's last push -> this step's block landed (TMA ring)
  levw   block landed -> every value of earlier levels landed (remote pushes)
  bar    -> CTA barrier passed
  work   barrier -> last warp computed and pushed its rows
and the producer->consumer hand-off: for each level, the latest 'work done' of a CTA at
level l-1 that pushes to the consumer vs the consumer's levw end (upper bound on push latency)."""
import sys
import numpy as np

secs, cur = [], None
for line in open(sys.argv[1]):
    if line.startswith("#"):
        cur = {"hdr": line[2:].strip(), "rows": []}
        secs.append(cur)
    else:
        cur["rows"].append([int(v) for v in line.split()])
last = int(sys.argv[2]) if len(sys.argv) > 2 else 0
for s in secs[-last:] if last else secs:
    a = np.array(s["rows"], dtype=np.int64)
    if a.size == 0:
        continue
    cta, step, lvl, nr, t_ring, t_lev, t_sync, t_done = a.T
    L = lvl.max() + 1
    span = (t_done.max() - t_sync.min()) / 1e3
    prev_done = np.r_[0, t_done[:-1]]
    first = np.r_[True, cta[1:] != cta[:-1]]
    ring = (t_ring - prev_done)[~first]
    levw = t_lev - t_ring
    bar = t_sync - t_lev
    work = t_done - t_sync
    # level hand-off: end of level l-1 (max t_done) -> first barrier pass at level l
    end = np.zeros(L, np.int64); start = np.full(L, np.iinfo(np.int64).max)
    for i in range(len(a)):
        end[lvl[i]] = max(end[lvl[i]], t_done[i]); start[lvl[i]] = min(start[lvl[i]], t_sync[i])
    hand = np.median(start[1:] - end[:-1])
    print(f"{s['hdr']}: span {span:.1f} us / {L} levels = {span / L * 1e3:.0f} ns/level | per step: ring {ring.mean():.0f} "
          f"levw {levw.mean():.0f} bar {bar.mean():.0f} work {work.mean():.0f} ns (rows {nr.mean():.1f}) | "
          f"level end -> next level start median {hand:.0f} ns")
