"""Hottest SASS instructions of one kernel in an ncu source-page CSV (--page source --csv
--print-source sass): samples, stall breakdown, shared-memory wavefronts (actual / ideal)."""
import csv
import sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
stall_cols = [h for h in hdr if h.startswith("stall_")]
data = []
for r in rows[2:]:
    if len(r) < len(hdr):
        continue
    try:
        s = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    except ValueError:
        continue
    data.append((s, r))
tot = sum(s for s, _ in data)
print("total samples", tot)
tops = {}
for s, r in data:
    for h in stall_cols:
        try:
            tops[h] = tops.get(h, 0) + int(r[ix[h]] or 0)
        except ValueError:
            pass
print("stall totals:", ", ".join(f"{k[6:]} {100 * v / tot:.1f}%" for k, v in sorted(tops.items(), key=lambda kv: -kv[1])[:8]))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
for s, r in sorted(data, key=lambda t: -t[0])[:n]:
    st = sorted(((int(r[ix[h]] or 0), h[6:]) for h in stall_cols if (r[ix[h]] or "0").isdigit()), reverse=True)[:3]
    wf = r[ix["L1 Wavefronts Shared"]]
    wi = r[ix["L1 Wavefronts Shared Ideal"]]
    print(f"{100 * s / tot:5.1f}% {r[ix['Address']]} {r[ix['Source']][:60]:60s} "
          + " ".join(f"{h}:{v}" for v, h in st) + (f" | smem wf {wf}/{wi}" if wf not in ("", "0") else ""))
