"""Summarise an ncu --metrics gpu__time_duration.sum CSV: last K launches (one PC apply)."""
import collections, csv, sys
path, k = sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 108
rows = list(csv.reader(open(path)))
hdr, data = None, []
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
sel = data[-k:]
agg = collections.defaultdict(lambda: [0, 0.0])
for d in sel:
    nm = d["Kernel Name"].split("(")[0][:50]
    agg[nm][0] += 1
    agg[nm][1] += float(d["Metric Value"]) / 1e3
tot = sum(v for _, v in agg.values())
for nm, (c, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{v:10.1f} us {100*v/tot:5.1f}%  x{c:<4d} {nm}")
print(f"total {tot:.1f} us over {len(sel)} launches")
if len(sys.argv) > 3:
    print([(d["Kernel Name"].split("(")[0][-12:], round(float(d["Metric Value"]) / 1e3, 1), d["Grid Size"]) for d in sel])
