"""Per-launch table from an ncu --csv launch list (gpu__time_duration + launch metrics)."""
import collections, csv, sys
lines = [l for l in open(sys.argv[1]) if l.startswith('"')]
rows = list(csv.reader(lines))
h = rows[0]
ki, mi, vi, ii, si = (h.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "ID", "Stream"))
d = collections.OrderedDict()
for r in rows[1:]:
    e = d.setdefault(r[ii], {"name": r[ki], "stream": r[si]})
    e[r[mi]] = r[vi]
skip = int(sys.argv[2]) if len(sys.argv) > 2 else 0
for k, v in list(d.items())[skip:]:
    print(k, v["stream"], v["name"].split("(")[0][:48], v.get("gpu__time_duration.sum"), v.get("launch__grid_size"),
          v.get("launch__block_size"), v.get("launch__cluster_size", ""))
