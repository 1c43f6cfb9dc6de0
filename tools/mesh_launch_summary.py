"""Per-kernel time and DRAM bytes of one device mesh generation (the second of two in
gpurun_out/mesh_launches*.csv, tools/mesh_prof.py under ncu) -> profiles/<tag>_mesh_launches.txt"""
import csv, sys, os, collections
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag = sys.argv[1] if len(sys.argv) > 1 else "r02"
out = []
for title, f in (("TET 40^3 (C2: 384,000 cells, 777,600 facets; single 51-bit key sort)", "mesh_launches.csv"),
                 ("HEX 64^3 (C3: 262,144 cells, 798,720 facets; two-key sort, 19-bit ids)", "mesh_launches_hex.csv")):
    rows = list(csv.reader(open(os.path.join(ROOT, "gpurun_out", f))))
    hdr = next(r for r in rows if r and r[0] == "ID")
    data = [dict(zip(hdr, r)) for r in rows if len(r) == len(hdr) and r[0] != "ID"]
    per = collections.OrderedDict()
    for d in data:
        k = int(d["ID"])
        e = per.setdefault(k, {"name": d["Kernel Name"].split("(")[0].replace("dpp::", "")[:60]})
        e[d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
        e["unit_" + d["Metric Name"]] = d["Metric Unit"]
    ids = list(per)
    half = ids[len(ids) // 2:]            # the second generation (warm)
    def ns(e):
        v, u = e["gpu__time_duration.sum"], e["unit_gpu__time_duration.sum"]
        return v * {"ns": 1, "us": 1e3, "ms": 1e6}.get(u, 1)
    def by(e, m):
        v, u = e.get(m, 0.0), e.get("unit_" + m, "byte")
        return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
    out.append(f"{title}: {len(half)} launches, "
               f"{sum(ns(per[i]) for i in half) / 1e3:.1f} us of kernel time (serialised under ncu), "
               f"{sum(by(per[i], 'dram__bytes_read.sum') + by(per[i], 'dram__bytes_write.sum') for i in half) / 1e6:.1f} MB DRAM")
    out.append("        us   DRAM MB  kernel")
    for i in half:
        e = per[i]
        out.append(f"  {ns(e) / 1e3:8.1f}  {(by(e, 'dram__bytes_read.sum') + by(e, 'dram__bytes_write.sum')) / 1e6:8.2f}  {e['name']}")
    out.append("")
txt = ("Device mesh generation (csrc/devmesh.cu, dpp_mesh_generate_device): ncu --metrics gpu__time_duration.sum,"
       "dram__bytes_read.sum,dram__bytes_write.sum --clock-control none of tools/mesh_prof.py (second of two generations).\n"
       "The read-back of the host arrays (not kernels) and their numpy export take the rest of the 36-100 ms the API call needs.\n\n"
       + "\n".join(out))
open(os.path.join(ROOT, "profiles", f"{tag}_mesh_launches.txt"), "w").write(txt)
print(txt)
