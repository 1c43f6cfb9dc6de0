"""Summaries of a profiling round (tools/profile_round.sh outputs in gpurun_out/) -> profiles/.

  r<NN>_bench_launches.csv.gz   the raw ncu launch list of `bench.py --steps 1 --warmup 1`
  r<NN>_bench_launch_summary.txt per-kernel count / total time / share of all launches
  r<NN>_arnoldi_step_dram.txt   one Arnoldi step (SpMV + PC apply), per kernel: time, DRAM bytes
  r<NN>_traffic.json            DRAM bytes per Arnoldi step (read by bench.py -> roofline.traffic)
  r<NN>_full_summary.txt        key --set full metrics of the captured dominant kernels
"""
import collections
import csv
import gzip
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")


def read_ncu_csv(path):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    return data


def short(name):
    return name.split("(")[0].replace("dpp::", "").replace("<unnamed>::", "")[:70]


def launch_summary(tag):
    src = os.path.join(OUT, "bench_launches.csv")
    with open(src, "rb") as f, gzip.open(os.path.join(PROF, f"{tag}_bench_launches.csv.gz"), "wb") as g:
        shutil.copyfileobj(f, g)
    data = [d for d in read_ncu_csv(src) if d["Metric Name"] == "gpu__time_duration.sum"]
    agg = collections.defaultdict(lambda: [0, 0.0])
    for d in data:
        agg[short(d["Kernel Name"])][0] += 1
        agg[short(d["Kernel Name"])][1] += float(d["Metric Value"]) / 1e3
    tot = sum(v for _, v in agg.values())
    lines = [f"ncu launch list of `python bench.py --steps 1 --warmup 1 --no-cpu-baseline` "
             f"(--metrics gpu__time_duration.sum --clock-control none): {len(data)} launches, "
             f"{tot / 1e3:.1f} ms of kernel time (serialised, cold caches under ncu).",
             "Covers warm-up + timed device step + e2e steps + the roofline profile; shares are what "
             "matter, not absolute times.", "",
             f"{'total us':>12} {'share':>6} {'count':>6}  kernel"]
    for nm, (c, v) in sorted(agg.items(), key=lambda x: -x[1][1])[:40]:
        lines.append(f"{v:12.1f} {100 * v / tot:5.1f}% {c:6d}  {nm}")
    open(os.path.join(PROF, f"{tag}_bench_launch_summary.txt"), "w").write("\n".join(lines) + "\n")
    print("\n".join(lines[:16]))


def step_dram(tag, pc_kernels):
    data = read_ncu_csv(os.path.join(OUT, "pc_dram.csv"))
    per = collections.OrderedDict()
    for d in data:
        per.setdefault(d["ID"], {"name": d["Kernel Name"]})[d["Metric Name"]] = float(d["Metric Value"])
    launches = list(per.values())[-(pc_kernels + 1):]   # last SpMV + one PC apply
    rows, tb, tt = [], 0.0, 0.0
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for d in launches:
        b = d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
        t = d.get("gpu__time_duration.sum", 0.0) / 1e3
        tb += b
        tt += t
        a = agg[short(d["name"])]
        a[0] += 1
        a[1] += t
        a[2] += b
    lines = [f"One Arnoldi step (CSR SpMV of K + one preconditioner apply = {pc_kernels} kernels), "
             "ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
             "(serialised; the two pore networks run concurrently outside ncu).",
             f"total DRAM traffic {tb / 1e6:.1f} MB, serialised kernel time {tt:.1f} us", "",
             f"{'us':>10} {'DRAM MB':>9} {'GB/s':>8} {'count':>6}  kernel"]
    for nm, (c, t, b) in sorted(agg.items(), key=lambda x: -x[1][1]):
        lines.append(f"{t:10.1f} {b / 1e6:9.2f} {b / max(t, 1e-9) / 1e3:8.1f} {c:6d}  {nm}")
    open(os.path.join(PROF, f"{tag}_arnoldi_step_dram.txt"), "w").write("\n".join(lines) + "\n")
    json.dump({"source": f"profiles/{tag}_arnoldi_step_dram.txt", "arnoldi_step_dram_bytes": tb,
               "spmv_dram_bytes": sum(l.get("dram__bytes_read.sum", 0) + l.get("dram__bytes_write.sum", 0)
                                      for l in launches[:1]),
               "pc_apply_dram_bytes": tb - sum(l.get("dram__bytes_read.sum", 0) +
                                               l.get("dram__bytes_write.sum", 0) for l in launches[:1])},
              open(os.path.join(PROF, f"{tag}_traffic.json"), "w"), indent=1)
    print("\n".join(lines[:14]))


def full_summary(tag):
    rep = os.path.join(OUT, f"{tag}_full.ncu-rep")
    out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr = rows[0]
    want = ["Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput", "Achieved Occupancy",
            "Registers Per Thread", "Grid Size", "Block Size", "Dynamic Shared Memory Per Block",
            "Executed Ipc Active", "L2 Hit Rate", "Cluster Size"]
    per = collections.OrderedDict()
    for r in rows[1:]:
        d = dict(zip(hdr, r))
        if d.get("Metric Name") in want:
            per.setdefault(d["ID"], {"name": short(d["Kernel Name"])})[d["Metric Name"]] = \
                f'{d["Metric Value"]} {d["Metric Unit"]}'.strip()
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics",
                          "dram__bytes_read.sum,dram__bytes_write.sum"], capture_output=True, text=True).stdout
    rr = list(csv.reader(raw.splitlines()))
    if len(rr) > 2:
        h = rr[0]
        for i, r in enumerate(rr[2:]):
            d = dict(zip(h, r))
            key = d.get("ID", str(i))
            if key in per:
                per[key]["dram bytes (read+write)"] = d.get("dram__bytes_read.sum", "?") + " + " + \
                    d.get("dram__bytes_write.sum", "?")
    lines = [f"ncu --set full --clock-control none --import-source on, kernels k_trsv_gs|k_spmv_sell|k_trsv_bd "
             f"of tools/prof_pc.py (C2 scale-split PC), report gpurun_out/{tag}_full.ncu-rep", ""]
    for k, d in per.items():
        lines.append(f"[{k}] {d.pop('name')}")
        for m, v in d.items():
            lines.append(f"    {m:36s} {v}")
    open(os.path.join(PROF, f"{tag}_full_summary.txt"), "w").write("\n".join(lines) + "\n")
    print("\n".join(lines[:40]))


if __name__ == "__main__":
    tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
    os.makedirs(PROF, exist_ok=True)
    launch_summary(tag)
    step_dram(tag, int(sys.argv[2]) if len(sys.argv) > 2 else 108)
    full_summary(tag)
