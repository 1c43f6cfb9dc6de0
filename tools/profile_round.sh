#!/bin/bash
# Round profiling: plain bench run, then launch list and full captures (one ncu use per call).
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/prof_bench_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/bench_launches.csv \
    python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/prof_bench_ncu.log 2>&1
echo "launch list rc=$?"
python tools/prof_pc.py > gpurun_out/prof_pc_plain.log 2>&1 && \
PROF_REPS=1 ncu --set full --clock-control none --import-source on -k regex:"k_trsv_cluster|k_spmv|k_trsv_block" -c 12 \
    -o gpurun_out/r01_full python tools/prof_pc.py > gpurun_out/prof_full.log 2>&1
echo "full capture rc=$?"
