#!/bin/bash
# Round profiling (each ncu use only after the same command exited 0 without ncu):
#   1. bench launch list (gpu__time_duration per kernel launch, clocks untouched)
#   2. DRAM bytes + duration of every kernel of one Arnoldi step (SpMV + PC apply)
#   3. full capture of the dominant kernels (push sweeps, block-dense sweep, SpMV)
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "bench rc=$?"
python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-c3 --no-c4 --no-fast --no-extras > gpurun_out/prof_bench_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/bench_launches.csv \
    python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-c3 --no-c4 --no-fast --no-extras > gpurun_out/prof_bench_ncu.log 2>&1
echo "launch list rc=$?"
PROF_REPS=1 python tools/prof_pc.py > gpurun_out/prof_pc_plain.log 2>&1 && \
PROF_REPS=1 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/pc_dram.csv python tools/prof_pc.py > gpurun_out/prof_pc_dram.log 2>&1
echo "dram pass rc=$?"
PROF_RANGE=1 PROF_REPS=1 ncu --profile-from-start off --set full --clock-control none --import-source on \
    -k regex:"k_trsv_gs|k_spmv_sell|k_trsv_bd" -c 10 -o gpurun_out/${ROUND:-r02}_full python tools/prof_pc.py > gpurun_out/prof_full.log 2>&1
echo "full capture rc=$?"
