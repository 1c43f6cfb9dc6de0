cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
export DPP_PU_MODE=ws
timeout -s KILL 900 python -m pytest tests -m "gpu" -q -p no:cacheprovider --maxfail=40 -rf > gpurun_out/ws_pytest.log 2>&1; echo "ws pytest rc=$?"
tail -5 gpurun_out/ws_pytest.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-c3 --no-fast > gpurun_out/ws_bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/ws_bench.log
DPP_TRACE=1 TRACE_STEPS=3 timeout 300 python tools/trace_step.py > gpurun_out/ws_trace.log 2>&1; echo "trace rc=$?"
PROF_REPS=1 python tools/prof_pc.py > gpurun_out/ws_prof_plain.log 2>&1 && \
PROF_REPS=1 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/ws_pc_dram.csv python tools/prof_pc.py > gpurun_out/ws_prof_dram.log 2>&1
echo "dram rc=$?"
