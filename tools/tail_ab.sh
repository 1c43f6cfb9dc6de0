#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
bash tools/ab_pc.sh "X=0" "DPP_AMG_TAIL=0" 2>&1 | tee gpurun_out/tail_ab.txt
python tools/ws_check.py 16 "DPP_AMG_TAIL=0" "X=0" 2>&1 | tail -3
python tools/ws_check.py 40 "DPP_AMG_TAIL=0" "X=0" 2>&1 | tail -3
DPP_TRACE=1 TRACE_STEPS=2 timeout 300 python tools/trace_step.py > gpurun_out/tail_trace.log 2>&1; grep -E "tail_collapse|^step|amg.total|pc.setup|join_smoothers" gpurun_out/tail_trace.log | tail -20
timeout -s KILL 900 python -m pytest tests -m "gpu and not slow" -q -p no:cacheprovider --maxfail=40 -rf > gpurun_out/pytest_fast.log 2>&1; echo "fast rc=$?"; tail -5 gpurun_out/pytest_fast.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-c3 --no-c4 --no-fast 2>&1 | tail -1 | cut -c1-1500
