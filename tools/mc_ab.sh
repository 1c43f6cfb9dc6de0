#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
DPP_TRACE=1 TRACE_STEPS=3 timeout 300 python tools/trace_step.py 2>&1 | grep -E "tail_collapse|^step" | tail -6
timeout 300 python tools/ws_check.py 16 "DPP_AMG_TAIL=0" "X=0" 2>&1 | tail -2
bash tools/bench3.sh
