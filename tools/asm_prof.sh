#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
python tools/assembly_launches.py 2>&1 | tail -4
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/asm_launches.csv python tools/assembly_launches.py > gpurun_out/asm_ncu.log 2>&1; echo "ncu rc=$?"
DPP_TRACE=ev TRACE_STEPS=3 timeout 300 python tools/trace_step.py 2>&1 | grep -E "evtrace.*assemble" | tail -12
