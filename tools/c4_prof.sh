#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
PROF_CFG=C4 PROF_REPS=1 DPP_TRACE=1 timeout 900 python tools/prof_pc.py > gpurun_out/c4_plain.log 2>&1; echo "plain rc=$?"; tail -1 gpurun_out/c4_plain.log
grep -E "make_tri|push_plan |gs_plan|ws_plan|bd_plan|amg level|levels=" gpurun_out/c4_plain.log | head -60
PROF_CFG=C4 PROF_REPS=1 PROF_RANGE=1 timeout 1500 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c4_launches.csv python tools/prof_pc.py > gpurun_out/c4_ncu.log 2>&1; echo "ncu rc=$?"
