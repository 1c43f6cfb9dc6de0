#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout -s KILL 1200 python -m pytest tests -m "gpu" -q -p no:cacheprovider --maxfail=40 -rf > gpurun_out/pytest_all.log 2>&1; echo "all rc=$?"; tail -4 gpurun_out/pytest_all.log
PROF_CFG=C3 PROF_REPS=1 PROF_RANGE=1 timeout 1500 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c3_launches.csv python tools/prof_pc.py > gpurun_out/c3_ncu.log 2>&1; echo "ncu rc=$?"
