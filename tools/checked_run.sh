#!/bin/bash
# GPU suite + determinism stress under the checked library (ab_libs/checked.so)
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
export DPP_LIB=$PWD/ab_libs/checked.so
timeout -s KILL 1500 python -m pytest tests -m "gpu" -q -p no:cacheprovider --maxfail=40 -rf > gpurun_out/checked_pytest.log 2>&1; echo "checked pytest rc=$?"; tail -4 gpurun_out/checked_pytest.log
timeout 900 python tools/stress_configs.py > gpurun_out/checked_stress.log 2>&1; echo "stress rc=$?"; grep -c MISMATCH gpurun_out/checked_stress.log; tail -8 gpurun_out/checked_stress.log
DPP_GS_MIN_CLUSTERS=2 timeout 900 python tools/stress_configs.py > gpurun_out/checked_stress_mc.log 2>&1; echo "stress (2 clusters) rc=$?"; grep -c MISMATCH gpurun_out/checked_stress_mc.log; tail -3 gpurun_out/checked_stress_mc.log
