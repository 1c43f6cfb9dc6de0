#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
PROF_CFG=C4 bash tools/ab_pc.sh "DPP_GS_CLUSTERS=3" "DPP_GS_CLUSTERS=4" "DPP_GS_CLUSTERS=8" "X=0"
PROF_CFG=C3 bash tools/ab_pc.sh "DPP_GS_CLUSTERS=3" "DPP_GS_CLUSTERS=4" "X=0"
PROF_CFG=C3 PROF_REPS=1 DPP_TRACE=1 timeout 900 python tools/prof_pc.py 2>&1 | grep -E "gs_plan|push_plan n=|gbd_plan" | head -20
