#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
bash tools/ab_pc.sh "X=0" "X=1"
timeout 300 python tools/ws_check.py 16 "DPP_PU_MODE=flow" "X=0" "DPP_GS_MIN_CLUSTERS=2" 2>&1 | tail -3
