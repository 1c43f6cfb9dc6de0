#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
bash tools/ab_pc.sh "X=0" "DPP_WS_SLOTS=3" "DPP_WS_WARPS=10" "DPP_WS_WARPS=12" "DPP_WS_WARPS=6" "DPP_WS_WARPS=16" > gpurun_out/ws_ab.txt 2>&1
cat gpurun_out/ws_ab.txt
python tools/ws_check.py 16 "DPP_PU_MODE=flow" "X=0" "DPP_PU_MODE=ws" 2>&1 | tail -4
WS_TL_EXTRA="" bash tools/ws_tl.sh 2>&1 | grep -A2 "n=68921" | cut -c1-330
