#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
rm -f gpurun_out/ws_ph.txt
PROF_CFG=${PROF_CFG:-C4} DPP_LIB=$PWD/ab_libs/wsph.so DPP_WS_PH=$PWD/gpurun_out/ws_ph.txt DPP_PC_NOGRAPH=1 PROF_REPS=1 timeout 600 python tools/prof_pc.py > gpurun_out/ws_ph.log 2>&1; echo "ph rc=$?"
python tools/gs_wave.py gpurun_out/ws_ph.txt | cut -c1-200
