#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
rm -f gpurun_out/ws_ph.txt gpurun_out/ws_ph.txt.hop
PROF_CFG=${PROF_CFG:-C2} DPP_LIB=$PWD/ab_libs/wsph.so DPP_WS_PH=$PWD/gpurun_out/ws_ph.txt DPP_PC_NOGRAPH=1 PROF_REPS=1 timeout 600 python tools/prof_pc.py > gpurun_out/ws_ph.log 2>&1; echo "ph rc=$?"
python tools/gs_hop.py gpurun_out/ws_ph.txt.hop | cut -c1-250
python tools/ws_phases.py gpurun_out/ws_ph.txt | cut -c1-220 | head -12
