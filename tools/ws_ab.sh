#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
L=$PWD/ab_libs
bash tools/ab_pc.sh "X=0" "DPP_GS_NAP=10" "DPP_GS_NAP=20" "DPP_GS_NAP=40" "DPP_GS_NAP=80" "DPP_GS_NAP=160" "DPP_GS_WARPS=12 DPP_GS_NAP=20" "DPP_LIB=$L/gs_16_4.so" "DPP_LIB=$L/gs_16_4.so DPP_GS_NAP=20" > gpurun_out/ws_ab.txt 2>&1
cat gpurun_out/ws_ab.txt
nvcc -arch=sm_100a -O3 -o /tmp/fp64lat tools/micro/fp64lat.cu && /tmp/fp64lat
