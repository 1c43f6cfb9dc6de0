#!/bin/bash
# ws sweep study: timeline of one un-graphed PC apply (variant build ab_libs/wstl.so)
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
for cfg in "X=0" "DPP_WS_SLOTS=2" ${WS_TL_EXTRA}; do
  tag=$(echo $cfg | tr ' =' '__')
  rm -f gpurun_out/ws_tl_$tag.txt
  env $cfg DPP_LIB=$PWD/ab_libs/wstl.so DPP_WS_TL=$PWD/gpurun_out/ws_tl_$tag.txt DPP_PC_NOGRAPH=1 PROF_REPS=1 timeout 300 python tools/prof_pc.py > gpurun_out/ws_tl.log 2>&1; echo "tl rc=$?"
  python tools/ws_timeline.py gpurun_out/ws_tl_$tag.txt > gpurun_out/ws_tl_summary_$tag.txt 2>&1
  grep -A3 "n=68921" gpurun_out/ws_tl_summary_$tag.txt | cut -c1-330
done
