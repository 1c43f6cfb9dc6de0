#!/bin/bash
# A/B of SpMV kernel choices on the C2 step profile (SpMV(K) and PC apply device times)
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
for v in "${@:-DPP_SPMV=stream DPP_SPMV=sell}"; do
  for e in $v; do :; done
  printf "%-40s " "$v"
  env $v PROF_REPS=20 PROF_FLUSH=1 python tools/prof_pc.py 2>&1 | tail -1
done
