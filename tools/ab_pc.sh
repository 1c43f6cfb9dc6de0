#!/bin/bash
# PC-apply timing (graph replay, CUDA events) for a list of env settings: ab_pc.sh "A=1" "A=2 B=3" ...
cd "${GRAFT_REPO_ROOT:-/root/repo}"
for envs in "$@"; do
  echo "== $envs"
  env $envs PROF_REPS=${PROF_REPS:-20} timeout 300 python tools/prof_pc.py 2>&1 | tail -1
done
