#!/bin/bash
# repeat the slow GPU parity tests to expose intermittent failures
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
for i in $(seq 1 ${REPS:-3}); do
  timeout -s KILL 600 python -m pytest tests -m "gpu and slow" -q -p no:cacheprovider -x > gpurun_out/flaky_$i.log 2>&1
  echo "run $i rc=$? $(tail -1 gpurun_out/flaky_$i.log)"
  grep -m3 "^E " gpurun_out/flaky_$i.log
done
