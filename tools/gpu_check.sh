#!/bin/bash
# One GPU session: parity tests, smoke, bench (each stage time-boxed).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/nvsmi.txt 2>&1
STAGES="${STAGES:-fast slow smoke bench}"
for s in $STAGES; do
  case $s in
    fast)  timeout -s KILL ${T_FAST:-900} python -m pytest tests -m "gpu and not slow" -q -p no:cacheprovider --maxfail=40 -rf > gpurun_out/pytest_fast.log 2>&1; echo "fast rc=$?" ;;
    slow)  timeout -s KILL ${T_SLOW:-1200} python -m pytest tests -m "gpu and slow" -q -s -p no:cacheprovider -rf > gpurun_out/pytest_slow.log 2>&1; echo "slow rc=$?" ;;
    smoke) timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" ;;
    bench) timeout -s KILL ${T_BENCH:-900} python bench.py ${BENCH_ARGS:---steps 3 --warmup 3} > gpurun_out/bench.log 2>&1; echo "bench rc=$?" ;;
  esac
done
tail -3 gpurun_out/pytest_fast.log 2>/dev/null
tail -3 gpurun_out/pytest_slow.log 2>/dev/null
tail -2 gpurun_out/smoke.log 2>/dev/null
tail -2 gpurun_out/bench.log 2>/dev/null
