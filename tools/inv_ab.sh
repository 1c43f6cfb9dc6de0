#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 300 python tools/ws_check.py 40 "DPP_BD_INV=sparse" "X=0" 2>&1 | tail -3
timeout 300 python tools/ws_check.py 16 "DPP_BD_INV=sparse" "X=0" 2>&1 | tail -3
for e in "DPP_BD_INV=sparse" "X=0"; do echo "== $e"; env $e timeout 600 python bench.py --steps 6 --warmup 3 --no-cpu-baseline --no-c3 --no-c4 --no-fast 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['value'], d['roofline']['pc_ms'], d['e2e']['value'])"; done
timeout -s KILL 900 python -m pytest tests -m "gpu and not slow" -q -p no:cacheprovider --maxfail=40 -rf -x > gpurun_out/pytest_fast.log 2>&1; echo "fast rc=$?"; tail -4 gpurun_out/pytest_fast.log
