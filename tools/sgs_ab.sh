#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
bash tools/ab_pc.sh "DPP_SGS_PLAIN=1" "X=0"
timeout 300 python tools/ws_check.py 40 "DPP_SGS_PLAIN=1" "X=0" 2>&1 | tail -3
timeout 300 python tools/ws_check.py 16 "DPP_SGS_PLAIN=1" "X=0" 2>&1 | tail -3
timeout -s KILL 1200 python -m pytest tests -m "gpu" -q -p no:cacheprovider --maxfail=40 -rf > gpurun_out/pytest_all.log 2>&1; echo "all rc=$?"; tail -6 gpurun_out/pytest_all.log
timeout 600 python bench.py --steps 6 --warmup 3 --no-cpu-baseline --no-c3 --no-fast 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['value'], d['roofline'], d['e2e']['value'], d['c4_sweep']['pc_ms'])"
