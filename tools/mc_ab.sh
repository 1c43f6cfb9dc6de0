#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
for e in "X=0" "DPP_FORK_MASK=5" "DPP_FORK_MASK=3" "DPP_FORK_MASK=1" "DPP_FORK_MASK=6" "DPP_SERIAL_SETUP=1" "X=1"; do echo "== $e"; env $e timeout 600 python bench.py --steps 8 --warmup 3 --no-cpu-baseline --no-c3 --no-c4 --no-fast 2>/dev/null | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['value'], d['config']['ksp'])"; done
