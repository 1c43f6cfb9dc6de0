#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
for e in "X=0" "CUDA_DEVICE_MAX_CONNECTIONS=32" "X=1" "CUDA_DEVICE_MAX_CONNECTIONS=32" "CUDA_DEVICE_MAX_CONNECTIONS=16"; do echo "== $e"; env $e timeout 600 python bench.py --steps 6 --warmup 3 --no-cpu-baseline --no-c3 --no-c4 --no-fast 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['value'], d['roofline']['pc_ms'], d['e2e']['value'])"; done
