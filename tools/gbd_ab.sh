#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
for e in "DPP_GBD_MAX=0" "X=0" "DPP_GBD_ROW=64"; do echo "== $e"; env $e timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-fast 2>&1 | tail -1 | python -c "
import sys,json; d=json.loads(sys.stdin.read()); print('c2', d['ms_per_step'], 'c3', d['c3_solve']['ms_per_step'], d['c3_solve']['ksp'], 'c4 pc', d['c4_sweep']['pc_ms'], d['c4_sweep']['pc_kernels_per_apply'])"; done
