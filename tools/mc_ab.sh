#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout -s KILL 1200 python -m pytest tests -m "gpu" -q -p no:cacheprovider --maxfail=40 -rf > gpurun_out/pytest_all.log 2>&1; echo "all rc=$?"; tail -4 gpurun_out/pytest_all.log
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/bench_now.json; python -c "
import json; d=json.load(open('gpurun_out/bench_now.json')); print('c2', d['ms_per_step'], d['value'], d['roofline']['pc_ms'], d['roofline']['frac'], 'e2e', d['e2e']['value']); print('c3', d['c3_solve']['ms_per_step'], d['c3_solve']['ksp']); print('c4', d['c4_sweep']['pc_ms'], d['c4_sweep']['roofline']['frac'], d['c4_sweep']['fast_mode']['pc_ms']); print('fast', d['fast_mode']['ms_per_step'], d['fast_mode']['pc_ms'])"
