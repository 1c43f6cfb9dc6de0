#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
for i in 1 2 3 4 5; do timeout 600 python bench.py --no-cpu-baseline --no-c3 --no-c4 --no-fast 2> gpurun_out/bench3_$i.err | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['value'], d['roofline']['pc_ms'], 'e2e', d['e2e']['value'], d['clocks'])"; grep "device step" gpurun_out/bench3_$i.err | tr '\n' ' '; echo; done
