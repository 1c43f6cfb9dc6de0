#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
bash tools/ab_pc.sh "X=0" "DPP_MERGE=2" "DPP_MERGE=2 DPP_WS_GMAX=32" "DPP_MERGE=3 DPP_WS_GMAX=32"
timeout 300 python tools/ws_check.py 40 "X=0" "DPP_MERGE=2 DPP_WS_GMAX=32" 2>&1 | tail -3
for e in "X=0" "DPP_MERGE=2 DPP_WS_GMAX=32"; do echo "== $e"; env $e DPP_TRACE=1 PROF_REPS=1 timeout 300 python tools/prof_pc.py 2>&1 | grep -E "merge_levels|gs_plan|push_plan n" | head -8; env $e timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-c3 --no-c4 --no-fast 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['value'], d['roofline']['pc_ms'], d['e2e']['value'])"; done
