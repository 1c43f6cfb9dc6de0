#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
REPS=3 DPP_TRACE=1 timeout 900 python tools/run_config.py C3 > gpurun_out/c3_trace.log 2>&1; tail -3 gpurun_out/c3_trace.log
python - <<'PY'
import re
lines=open('gpurun_out/c3_trace.log').read().split('\n')
# last rep: find index of last 'rep 1' line; take trace lines between rep1 and rep2
idx=[i for i,l in enumerate(lines) if l.strip().startswith('rep ')]
seg=lines[idx[-2]+1:idx[-1]] if len(idx)>=2 else lines
ev=[]
for l in seg:
    m=re.match(r"\[dpp-trace\] (\S+)\s+([\d.]+) ms", l)
    if m: ev.append((float(m.group(2)), m.group(1)))
import collections
agg=collections.defaultdict(lambda:[0,0.0])
for d,n in ev:
    agg[n][0]+=1; agg[n][1]+=d
for n,(c,t) in sorted(agg.items(), key=lambda x:-x[1][1])[:28]:
    print(f"{t:9.1f} ms x{c:3d} {n}")
PY
