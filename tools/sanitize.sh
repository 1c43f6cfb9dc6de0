#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over one small C2-type solve (TET 6^3,
# scale split: ILU(0) k_ilu0, level analysis k_levels, dataflow / block-dense / level-mbarrier
# sweeps), logs into gpurun_out/sanitize_*.log
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
cat > /tmp/san_case.py <<'PY'
import sys, os
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import paper_1808_08328_b200 as dpp
p = dpp.DppParameters(k2=0.01, gamma_b=(0.0, 0.0, 0.0))
m = dpp.generate_unit_mesh(3, "tet", int(os.environ.get("SAN_N", "6")))
bs = dpp.assemble(m, "cgvms", p, dpp.boundary_data(dpp.mms_3d(p), m))
r = dpp.solve(bs, dpp.method_config("scale", rtol=1e-8))
print("converged", r.converged, "its", r.stats.iterations)
PY
for tool in memcheck racecheck synccheck; do
  for mode in flow lvl; do
    DPP_PU_MODE=$mode DPP_PC_NOGRAPH=1 timeout 1200 compute-sanitizer --tool $tool --print-limit 50 \
      python /tmp/san_case.py > gpurun_out/sanitize_${tool}_${mode}.log 2>&1
    echo "$tool $mode rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|converged' gpurun_out/sanitize_${tool}_${mode}.log | tr '\n' ' ')"
  done
done
