#!/bin/bash
# EA side-stream grid cap sweep (cfg4 bench)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
for cap in ${CAPS:-0 16 32 64}; do
  BKFAC_EA_CAP=$cap timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_cap$cap.log 2>&1
  python - <<PY
import json
l=[x for x in open("gpurun_out/bench_cap$cap.log") if x.startswith("{")][-1]
d=json.loads(l); print("cap $cap", d["ms_per_step"], [(s["stage"], round(s["ms"]/d["steps"],3)) for s in d["stages"]][:3])
PY
done
