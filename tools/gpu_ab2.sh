#!/bin/bash
# A/B: EA + precondition stages + cfg4 bench for the current library vs libbkfac_$1.so
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
for lib in libbkfac.so libbkfac_$1.so; do
  echo "== $lib"
  BKFAC_LIB=$PWD/paper_2210_08494_b200/$lib timeout 120 python tools/prof_ea.py time 2>&1 | grep -E "gemm|rror"
  BKFAC_LIB=$PWD/paper_2210_08494_b200/$lib timeout 120 python tools/prof_prec.py time 2>&1 | grep -E "gemm_prec|total|rror"
  BKFAC_LIB=$PWD/paper_2210_08494_b200/$lib timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/ab_$lib.log 2>&1
  python - <<PY
import json
l=[x for x in open("gpurun_out/ab_$lib.log") if x.startswith("{")][-1]
d=json.loads(l); print("bench", d["ms_per_step"], [(s["stage"], round(s["ms"]/d["steps"],3)) for s in d["stages"]][:12])
PY
done
