#!/bin/bash
# cfg4 bench for several library variants: bash tools/gpu_libs.sh name1 name2 ... ("" = libbkfac.so)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
for v in "$@"; do
  lib=libbkfac${v:+_$v}.so
  BKFAC_LIB=$PWD/paper_2210_08494_b200/$lib timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/lib_$v.log 2>&1
  python - <<PY
import json
l=[x for x in open("gpurun_out/lib_$v.log") if x.startswith("{")][-1]
d=json.loads(l); print("$lib", d["ms_per_step"], [(s["stage"], round(s["ms"]/d["steps"],3)) for s in d["stages"] if s["stage"].startswith("eig")])
PY
done
