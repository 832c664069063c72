#!/bin/bash
# Cholesky A/B (cfg4 cores and cfg5r8) for the current library vs libbkfac_$1.so
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
for lib in libbkfac.so libbkfac_$1.so; do
  echo "== $lib"
  BKFAC_LIB=$PWD/paper_2210_08494_b200/$lib timeout 120 python tools/prof_sytrd.py 577 256 220 23 time 2>&1 | grep -E "chol|rror"
  for c in cfg4 cfg5r8; do
    BKFAC_LIB=$PWD/paper_2210_08494_b200/$lib timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/cab_$c.log 2>&1
    python - <<PY
import json
l=[x for x in open("gpurun_out/cab_$c.log") if x.startswith("{")][-1]
d=json.loads(l); print("$c", d["ms_per_step"], [(s["stage"], round(s["ms"]/d["steps"],3)) for s in d["stages"] if s["stage"].startswith("chol")])
PY
  done
done
