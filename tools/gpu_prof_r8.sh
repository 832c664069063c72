#!/bin/bash
# ncu --set full of the cluster (few-factor) eigensolver / Cholesky kernels on cfg5r8
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
CMD="python bench.py --config cfg5r8 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-graphs"
timeout 600 $CMD > gpurun_out/r8_plain.log 2>&1 || { echo "plain run failed"; tail -3 gpurun_out/r8_plain.log; exit 1; }
for spec in "sytrd_tiled:2:1" "chol_tiled:2:1" "gemm_tc_kernel:20:4"; do
  k=${spec%%:*}; rest=${spec#*:}; s=${rest%%:*}; c=${rest#*:}
  timeout 900 ncu --set full --clock-control none -k regex:$k -s $s -c $c -o gpurun_out/r8_${k} -f $CMD > gpurun_out/ncu_r8_${k}.log 2>&1
  echo "$k: $(tail -1 gpurun_out/ncu_r8_${k}.log)"
done
python tools/ncu_full_summary.py gpurun_out/r01_ncu_full_cfg5r8.txt \
  "r01 ncu --set full --clock-control none (bench.py --config cfg5r8, eager steps; cluster sytrd / Cholesky, GEMMs)" \
  gpurun_out/r8_sytrd_tiled.ncu-rep gpurun_out/r8_chol_tiled.ncu-rep gpurun_out/r8_gemm_tc_kernel.ncu-rep
rm -f gpurun_out/r8_*.ncu-rep
