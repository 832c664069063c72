#!/bin/bash
# targeted ncu --set full captures of the cfg4 bench's kernels (one GPU, after a clean run)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 600 $CMD > gpurun_out/prof_plain_bench.log 2>&1 || { echo "plain run failed"; exit 1; }
for spec in "sytrd_tiled:8:2" "chol_smem:8:2" "invit:3:1" "bisect:3:1" "cluster_kernel:3:1" "gemm_tc_kernel:250:40"; do
  k=${spec%%:*}; rest=${spec#*:}; s=${rest%%:*}; c=${rest#*:}
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s $s -c $c \
    -o gpurun_out/prof_${k} -f $CMD > gpurun_out/ncu_${k}.log 2>&1
  echo "$k: $(tail -1 gpurun_out/ncu_${k}.log)"
done
python tools/ncu_full_summary.py gpurun_out/r01_ncu_full_cfg4.txt \
  "r01 ncu --set full --clock-control none (bench.py --steps 3 --warmup 3 cfg4; targeted captures per kernel)" \
  gpurun_out/prof_sytrd_tiled.ncu-rep gpurun_out/prof_chol_smem.ncu-rep gpurun_out/prof_invit.ncu-rep \
  gpurun_out/prof_bisect.ncu-rep gpurun_out/prof_cluster_kernel.ncu-rep gpurun_out/prof_gemm_tc_kernel.ncu-rep
# keep only the (small) sytrd report locally: the 64 MiB merge limit
rm -f gpurun_out/prof_gemm_tc_kernel.ncu-rep gpurun_out/prof_chol_smem.ncu-rep gpurun_out/prof_invit.ncu-rep \
      gpurun_out/prof_bisect.ncu-rep gpurun_out/prof_cluster_kernel.ncu-rep
du -sh gpurun_out
