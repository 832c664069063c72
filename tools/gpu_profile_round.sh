#!/bin/bash
# round profile: plain bench, launch list, full ncu captures of the top kernels
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 600 $CMD > gpurun_out/prof_plain_bench.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_cfg4.csv $CMD > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"sytrd_tiled|gemm_tc_kernel|chol_smem|invit|bisect" -s 60 -c 10 -o gpurun_out/prof_round1 $CMD > gpurun_out/ncu_full.log 2>&1
echo done
