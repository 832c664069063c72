# Scratch job for one gpurun call (rewritten per call; the outputs land in gpurun_out/).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python tools/prof_cfg5.py --stage-nvtx > gpurun_out/s2h_prof_plain.log 2>&1 && \
ncu --set full --import-source on --nvtx --nvtx-include "gemm_sbr_update/" -k regex:gemm_tc -c 1 -o gpurun_out/s2h_sbrupd python tools/prof_cfg5.py --stage-nvtx > gpurun_out/s2h_ncu1.log 2>&1
ncu --set full --import-source on --nvtx --nvtx-include "gemm_resid/" -k regex:gemm_tc -c 1 -o gpurun_out/s2h_resid python tools/prof_cfg5.py --stage-nvtx > gpurun_out/s2h_ncu2.log 2>&1
ncu --set full --import-source on --nvtx --nvtx-include "gemm_sbr_x/" -k regex:gemm_tc -c 1 -o gpurun_out/s2h_sbrx python tools/prof_cfg5.py --stage-nvtx > gpurun_out/s2h_ncu3.log 2>&1
timeout 600 python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/s2h_bench_small.json 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"gemm_tc|gemm_splitk|sbr_|chol|bisect|invit|cluster|backtr|ew_|prec_|nonfinite|sytrd|philox|colidx" --csv --log-file gpurun_out/s2h_launches_cfg5.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/s2h_ncu_launches.log 2>&1
echo done
