cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2_pytest_f1.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2_pytest_f1.log
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv > gpurun_out/r2_smi_f1.txt
timeout 900 python bench.py > gpurun_out/r2_bench_f1.json 2> gpurun_out/r2_bench_f1.err
echo "bench rc=$?" >> gpurun_out/r2_bench_f1.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2_bench_ref_f1.json 2> gpurun_out/r2_bench_ref_f1.err
timeout 300 python tools/prof_cfg5.py > gpurun_out/r2_prof_plain_f1.log 2>&1 && \
ncu --set full --import-source on --nvtx --nvtx-include "prec/" -k regex:gemm_tc -s 4 -c 1 -o gpurun_out/r2_precout python tools/prof_cfg5.py > gpurun_out/r2_ncu_precout.log 2>&1
timeout 600 python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/r2_bench_small.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/r2_launches_cfg5.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/r2_ncu_launches.log 2>&1
