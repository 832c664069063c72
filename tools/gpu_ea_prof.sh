cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 300 python tools/bench_ea.py > gpurun_out/bench_ea.log 2>&1; cat gpurun_out/bench_ea.log
timeout 300 python tools/bench_ea.py --once > /dev/null 2>&1 && \
timeout 600 ncu --set full --import-source on --clock-control none -k regex:gemm_tc_kernel -s 3 -c 1 -o gpurun_out/ea_full -f python tools/bench_ea.py --once > gpurun_out/ea_ncu.log 2>&1; tail -3 gpurun_out/ea_ncu.log
