cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "two_stage or global_tile or cfg5" --durations=10 > gpurun_out/r2_pytest3a.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2_pytest3a.log
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2_bench3.json 2> gpurun_out/r2_bench3.err
echo "bench rc=$?" >> gpurun_out/r2_bench3.err
