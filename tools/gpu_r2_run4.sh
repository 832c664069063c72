cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "cholesky_large or two_stage" > gpurun_out/r2_pytest4a.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2_pytest4a.log
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2_bench4.json 2> gpurun_out/r2_bench4.err
echo "bench rc=$?" >> gpurun_out/r2_bench4.err
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2_pytest4b.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2_pytest4b.log
