cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_gemm.py -x -q > gpurun_out/r2_pytest_gemm.log 2>&1
echo "pytest gemm rc=$?" >> gpurun_out/r2_pytest_gemm.log
timeout 1500 python -m pytest tests -m gpu -x -q --durations=5 > gpurun_out/r2_pytest2.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2_pytest2.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/r2_bench2.json 2> gpurun_out/r2_bench2.err
echo "bench rc=$?" >> gpurun_out/r2_bench2.err
