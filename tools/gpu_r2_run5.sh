cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "two_stage or cfg5_factor_chain_20_steps[4097]" > gpurun_out/r2_pytest5a.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2_pytest5a.log
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2_bench5.json 2> gpurun_out/r2_bench5.err
echo "bench rc=$?" >> gpurun_out/r2_bench5.err
