cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_gemm.py -x -q -k "two_stage or chain_20 or gemm or block_stack" > gpurun_out/r2_pytest12.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2_pytest12.log
timeout 600 python bench.py --steps 6 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2_bench12.json 2> gpurun_out/r2_bench12.err
timeout 600 python bench.py --config cfg4 --steps 25 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r2_bench12_cfg4.json 2>&1
timeout 600 python bench.py --config cfg4 --steps 25 --warmup 5 --no-cpu-baseline --no-e2e --opt TWO_STAGE=2 > gpurun_out/r2_bench12_cfg4_ts.json 2>&1
timeout 600 python tools/f4_protocol.py > gpurun_out/r2_f4.log 2>&1
