# Scratch job for one gpurun call (rewritten per call; the outputs land in gpurun_out/).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "not cfg5_factor_chain and not cfg4_stack and not cfg5_block and not cfg2_chain" > gpurun_out/s4am_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/s4am_pytest.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/s4am_base.json 2> gpurun_out/s4am_base.err
