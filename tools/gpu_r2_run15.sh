cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "two_stage or rank_share or block_stack" > gpurun_out/r2_pytest15.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2_pytest15.log
timeout 600 python bench.py --config cfg5r8 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2_bench15_r8.json 2>&1
timeout 600 python bench.py --config cfg5r8 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --opt TWO_STAGE=1 > gpurun_out/r2_bench15_r8_one.json 2>&1
timeout 600 python bench.py --steps 6 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2_bench15.json 2>&1
