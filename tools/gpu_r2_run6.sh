cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "two_stage or chain_20" > gpurun_out/r2_pytest6a.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2_pytest6a.log
timeout 600 python bench.py --steps 6 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2_bench6.json 2> gpurun_out/r2_bench6.err
BKFAC_LIB=$PWD/paper_2210_08494_b200/libbkfac_spin.so timeout 600 python bench.py --steps 6 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2_bench6_spin.json 2> gpurun_out/r2_bench6_spin.err
