cd $GRAFT_REPO_ROOT
BKFAC_LIB=$PWD/paper_2210_08494_b200/libbkfac_chaset.so timeout 300 python tools/chase_timing.py > gpurun_out/r2_chase_timing.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_gemm.py -x -q -k "two_stage or rank_share or gemm" > gpurun_out/r2_pytest9.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2_pytest9.log
timeout 600 python bench.py --steps 6 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2_bench9.json 2> gpurun_out/r2_bench9.err
