cd $GRAFT_REPO_ROOT
BKFAC_LIB=$PWD/paper_2210_08494_b200/libbkfac_chaset.so timeout 300 python tools/chase_timing.py > gpurun_out/r2_chase_timing2.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "two_stage or chain_20 or rank_share" > gpurun_out/r2_pytest11.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2_pytest11.log
timeout 600 python bench.py --steps 6 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2_bench11.json 2> gpurun_out/r2_bench11.err
timeout 300 python tools/sanitize_run.py > gpurun_out/r2_sanitize_plain.log 2>&1 && \
timeout 1200 compute-sanitizer --tool memcheck --print-limit 50 python tools/sanitize_run.py > gpurun_out/r2_memcheck.log 2>&1
echo "memcheck rc=$?" >> gpurun_out/r2_memcheck.log
