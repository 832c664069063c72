cd $GRAFT_REPO_ROOT
BKFAC_LIB=$PWD/paper_2210_08494_b200/libbkfac_chaset.so timeout 300 python tools/chase_timing.py > gpurun_out/r2_chase_timing3.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "two_stage or rank_share" > gpurun_out/r2_pytest18.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2_pytest18.log
timeout 600 python bench.py --steps 6 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2_b18_cfg5.json 2>&1
python tools/prof_cfg5.py --blocks 24 > gpurun_out/r2_prof_plain2.log 2>&1 && \
ncu --set full --import-source on --nvtx --nvtx-include "brand/" --kernel-name-base demangled -k "regex:gemm_tc_kernel<.bool.0, .bool.1, .int.128, .int.16, .int.1, .int.8, .bool.0>" -c 6 -o gpurun_out/r2_upd python tools/prof_cfg5.py --blocks 24 > gpurun_out/r2_ncu_upd.log 2>&1
