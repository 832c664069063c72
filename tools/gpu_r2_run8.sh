cd $GRAFT_REPO_ROOT
for v in libbkfac.so libbkfac_epi8.so libbkfac_n32.so libbkfac_n32e8.so; do
  BKFAC_LIB=$PWD/paper_2210_08494_b200/$v timeout 300 python tools/gemm_variants.py >> gpurun_out/r2_gemm_variants.jsonl 2>&1
done
timeout 600 python bench.py --steps 6 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2_bench8.json 2> gpurun_out/r2_bench8.err
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2_pytest8.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2_pytest8.log
python tools/prof_cfg5.py --blocks 4 > gpurun_out/r2_prof_plain.log 2>&1 && \
ncu --set full --import-source on --nvtx --nvtx-include "brand/" -k regex:"sbr_chase|sbr_q2" -c 2 -o gpurun_out/r2_chase python tools/prof_cfg5.py --blocks 4 > gpurun_out/r2_ncu_chase.log 2>&1
