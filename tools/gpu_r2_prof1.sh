cd $GRAFT_REPO_ROOT
python tools/prof_cfg5.py --blocks 4 > gpurun_out/r2_prof_plain.log 2>&1 && \
ncu --set full --import-source on --nvtx --nvtx-include "brand/" -k regex:"sbr_chase|sbr_q2|sbr_panel|sbr_w" -c 4 -o gpurun_out/r2_sbr python tools/prof_cfg5.py --blocks 4 > gpurun_out/r2_ncu_sbr.log 2>&1
ncu --set full --import-source on --nvtx --nvtx-include "prec/" -k regex:gemm_tc -c 5 -o gpurun_out/r2_prec python tools/prof_cfg5.py --blocks 4 > gpurun_out/r2_ncu_prec.log 2>&1
ncu --set full --import-source on --nvtx --nvtx-include "brand/" -k regex:gemm_tc -s 9 -c 3 -o gpurun_out/r2_brandgemm python tools/prof_cfg5.py --blocks 4 > gpurun_out/r2_ncu_brandgemm.log 2>&1
BKFAC_LIB=$PWD/paper_2210_08494_b200/libbkfac_epi8.so timeout 600 python bench.py --steps 6 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2_bench7_epi8.json 2> gpurun_out/r2_bench7_epi8.err
