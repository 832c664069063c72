# Scratch job for one gpurun call (rewritten per call; the outputs land in gpurun_out/).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --nvtx --nvtx-include "brand/" --nvtx-include "prec/" --csv --log-file gpurun_out/s5w_launches.csv python tools/prof_cfg5.py > gpurun_out/s5w_ncu1.log 2>&1
echo "rc=$?" >> gpurun_out/s5w_ncu1.log
timeout 1200 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "gemm_prec_out/" --nvtx-include "gemm_prec_proj/" -k regex:gemm_tc -c 3 -o gpurun_out/s5w_prec python tools/prof_cfg5.py --stage-nvtx > gpurun_out/s5w_ncu2.log 2>&1
echo "rc=$?" >> gpurun_out/s5w_ncu2.log
python tools/ncu_full_summary.py gpurun_out/s5w_prec_summary.txt "ncu --set full --clock-control none, configs[4] preconditioner GEMMs (prec_proj x2, prec_out; all 48 layers per launch), session 5 final build, default options (256-term TMEM blocks)" gpurun_out/s5w_prec.ncu-rep >> gpurun_out/s5w_ncu2.log 2>&1
