# Scratch job for one gpurun call (rewritten per call; the outputs land in gpurun_out/).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python tools/prof_cfg5.py --stage-nvtx > gpurun_out/s4ae_plain.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "gemm_gram/" -k regex:gemm_tc -c 1 -o gpurun_out/s4ae_gram python tools/prof_cfg5.py --stage-nvtx > gpurun_out/s4ae_ncu.log 2>&1
echo "rc=$?" >> gpurun_out/s4ae_ncu.log
