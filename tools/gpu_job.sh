# Scratch job for one gpurun call (rewritten per call; the outputs land in gpurun_out/).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
BKFAC_LIB=paper_2210_08494_b200/libbkfac_ctime.so timeout 600 python tools/chase_timing.py > gpurun_out/s4ar_ctime.log 2>&1
