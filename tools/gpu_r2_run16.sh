cd $GRAFT_REPO_ROOT
BKFAC_LIB=$PWD/paper_2210_08494_b200/libbkfac_q2t.so timeout 300 python tools/chase_timing.py q2 > gpurun_out/r2_q2_timing.log 2>&1
