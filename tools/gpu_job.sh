# Scratch job for one gpurun call (rewritten per call; the outputs land in gpurun_out/).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
BKFAC_LIB=paper_2210_08494_b200/libbkfac_l2pf.so timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/s4ad_l2pf.json 2> gpurun_out/s4ad_l2pf.err
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/s4ad_base.json 2> gpurun_out/s4ad_base.err
