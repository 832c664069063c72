# Scratch job for one gpurun call (rewritten per call; the outputs land in gpurun_out/).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for v in pt1024 pt256; do
  lib=paper_2210_08494_b200/libbkfac_$v.so
  BKFAC_LIB=$lib timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/s4z_$v.json 2> gpurun_out/s4z_$v.err
done
