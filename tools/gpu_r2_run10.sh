cd $GRAFT_REPO_ROOT
for v in libbkfac.so libbkfac_s16.so libbkfac_s16n16.so; do
  BKFAC_LIB=$PWD/paper_2210_08494_b200/$v timeout 600 python bench.py --steps 6 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2_b10_cfg5_$v.json 2>&1
  BKFAC_LIB=$PWD/paper_2210_08494_b200/$v timeout 600 python bench.py --config cfg4 --steps 25 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r2_b10_cfg4_$v.json 2>&1
done
