cd $GRAFT_REPO_ROOT
BKFAC_LIB=$PWD/paper_2210_08494_b200/libbkfac_q2t.so timeout 300 python tools/chase_timing.py q2 > gpurun_out/r2_q2_timing2.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "two_stage or rank_share or chain_20_steps" > gpurun_out/r2_pytest17.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2_pytest17.log
timeout 600 python bench.py --steps 6 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2_b17_cfg5.json 2>&1
for c in cfg5r2 cfg5r4 cfg5r8; do
  for o in 1 2; do
    timeout 600 python bench.py --config $c --steps 6 --warmup 3 --no-cpu-baseline --no-e2e --opt TWO_STAGE=$o > gpurun_out/r2_b17_${c}_ts$o.json 2>&1
  done
done
