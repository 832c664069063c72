# Scratch job for one gpurun call (rewritten per call; the outputs land in gpurun_out/).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for c in cfg5r8 cfg5r4 cfg5r2; do
  for t in 1 2; do
    timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --opt TWO_STAGE=$t > gpurun_out/s4u_${c}_t$t.json 2> gpurun_out/s4u_${c}_t$t.err
  done
done
