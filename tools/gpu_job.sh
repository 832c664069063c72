# Scratch job for one gpurun call (rewritten per call; the outputs land in gpurun_out/).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for C in cfg5r2 cfg5r4 cfg5r8; do
  timeout 300 python bench.py --config $C --no-e2e --no-cpu-baseline > gpurun_out/s5u_$C.json 2> gpurun_out/s5u_$C.err
done
timeout 300 python bench.py --config cfg1 > gpurun_out/s5u_cfg1.json 2> gpurun_out/s5u_cfg1.err
timeout 300 python bench.py --config cfg2 > gpurun_out/s5u_cfg2.json 2> gpurun_out/s5u_cfg2.err
