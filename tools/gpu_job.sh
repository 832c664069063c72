# Scratch job for one gpurun call (rewritten per call; the outputs land in gpurun_out/).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/s5f_cfg5.json 2> gpurun_out/s5f_cfg5.err
for C in cfg5r2 cfg5r4 cfg5r8; do
  timeout 300 python bench.py --config $C --no-e2e --no-cpu-baseline > gpurun_out/s5f_$C.json 2> gpurun_out/s5f_$C.err
  timeout 300 python bench.py --config $C --no-e2e --no-cpu-baseline --pipeline 0 > gpurun_out/s5f_${C}_nopipe.json 2> gpurun_out/s5f_${C}_nopipe.err
done
for C in cfg3 cfg4; do
  timeout 300 python bench.py --config $C > gpurun_out/s5f_$C.json 2> gpurun_out/s5f_$C.err
done
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/s5f_gputests.log 2>&1
echo "tests rc=$?" >> gpurun_out/s5f_gputests.log
