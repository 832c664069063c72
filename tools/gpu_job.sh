# Scratch job for one gpurun call (rewritten per call; the outputs land in gpurun_out/).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_pipeline.py -q > gpurun_out/s5_pipe_tests3.log 2>&1
echo "tests rc=$?" >> gpurun_out/s5_pipe_tests3.log
for P in 36 40 44; do
  timeout 300 python bench.py --config cfg5r2 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --pipeline $P > gpurun_out/s5_r2_$P.json 2> gpurun_out/s5_r2_$P.err
done
for P in 36 40 48; do
  timeout 300 python bench.py --config cfg5r4 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --pipeline $P > gpurun_out/s5_r4_$P.json 2> gpurun_out/s5_r4_$P.err
done
for P in 36 44 48; do
  timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --pipeline $P > gpurun_out/s5_cfg5_$P.json 2> gpurun_out/s5_cfg5_$P.err
done
for C in cfg3 cfg4; do for P in 0 44; do
  timeout 300 python bench.py --config $C --steps 25 --warmup 5 --no-e2e --no-cpu-baseline --pipeline $P > gpurun_out/s5_${C}_$P.json 2> gpurun_out/s5_${C}_$P.err
done; done
