# Scratch job for one gpurun call (rewritten per call; the outputs land in gpurun_out/).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/s2c_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/s2c_pytest.log
timeout 900 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/s2c_bench.json 2> gpurun_out/s2c_bench.err
echo "bench rc=$?" >> gpurun_out/s2c_bench.err
