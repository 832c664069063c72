# Scratch job for one gpurun call (rewritten per call; the outputs land in gpurun_out/).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x -k "not cfg5_factor_chain" > gpurun_out/s4ab_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/s4ab_pytest.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/s4ab_base.json 2> gpurun_out/s4ab_base.err
