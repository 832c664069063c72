# Scratch job for one gpurun call (rewritten per call; the outputs land in gpurun_out/).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q --durations=10 > gpurun_out/s4z_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/s4z_pytest.log
timeout 900 python bench.py > gpurun_out/s4z_bench.json 2> gpurun_out/s4z_bench.err
echo "bench rc=$?" >> gpurun_out/s4z_bench.err
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/s4z_smoke.log 2>&1
