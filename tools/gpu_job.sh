# Scratch job for one gpurun call (rewritten per call; the outputs land in gpurun_out/).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/s2f_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/s2f_pytest.log
