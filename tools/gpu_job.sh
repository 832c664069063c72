# Scratch job for one gpurun call (rewritten per call; the outputs land in gpurun_out/).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_parity.py -x -q -k "gemm or two_stage or leading or cfg5_factor_shape or ea_accumulate" > gpurun_out/s2i_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/s2i_pytest.log
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/s2i_bench.json 2> gpurun_out/s2i_bench.err
echo "bench rc=$?" >> gpurun_out/s2i_bench.err
