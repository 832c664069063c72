# Scratch job for one gpurun call (rewritten per call; the outputs land in gpurun_out/).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
B="timeout 400 python bench.py --no-e2e --no-cpu-baseline"
$B > gpurun_out/s5k_cfg5_ld2.json 2> gpurun_out/s5k_cfg5_ld2.err
BKFAC_LIB=$PWD/paper_2210_08494_b200/libbkfac_ld0.so $B > gpurun_out/s5k_cfg5_ld0.json 2> gpurun_out/s5k_cfg5_ld0.err
$B > gpurun_out/s5k_cfg5_ld2_b.json 2> gpurun_out/s5k_cfg5_ld2_b.err
BKFAC_LIB=$PWD/paper_2210_08494_b200/libbkfac_ld0.so $B > gpurun_out/s5k_cfg5_ld0_b.json 2> gpurun_out/s5k_cfg5_ld0_b.err
timeout 600 python -m pytest tests/test_gpu_gemm.py -m gpu -q -x > gpurun_out/s5k_gemmtests.log 2>&1
echo "tests rc=$?" >> gpurun_out/s5k_gemmtests.log
