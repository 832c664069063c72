# Scratch job for one gpurun call (rewritten per call; the outputs land in gpurun_out/).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
B="timeout 400 python bench.py --no-e2e --no-cpu-baseline"
$B > gpurun_out/s5g_cfg5_wholeK.json 2> gpurun_out/s5g_cfg5_wholeK.err
$B --opt prec_block=8 > gpurun_out/s5g_cfg5_pb8.json 2> gpurun_out/s5g_cfg5_pb8.err
$B --opt prec_block=16 > gpurun_out/s5g_cfg5_pb16.json 2> gpurun_out/s5g_cfg5_pb16.err
$B > gpurun_out/s5g_cfg5_wholeK_b.json 2> gpurun_out/s5g_cfg5_wholeK_b.err
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/s5g_gputests.log 2>&1
echo "tests rc=$?" >> gpurun_out/s5g_gputests.log
