# Scratch job for one gpurun call (rewritten per call; the outputs land in gpurun_out/).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q --durations=15 > gpurun_out/s4p_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/s4p_pytest.log
timeout 900 python bench.py > gpurun_out/s4p_bench.json 2> gpurun_out/s4p_bench.err
echo "bench rc=$?" >> gpurun_out/s4p_bench.err
timeout 600 python tools/prof_cfg5.py > gpurun_out/s4p_prof_plain.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"sbr_x_kernel|sbr_update_kernel" -s 200 -c 2 -o gpurun_out/s4p_sbr python tools/prof_cfg5.py > gpurun_out/s4p_ncu.log 2>&1
echo "ncu rc=$?" >> gpurun_out/s4p_ncu.log
