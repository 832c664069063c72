# Scratch job for one gpurun call (rewritten per call; the outputs land in gpurun_out/).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/s4f2_smi.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q --durations=10 > gpurun_out/s4f2_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/s4f2_pytest.log
timeout 900 python bench.py > gpurun_out/s4f2_bench.json 2> gpurun_out/s4f2_bench.err
echo "bench rc=$?" >> gpurun_out/s4f2_bench.err
timeout 600 python tools/prof_cfg5.py > gpurun_out/s4f2_prof_plain.log 2>&1 && \
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --nvtx --nvtx-include "brand/" --nvtx-include "prec/" --csv --log-file gpurun_out/s4f2_launches.csv python tools/prof_cfg5.py > gpurun_out/s4f2_ncu.log 2>&1
echo "ncu rc=$?" >> gpurun_out/s4f2_ncu.log
