#!/bin/bash
# end-of-round refresh: GPU suite, smoke, cfg4/cfg5 bench lines, reference arm, launch list
# and targeted ncu captures (summaries written on the box; big reports deleted)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "exit $?" >> gpurun_out/pytest_gpu.log
tail -2 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_cfg4.json 2> gpurun_out/bench_cfg4.err; echo "cfg4 exit $?"
timeout 900 python bench.py --config cfg5 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg5.json 2> gpurun_out/bench_cfg5.err; echo "cfg5 exit $?"
timeout 900 python bench.py --config cfg5r8 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg5r8.json 2> gpurun_out/bench_cfg5r8.err; echo "cfg5r8 exit $?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref exit $?"
if [ "$SKIP_NCU" != 1 ]; then
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/launches_cfg4.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo "launch list exit $?"
bash tools/gpu_profile_kernels.sh
python tools/summarize_profiles.py gpurun_out/launches_cfg4.csv gpurun_out/prof_sytrd_tiled.ncu-rep r01 > gpurun_out/summ.log 2>&1
cp profiles/r01_launches_cfg4.txt profiles/traffic.json gpurun_out/ 2>/dev/null
rm -f gpurun_out/prof_sytrd_tiled.ncu-rep gpurun_out/launches_cfg4.csv
fi
du -sh gpurun_out
