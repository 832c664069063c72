#!/bin/bash
# quick GPU check: parity suite + cfg4 bench (no cpu baseline / e2e) [+ cfg5 if QUICK_CFG5=1]
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "exit $?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_cfg4.log 2>&1; echo "exit $?" >> gpurun_out/bench_cfg4.log
tail -2 gpurun_out/bench_cfg4.log | cut -c1-600
if [ "$QUICK_CFG5" = 1 ]; then
timeout 900 python bench.py --config cfg5 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_cfg5.log 2>&1; echo "exit $?" >> gpurun_out/bench_cfg5.log
tail -2 gpurun_out/bench_cfg5.log | cut -c1-400
fi
echo done
