#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "exit $?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "exit $?" >> gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench_cfg4.log 2>&1; echo "exit $?" >> gpurun_out/bench_cfg4.log
timeout 900 python bench.py --config cfg5 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_cfg5.log 2>&1; echo "exit $?" >> gpurun_out/bench_cfg5.log
timeout 120 python tools/prof_gemm.py prec_out > gpurun_out/prof_plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_tc -s 2 -c 1 -o gpurun_out/prof_gemm_precout python tools/prof_gemm.py prec_out > gpurun_out/ncu_full.log 2>&1
echo done
