cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
for m in 0 2; do echo "== pair $m"; BKFAC_GEMM_PAIR=$m timeout 300 python tools/bench_gemm.py --tc-only 2>&1 | cut -c1-160; done
BKFAC_GEMM_PAIR=2 timeout 600 python -m pytest tests/test_gpu_gemm.py -x -q 2>&1 | tail -1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -1 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_cfg4.log 2>&1; tail -1 gpurun_out/bench_cfg4.log | cut -c1-300
timeout 900 python bench.py --config cfg5 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_cfg5.log 2>&1; tail -1 gpurun_out/bench_cfg5.log | cut -c1-300
