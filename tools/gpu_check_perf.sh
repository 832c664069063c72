cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; tail -1 gpurun_out/pytest_gpu.log
python tools/bench_ea.py 2>&1 | head -3
timeout 300 python tools/bench_gemm.py --tc-only 2>&1 | cut -c1-150
timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_cfg4.log 2>&1; tail -1 gpurun_out/bench_cfg4.log | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print(d['ms_per_step'], [(s['stage'], round(s['ms']/d['steps'],3)) for s in d['stages'][:12]])"
if [ "$CFG5" = 1 ]; then timeout 900 python bench.py --config cfg5 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_cfg5.log 2>&1; tail -1 gpurun_out/bench_cfg5.log | cut -c1-250; fi
