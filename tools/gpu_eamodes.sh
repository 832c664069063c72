cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
for m in ${EA_MODES:-1 2}; do BKFAC_EA_MODE=$m timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_ea$m.log 2>&1; echo "mode $m"; tail -1 gpurun_out/bench_ea$m.log | cut -c1-260;
python - <<PY
import json
l=[x for x in open('gpurun_out/bench_ea$m.log') if x.startswith('{')][-1]
d=json.loads(l)
print([(s['stage'], round(s['ms']/d['steps'],3)) for s in sorted(d['stages'], key=lambda s:-s.get('ms',0))[:10]])
PY
done
