#!/bin/bash
# bench lines of the NEXT rows at cfg4 (f1 full rank, f2 factored, f3 light correction)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 600 python bench.py --full-rank --no-cpu-baseline > gpurun_out/bench_f1.json 2> gpurun_out/bench_f1.err; echo "f1 $?"
timeout 600 python bench.py --factored --no-cpu-baseline > gpurun_out/bench_f2.json 2> gpurun_out/bench_f2.err; echo "f2 $?"
timeout 600 python bench.py --correct-every 5 --no-cpu-baseline > gpurun_out/bench_f3.json 2> gpurun_out/bench_f3.err; echo "f3 $?"
