# ncu --set full of selected kernels in the cfg4 bench (one GPU); KREGEX, KCOUNT, KSKIP, OUT
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 3 --warmup 3 > gpurun_out/prof_plain.log 2>&1 || { echo "plain run failed"; tail -5 gpurun_out/prof_plain.log; exit 1; }
timeout 900 ncu --set full --import-source on --clock-control none -k "regex:${KREGEX}" -s ${KSKIP:-6} -c ${KCOUNT:-3} -o gpurun_out/${OUT:-kfull} -f \
  python bench.py --no-cpu-baseline --no-e2e --steps 3 --warmup 3 > gpurun_out/prof_ncu.log 2>&1; tail -2 gpurun_out/prof_ncu.log
