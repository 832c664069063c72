#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out; : > gpurun_out/variants.log
for v in ${VARIANTS:-n16d1p4 noload onepass noload1p}; do
  echo "== $v" >> gpurun_out/variants.log
  BKFAC_LIB=paper_2210_08494_b200/libbkfac_$v.so timeout 300 python tools/bench_gemm.py --tc-only >> gpurun_out/variants.log 2>&1
done
