#!/bin/bash
# build GEMM tuning variants of libbkfac.so (in-tree, git-ignored): name:defines
cd "$(dirname "$0")/.."
for v in "$@"; do
  name=${v%%:*}; defs=${v#*:}
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared \
    -Iinclude $defs -o paper_2210_08494_b200/libbkfac_$name.so paper_2210_08494_b200/csrc/bkfac_api.cu -Xptxas -v 2>&1 \
    | grep -A2 "gemm_tc_kernel" | grep -E "registers|spill" | head -2 | sed "s/^/$name: /"
done
