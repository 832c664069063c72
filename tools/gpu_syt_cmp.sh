#!/bin/bash
# sytrd A/B: stage times for the current library vs libbkfac_$1.so on cfg4-shaped cores
cd "$GRAFT_REPO_ROOT"
for lib in libbkfac.so libbkfac_$1.so; do
  echo "== $lib"
  BKFAC_LIB=$PWD/paper_2210_08494_b200/$lib python tools/prof_sytrd.py 577 256 220 23 time 2>&1 | grep -E "eig|chol|Error|error" | head -9
  BKFAC_LIB=$PWD/paper_2210_08494_b200/$lib python tools/prof_sytrd.py 1600 1024 512 4 time 2>&1 | grep -E "eig_sytrd|Error|error" | head -3
done
