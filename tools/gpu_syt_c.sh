#!/bin/bash
# sytrd cluster-width sweep on cfg4-shaped cores (23 x m=476)
cd "$GRAFT_REPO_ROOT"
for c in 0 5 6 8; do
  echo "== BKFAC_SYT_C=$c"
  BKFAC_SYT_C=$c python tools/prof_sytrd.py 577 256 220 23 time 2>&1 | grep -E "eig_sytrd|rror" | head -3
done
