cd "$GRAFT_REPO_ROOT"
BKFAC_LIB=paper_2210_08494_b200/libbkfac_epi8.so timeout 600 python -m pytest tests/test_gpu_gemm.py -x -q 2>&1 | tail -1
for lib in libbkfac.so libbkfac_epi8.so; do echo "== $lib"; BKFAC_LIB=paper_2210_08494_b200/$lib python tools/bench_ea.py 2>&1 | head -2; BKFAC_LIB=paper_2210_08494_b200/$lib python tools/bench_gemm.py --tc-only 2>&1 | cut -c1-150; done
