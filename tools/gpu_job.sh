# Scratch job for one gpurun call (rewritten per call; the outputs land in gpurun_out/).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/s5j_cfg5.json 2> gpurun_out/s5j_cfg5.err
timeout 600 python bench.py --impl reference > gpurun_out/s5j_reference.json 2> gpurun_out/s5j_reference.err
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/s5j_smoke.log 2>&1
