# Scratch job for one gpurun call (rewritten per call; the outputs land in gpurun_out/).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/s5t_cfg5.json 2> gpurun_out/s5t_cfg5.err
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/s5t_gputests.log 2>&1
echo "tests rc=$?" >> gpurun_out/s5t_gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/s5t_smoke.log 2>&1
timeout 600 python tools/prec_block_error.py > gpurun_out/s5t_prec_block_error.json 2> gpurun_out/s5t_prec_block_error.err
for C in cfg3 cfg4; do timeout 300 python bench.py --config $C > gpurun_out/s5t_$C.json 2> gpurun_out/s5t_$C.err; done
