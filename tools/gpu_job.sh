# Scratch job for one gpurun call (rewritten per call; the outputs land in gpurun_out/).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python tools/prec_block_error.py 16384 4097 512 512 4 8 16 32 > gpurun_out/s5v_prec_block_error_cfg5a.json 2> gpurun_out/s5v_prec_block_error_cfg5a.err
timeout 900 python tools/prec_block_error.py 4096 16385 512 512 4 8 16 32 > gpurun_out/s5v_prec_block_error_cfg5b.json 2> gpurun_out/s5v_prec_block_error_cfg5b.err
