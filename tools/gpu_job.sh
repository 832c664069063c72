# Scratch job for one gpurun call (rewritten per call; the outputs land in gpurun_out/).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/s5m_gputests.log 2>&1
echo "tests rc=$?" >> gpurun_out/s5m_gputests.log
timeout 600 python bench.py > gpurun_out/s5m_cfg5.json 2> gpurun_out/s5m_cfg5.err
for C in cfg1 cfg2 cfg3 cfg4; do
  timeout 300 python bench.py --config $C > gpurun_out/s5m_$C.json 2> gpurun_out/s5m_$C.err
done
timeout 300 python bench.py --config cfg4 --full-rank --no-e2e --no-cpu-baseline > gpurun_out/s5m_cfg4_f1.json 2> gpurun_out/s5m_cfg4_f1.err
timeout 300 python bench.py --config cfg4 --factored --no-e2e --no-cpu-baseline > gpurun_out/s5m_cfg4_f2.json 2> gpurun_out/s5m_cfg4_f2.err
timeout 300 python bench.py --config cfg4 --correct-every 5 --no-e2e --no-cpu-baseline > gpurun_out/s5m_cfg4_f3.json 2> gpurun_out/s5m_cfg4_f3.err
timeout 600 python bench.py > gpurun_out/s5m_cfg5_b.json 2> gpurun_out/s5m_cfg5_b.err
