# Scratch job for one gpurun call (rewritten per call; the outputs land in gpurun_out/).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python tools/prof_cfg5.py > gpurun_out/s4aa_plain.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"sbr_panel_kernel|sbr_chase_kernel" -s 96 -c 2 -o gpurun_out/s4aa_lat python tools/prof_cfg5.py > gpurun_out/s4aa_ncu.log 2>&1
echo "rc=$?" >> gpurun_out/s4aa_ncu.log
