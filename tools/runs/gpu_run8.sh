mkdir -p gpurun_out
timeout 300 python tools/profile_sweep.py --cfg 5 --quiet --cells-npz gpurun_out/cells_cfg5_v4.npz > gpurun_out/cells_v4.log 2>&1; echo cells rc=$?
timeout 300 python tools/profile_sweep.py --cfg 5 --profile-last --quiet > gpurun_out/plain8.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:k1_cell -o gpurun_out/k1_full_v4 -f python tools/profile_sweep.py --cfg 5 --profile-last --quiet > gpurun_out/ncu_full_v4.log 2>&1; echo ncu rc=$?
