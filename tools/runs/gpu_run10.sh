mkdir -p gpurun_out
timeout 300 python tools/profile_sweep.py --cfg 4 --profile-last --quiet > gpurun_out/plain10.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:k1_cell -o gpurun_out/k1_full_cfg4_v5 -f python tools/profile_sweep.py --cfg 4 --profile-last --quiet > gpurun_out/ncu_cfg4_v5.log 2>&1; echo ncu rc=$?
tail -2 gpurun_out/ncu_cfg4_v5.log
