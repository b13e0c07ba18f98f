export DD_SERIAL_TIERS=1
timeout 1700 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:k1_cell -o gpurun_out/k1_full_r01c -f python tools/profile_sweep.py --cfg 5 --profile-last --quiet > gpurun_out/ncu_full_r01c.log 2>&1; echo ncu rc=$?
