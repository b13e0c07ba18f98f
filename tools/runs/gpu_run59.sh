export DD_SERIAL_TIERS=1
timeout 1200 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:k1_cell --launch-skip 1 --launch-count 1 -o gpurun_out/k1_t1_r01g -f python tools/profile_sweep.py --cfg 5 --profile-last --quiet > gpurun_out/ncu_t1.log 2>&1; echo ncu1 rc=$?
timeout 1200 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:k1_cell --launch-count 1 -o gpurun_out/k1_t2_r01g -f python tools/profile_sweep.py --cfg 5 --profile-last --quiet > gpurun_out/ncu_t2.log 2>&1; echo ncu2 rc=$?
