mkdir -p gpurun_out
python tools/profile_sweep.py --cfg 5 --quiet > /dev/null 2>&1; echo plain rc=$?
DD_SERIAL_TIERS=1 timeout 1500 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:k1_cell -c 3 -o gpurun_out/r02_k1_full python tools/profile_sweep.py --cfg 5 --profile-last --quiet > gpurun_out/ncu_full.log 2>&1; echo ncu rc=$?
tail -3 gpurun_out/ncu_full.log
