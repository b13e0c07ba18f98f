mkdir -p gpurun_out
timeout 300 python tools/profile_sweep.py --cfg 5 --json gpurun_out/sweeps_cfg5.json > gpurun_out/sweeps_cfg5.log 2>&1; echo sweeps rc=$?
tail -3 gpurun_out/sweeps_cfg5.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r01.csv python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo ncu1 rc=$?
timeout 1200 ncu --set full --clock-control none --import-source on --profile-from-start off -o gpurun_out/k1_full_r01 -f python tools/profile_sweep.py --cfg 5 --profile-last --quiet > gpurun_out/ncu_full.log 2>&1; echo ncu2 rc=$?
tail -5 gpurun_out/ncu_full.log
