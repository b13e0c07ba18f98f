mkdir -p gpurun_out
for b in 18 24 32; do
timeout 300 python tools/profile_sweep.py --cfg 5 --quiet --bcap $b --json gpurun_out/sweeps_cfg5_b$b.json > gpurun_out/cells_b$b.log 2>&1; echo b=$b rc=$?
tail -1 gpurun_out/cells_b$b.log | cut -c1-60
done
timeout 300 python tools/phase_profile.py --cfg 5 --min-side 2048 > gpurun_out/phase_b.log 2>&1
