mkdir -p gpurun_out
for b in 64 120 200; do
timeout 300 python tools/profile_sweep.py --cfg 5 --quiet --bcap-big $b --json gpurun_out/sweeps_cfg5_bb$b.json --cells-npz gpurun_out/cells_bb$b.npz > gpurun_out/cells_bb$b.log 2>&1; echo bb=$b rc=$?
tail -1 gpurun_out/cells_bb$b.log | cut -c1-100
done
