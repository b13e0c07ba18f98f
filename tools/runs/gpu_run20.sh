mkdir -p gpurun_out
timeout 300 python tools/profile_sweep.py --cfg 5 --quiet --json gpurun_out/sweeps_cfg5_v8.json --cells-npz gpurun_out/cells_cfg5_v8.npz > gpurun_out/cells_v8.log 2>&1; echo rc=$?
tail -1 gpurun_out/cells_v8.log | cut -c1-80
