mkdir -p gpurun_out
timeout 300 python tools/profile_sweep.py --cfg 5 --quiet --cells-npz gpurun_out/cells_cfg5.npz > gpurun_out/cells_cfg5.log 2>&1; echo cells rc=$?
timeout 900 python tools/box_stats.py --cfg 5 --min-side 512 > gpurun_out/box_stats_cfg5.log 2>&1; echo box rc=$?
tail -3 gpurun_out/box_stats_cfg5.log | cut -c1-2000
