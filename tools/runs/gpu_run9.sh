mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "big" > gpurun_out/pytest_big.log 2>&1; echo big rc=$?
tail -3 gpurun_out/pytest_big.log
timeout 300 python tools/profile_sweep.py --cfg 5 --quiet --json gpurun_out/sweeps_cfg5_v5.json --cells-npz gpurun_out/cells_cfg5_v5.npz > gpurun_out/cells_v5.log 2>&1; echo cells rc=$?
tail -1 gpurun_out/cells_v5.log | cut -c1-300
