mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "big" > gpurun_out/pytest_big.log 2>&1; echo big rc=$?
tail -15 gpurun_out/pytest_big.log
timeout 300 python tools/profile_sweep.py --cfg 5 --json gpurun_out/sweeps_cfg5_v3.json > gpurun_out/sweeps_cfg5_v3.log 2>&1; echo sweeps rc=$?
tail -4 gpurun_out/sweeps_cfg5_v3.log | cut -c1-600
