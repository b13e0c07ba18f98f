mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "big or single_sweep or trajectory" > gpurun_out/pytest_big.log 2>&1; echo big rc=$?
tail -5 gpurun_out/pytest_big.log
timeout 300 python tools/profile_sweep.py --cfg 5 --json gpurun_out/sweeps_cfg5_v4.json > gpurun_out/sweeps_cfg5_v4.log 2>&1; echo sweeps rc=$?
tail -2 gpurun_out/sweeps_cfg5_v4.log | cut -c1-700
