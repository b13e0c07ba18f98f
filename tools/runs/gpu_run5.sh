mkdir -p gpurun_out
timeout 300 python tools/profile_sweep.py --cfg 5 --json gpurun_out/sweeps_cfg5_v3.json > gpurun_out/sweeps_cfg5_v3.log 2>&1; echo sweeps rc=$?
tail -2 gpurun_out/sweeps_cfg5_v3.log | cut -c1-700
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_gpu.log
