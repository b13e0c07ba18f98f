mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "big or trajectory or single" > gpurun_out/pytest_big.log 2>&1; echo big rc=$?
tail -3 gpurun_out/pytest_big.log
timeout 300 python tools/profile_sweep.py --cfg 5 --quiet --json gpurun_out/sweeps_cfg5_v6.json > gpurun_out/cells_v6.log 2>&1; echo sweeps rc=$?
tail -1 gpurun_out/cells_v6.log | cut -c1-150
timeout 300 python tools/phase_profile.py --cfg 5 --min-side 2048 > gpurun_out/phase_cfg5_v6.log 2>&1; echo phase rc=$?
cat gpurun_out/phase_cfg5_v6.log
