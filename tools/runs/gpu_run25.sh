mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_striped_gpu.py -x -q -k "big or trajectory or single or virtual" > gpurun_out/pytest_big.log 2>&1; echo tests rc=$?
tail -2 gpurun_out/pytest_big.log
timeout 300 python tools/profile_sweep.py --cfg 5 --quiet --json gpurun_out/sweeps_ri.json > gpurun_out/ri.log 2>&1; echo rc=$?
tail -1 gpurun_out/ri.log | cut -c1-330
