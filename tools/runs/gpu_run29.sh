timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "big" > gpurun_out/pytest_big.log 2>&1; echo big rc=$?; tail -1 gpurun_out/pytest_big.log
bash tools/gpu_run26.sh
