mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_striped_gpu.py -x -q > gpurun_out/pytest_striped.log 2>&1; echo striped rc=$?
tail -30 gpurun_out/pytest_striped.log
