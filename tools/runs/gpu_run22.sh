mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "ladder or big_tier_parity_s8" > gpurun_out/pytest_glue.log 2>&1; echo tests rc=$?
tail -3 gpurun_out/pytest_glue.log
timeout 300 python tools/profile_sweep.py --cfg 5 --json gpurun_out/sweeps_cfg5_glue.json > gpurun_out/glue.log 2>&1; echo rc=$?
tail -1 gpurun_out/glue.log | cut -c1-400
