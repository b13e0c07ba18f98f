mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_tier_g_gpu.py tests/test_general_cost.py -m gpu -q -rs --durations=6 > gpurun_out/pytest_tg.log 2>&1; echo tg rc=$?
tail -15 gpurun_out/pytest_tg.log
timeout 900 python -m pytest tests/test_cluster_gpu.py tests/test_gpu_parity.py tests/test_striped_gpu.py tests/test_batch_gpu.py -m gpu -q -x > gpurun_out/pytest_v5.log 2>&1; echo core rc=$?
tail -3 gpurun_out/pytest_v5.log
timeout 900 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_v5.log 2>&1; echo bench rc=$?
tail -1 gpurun_out/bench_v5.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['frac'], d['finest_sweep']['ms'], d['time_to_solution_ms'])"
