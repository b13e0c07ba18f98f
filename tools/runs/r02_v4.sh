mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_general_cost.py tests/test_safeguard.py -m gpu -q -rs --durations=10 > gpurun_out/pytest_gc4.log 2>&1; echo gc rc=$?
tail -30 gpurun_out/pytest_gc4.log
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_v4.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_v4.log
timeout 900 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_v4.log 2>&1; echo bench rc=$?
tail -1 gpurun_out/bench_v4.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['frac'], d['finest_sweep']['ms'], d['time_to_solution_ms'])"
