# general costs / s=16 on the SMEM tier: new GPU tests, full suite, bench
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_general_cost.py -m gpu -x -q -rs --durations=8 > gpurun_out/pytest_gc.log 2>&1; echo gc rc=$?
tail -30 gpurun_out/pytest_gc.log
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_v3.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_v3.log
timeout 900 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_v3.log 2>&1; echo bench rc=$?
tail -1 gpurun_out/bench_v3.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['frac'], d['finest_sweep']['ms'], d['time_to_solution_ms'])"
