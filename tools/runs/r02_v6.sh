mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_tier_g_gpu.py -m gpu -q > gpurun_out/pytest_tg6.log 2>&1; echo tg rc=$?; tail -1 gpurun_out/pytest_tg6.log
bash tools/ab_test.sh P2 P4
timeout 900 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_v6.log 2>&1; echo bench rc=$?
tail -1 gpurun_out/bench_v6.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['frac'], d['finest_sweep']['ms'], d['time_to_solution_ms'])"
