# X side staged by the bulk-copy engine (cp.async.bulk + mbarrier): smoke, parity, full suite, bench
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_v8.log 2>&1; echo smoke rc=$?; tail -1 gpurun_out/smoke_v8.log
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x > gpurun_out/pytest_v8a.log 2>&1; echo parity rc=$?; tail -1 gpurun_out/pytest_v8a.log
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_v8.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/pytest_v8.log
timeout 900 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_v8.log 2>&1; echo bench rc=$?
tail -1 gpurun_out/bench_v8.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['frac'], d['finest_sweep']['ms'], d['time_to_solution_ms'])"
