# HEAD verification after the bulk-copy staging: smoke, full GPU suite, default bench (cpu_baseline + e2e), launch list
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_v9.log 2>&1; echo smoke rc=$?; tail -1 gpurun_out/smoke_v9.log
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_v9.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/pytest_v9.log
timeout 900 python bench.py > gpurun_out/bench_v9.log 2>&1; echo bench rc=$?
tail -1 gpurun_out/bench_v9.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['frac'], d['finest_sweep']['ms'], d['time_to_solution_ms'], d['e2e']['value'])"
