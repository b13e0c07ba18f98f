# tier-0 lse_pass with compile-time G and warp-uniform modes: parity + bench A/B
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_v2.log 2>&1; echo smoke rc=$?
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_v2.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_v2.log
timeout 900 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_v2.log 2>&1; echo bench rc=$?
tail -1 gpurun_out/bench_v2.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['frac'], d['finest_sweep']['ms'], d['time_to_solution_ms'])"
