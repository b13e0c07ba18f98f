# HEAD check in the driver's order: smoke, the GPU suite (-x), the default bench line
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_h.log 2>&1; echo smoke rc=$?
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_h.log 2>&1; echo pytest rc=$?
tail -2 gpurun_out/pytest_h.log
timeout 900 python bench.py > gpurun_out/bench_h.log 2>&1; echo bench rc=$?
tail -1 gpurun_out/bench_h.log | cut -c1-200
