set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
timeout 2400 python -m pytest tests -m gpu -x -q -rs --durations=15 > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -25 gpurun_out/pytest_gpu.log
timeout 1200 python bench.py > gpurun_out/bench_v1.log 2>&1; echo bench rc=$?
tail -c 4000 gpurun_out/bench_v1.log
