mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -2 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/bench.log 2>&1; echo bench rc=$?
python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/plain30.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r01c.csv python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch_c.log 2>&1; echo launch rc=$?
timeout 300 python tools/profile_sweep.py --cfg 5 --quiet --json gpurun_out/sweeps_r01c.json --cells-npz gpurun_out/cells_r01c.npz > gpurun_out/sweeps_r01c.log 2>&1; echo sweeps rc=$?
timeout 300 python tools/phase_profile.py --cfg 5 --min-side 512 > gpurun_out/phase_r01c.log 2>&1; echo phase rc=$?
