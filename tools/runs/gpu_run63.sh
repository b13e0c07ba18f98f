mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -2 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_r01h.log 2>&1; echo bench rc=$?
tail -1 gpurun_out/bench_r01h.log
timeout 900 python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/bench_ref_r01h.log 2>&1; echo ref rc=$?
python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/plain63.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r01h.csv python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch_e.log 2>&1; echo launch rc=$?
DD_SERIAL_TIERS=1 timeout 1200 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --profile-from-start off -k regex:k1_cell --csv --log-file gpurun_out/k1_traffic_r01h.csv python tools/profile_sweep.py --cfg 5 --profile-last --quiet > gpurun_out/ncu_traffic_e.log 2>&1; echo traffic rc=$?
timeout 300 python tools/profile_sweep.py --cfg 5 --quiet --json gpurun_out/sweeps_r01h.json > gpurun_out/sweeps_r01h.log 2>&1; echo sweeps rc=$?
timeout 300 python tools/phase_profile.py --cfg 5 --min-side 512 > gpurun_out/phase_r01h.log 2>&1; echo phase rc=$?
