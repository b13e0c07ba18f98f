mkdir -p gpurun_out
python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/plain23.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r01b.csv python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch_b.log 2>&1; echo launch rc=$?
timeout 300 python tools/profile_sweep.py --cfg 5 --profile-last --quiet > gpurun_out/plain23b.log 2>&1 && \
timeout 1500 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__inst_executed_pipe_xu.sum,smsp__inst_executed.sum --clock-control none --profile-from-start off -k regex:k1_cell --csv --log-file gpurun_out/k1_traffic_r01b.csv python tools/profile_sweep.py --cfg 5 --profile-last --quiet > gpurun_out/ncu_traffic.log 2>&1; echo traffic rc=$?
timeout 300 python tools/phase_profile.py --cfg 5 --min-side 256 > gpurun_out/phase_r01b.log 2>&1; echo phase rc=$?
timeout 300 python tools/profile_sweep.py --cfg 5 --quiet --json gpurun_out/sweeps_r01b.json --cells-npz gpurun_out/cells_r01b.npz > gpurun_out/sweeps_r01b.log 2>&1; echo sweeps rc=$?
