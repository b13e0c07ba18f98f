# round-2 evidence run: tests, bench lines (cfg 5 headline, cfg 3, cfg 4, reference arm), ncu launch list,
# K1 DRAM traffic, ncu --set full of the last cfg-5 sweep, per-stage sweeps
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_f.log 2>&1; echo smoke rc=$?
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_f.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_f.log
timeout 900 python bench.py > gpurun_out/bench_f.log 2>&1; echo bench rc=$?
tail -1 gpurun_out/bench_f.log | cut -c1-400
timeout 600 python bench.py --config 4 --no-cpu-baseline > gpurun_out/bench_f_cfg4.log 2>&1; echo cfg4 rc=$?
timeout 600 python bench.py --config 3 --no-cpu-baseline > gpurun_out/bench_f_cfg3.log 2>&1; echo cfg3 rc=$?
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_f_ref.log 2>&1; echo ref rc=$?
python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --pairs 1 > gpurun_out/plain_f.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r02.csv python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --pairs 1 > gpurun_out/ncu_launch_f.log 2>&1; echo launch rc=$?
DD_SERIAL_TIERS=1 timeout 1200 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --profile-from-start off -k regex:k1_cell --csv --log-file gpurun_out/k1_traffic_r02.csv python tools/profile_sweep.py --cfg 5 --profile-last --quiet > gpurun_out/ncu_traffic_f.log 2>&1; echo traffic rc=$?
DD_SERIAL_TIERS=1 timeout 1500 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:k1_cell -c 3 -o gpurun_out/r02f_k1_full python tools/profile_sweep.py --cfg 5 --profile-last --quiet > gpurun_out/ncu_full_f.log 2>&1; echo full rc=$?
timeout 300 python tools/profile_sweep.py --cfg 5 --quiet --json gpurun_out/sweeps_r02.json > gpurun_out/sweeps_r02.log 2>&1; echo sweeps rc=$?
