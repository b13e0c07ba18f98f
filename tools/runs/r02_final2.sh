# round-2 final evidence on the DD_FV2 tree (the GPU suite ran green on this same libdd_gpu.so in r02_v13.sh):
# smoke, bench A/B against the DD_FV2=0 build (F0), bench lines (cfg 5 headline, cfg 4 one pair, cfg 3, reference arm),
# ncu launch list, K1 DRAM traffic, ncu --set full of the last cfg-5 sweep, per-stage sweeps
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_f.log 2>&1; echo smoke rc=$?
DD_LIB=paper_2001_10986_b200/libdd_gpu_F0.so timeout 600 python bench.py --no-e2e --no-cpu-baseline --steps 3 > gpurun_out/bench_F0_a.log 2>&1; echo F0a rc=$?
tail -1 gpurun_out/bench_F0_a.log | cut -c1-120
timeout 900 python bench.py > gpurun_out/bench_f.log 2>&1; echo bench rc=$?
tail -1 gpurun_out/bench_f.log | cut -c1-400
DD_LIB=paper_2001_10986_b200/libdd_gpu_F0.so timeout 600 python bench.py --no-e2e --no-cpu-baseline --steps 3 > gpurun_out/bench_F0_b.log 2>&1; echo F0b rc=$?
tail -1 gpurun_out/bench_F0_b.log | cut -c1-120
timeout 600 python bench.py --config 4 --pairs 1 --no-cpu-baseline > gpurun_out/bench_f_cfg4.log 2>&1; echo cfg4 rc=$?
timeout 600 python bench.py --config 3 --no-cpu-baseline > gpurun_out/bench_f_cfg3.log 2>&1; echo cfg3 rc=$?
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_f_ref.log 2>&1; echo ref rc=$?
python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --pairs 1 > gpurun_out/plain_f.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r02.csv python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --pairs 1 > gpurun_out/ncu_launch_f.log 2>&1; echo launch rc=$?
DD_SERIAL_TIERS=1 timeout 1200 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --profile-from-start off -k regex:k1_cell --csv --log-file gpurun_out/k1_traffic_r02.csv python tools/profile_sweep.py --cfg 5 --profile-last --quiet > gpurun_out/ncu_traffic_f.log 2>&1; echo traffic rc=$?
DD_SERIAL_TIERS=1 timeout 1500 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:k1_cell -c 3 -o gpurun_out/r02g_k1_full python tools/profile_sweep.py --cfg 5 --profile-last --quiet > gpurun_out/ncu_full_f.log 2>&1; echo full rc=$?
timeout 300 python tools/profile_sweep.py --cfg 5 --quiet --json gpurun_out/sweeps_r02.json > gpurun_out/sweeps_r02.log 2>&1; echo sweeps rc=$?
