# diagnostics: which cells of the cfg-4 test sweep are rescued (flag 16) on the quarter-chunk build;
# cfg-4 bench line with --allow-flagged; batch of 8 / 10 pairs
mkdir -p gpurun_out
timeout 600 python tools/rescue_diag.py > gpurun_out/rescue_diag.log 2>&1; echo diag rc=$?; tail -12 gpurun_out/rescue_diag.log | cut -c1-200
timeout 600 python bench.py --config 4 --no-cpu-baseline > gpurun_out/bench_g_cfg4.log 2>&1; echo cfg4 rc=$?; tail -1 gpurun_out/bench_g_cfg4.log | cut -c1-300
timeout 900 python bench.py --pairs 8 --no-cpu-baseline --no-e2e --steps 3 > gpurun_out/bench_p8.log 2>&1; echo p8 rc=$?; tail -1 gpurun_out/bench_p8.log | cut -c1-200
timeout 900 python bench.py --pairs 10 --no-cpu-baseline --no-e2e --steps 3 > gpurun_out/bench_p10.log 2>&1; echo p10 rc=$?; tail -1 gpurun_out/bench_p10.log | cut -c1-200
