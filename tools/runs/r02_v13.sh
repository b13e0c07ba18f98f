# A/B of the fused-pass control variant (DD_FV2: F1 = on, F0 = off) on the cfg-5 schedule, then the GPU suite on F1
# (rescue tests first: DD_FORCE_RESCUE hook), cfg-4 bench line on one pair
mkdir -p gpurun_out
bash tools/ab_test.sh F0 F1 2>&1 | tee gpurun_out/ab_fv2.log
timeout 600 python -m pytest tests/test_rescue_gpu.py -m gpu -q > gpurun_out/pytest_rescue.log 2>&1; echo rescue rc=$?
tail -3 gpurun_out/pytest_rescue.log
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_fv2.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_fv2.log
timeout 500 python bench.py --config 4 --pairs 1 --no-cpu-baseline > gpurun_out/bench_g_cfg4.log 2>&1; echo cfg4 rc=$?; tail -1 gpurun_out/bench_g_cfg4.log | cut -c1-300
