timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "big" > gpurun_out/pytest_big.log 2>&1; echo big rc=$?; tail -1 gpurun_out/pytest_big.log
for v in base cw base cw; do
DD_LIB=paper_2001_10986_b200/libdd_gpu_$v.so timeout 300 python tools/profile_sweep.py --cfg 5 --quiet > gpurun_out/ab_$v.log 2>&1; echo $v $(tail -1 gpurun_out/ab_$v.log | cut -c1-40)
done
