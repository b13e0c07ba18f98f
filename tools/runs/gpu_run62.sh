DD_LIB=paper_2001_10986_b200/libdd_gpu_C2.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_striped_gpu.py -m gpu -x -q 2>&1 | tail -1
for v in C1 C2 C1 C2; do
DD_LIB=paper_2001_10986_b200/libdd_gpu_$v.so timeout 300 python tools/profile_sweep.py --cfg 5 --quiet --json gpurun_out/sw_$v.json > gpurun_out/ab_$v.log 2>&1; echo $v $(tail -1 gpurun_out/ab_$v.log | cut -c1-60)
done
