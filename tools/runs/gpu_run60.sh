DD_LIB=paper_2001_10986_b200/libdd_gpu_B2.so timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "big_tier or s8 or edge" 2>&1 | tail -1
for v in B1 B2 B1 B2; do
DD_LIB=paper_2001_10986_b200/libdd_gpu_$v.so timeout 300 python tools/profile_sweep.py --cfg 5 --quiet > gpurun_out/ab_$v.log 2>&1; echo $v $(tail -1 gpurun_out/ab_$v.log | cut -c1-60)
done
