timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for v in K2 gpu K2 gpu; do
DD_LIB=paper_2001_10986_b200/libdd_$v.so; [ $v = K2 ] && DD_LIB=paper_2001_10986_b200/libdd_gpu_K2.so
DD_LIB=$DD_LIB timeout 300 python tools/profile_sweep.py --cfg 5 --quiet > gpurun_out/ab_$v.log 2>&1; echo $v $(tail -1 gpurun_out/ab_$v.log | cut -c1-60)
done
