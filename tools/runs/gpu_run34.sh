for v in A B C; do DD_LIB=paper_2001_10986_b200/libdd_gpu_$v.so timeout 300 python tools/debug_s8.py 2>&1 | tail -30; done
