# A/B: phase A on live (row, column) points (DD_PA_LIVE=1) vs the chunk layout; parity of the variant first
mkdir -p gpurun_out
DD_LIB=paper_2001_10986_b200/libdd_gpu_PAL.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_cluster_gpu.py tests/test_fullsize_gpu.py -m gpu -q -x > gpurun_out/pytest_pal.log 2>&1; echo pal-tests rc=$?
tail -3 gpurun_out/pytest_pal.log
bash tools/ab_test.sh BASE PAL
DD_LIB=paper_2001_10986_b200/libdd_gpu_BASE.so timeout 300 python tools/waste_model.py --cfg 5 > gpurun_out/waste_r02.log 2>&1; echo waste rc=$?
tail -20 gpurun_out/waste_r02.log
