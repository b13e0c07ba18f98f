# Phase A quarter chunks (DD_PA_Q=1, default build = libdd_gpu_Q.so) vs BASE (DD_PA_Q=0): parity of Q, then alternating A/B, waste model
mkdir -p gpurun_out
cp paper_2001_10986_b200/libdd_gpu_Q.so paper_2001_10986_b200/libdd_gpu.so
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_cluster_gpu.py tests/test_fullsize_gpu.py -m gpu -q -x > gpurun_out/pytest_q.log 2>&1; echo q-tests rc=$?
tail -3 gpurun_out/pytest_q.log
bash tools/ab_test.sh BASE Q
bash tools/ab_test.sh BASE Q
DD_LIB=paper_2001_10986_b200/libdd_gpu_Q.so timeout 300 python tools/waste_model.py --cfg 5 > gpurun_out/waste_q.log 2>&1; echo waste rc=$?
tail -9 gpurun_out/waste_q.log
DD_LIB=paper_2001_10986_b200/libdd_gpu_Q.so DD_SERIAL_TIERS=1 timeout 1500 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:k1_cell -c 3 -o gpurun_out/r02_q_k1_full python tools/profile_sweep.py --cfg 5 --profile-last --quiet > gpurun_out/ncu_q_full.log 2>&1; echo ncu rc=$?
tail -3 gpurun_out/ncu_q_full.log
