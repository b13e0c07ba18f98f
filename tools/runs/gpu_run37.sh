for v in A H A H; do
DD_LIB=paper_2001_10986_b200/libdd_gpu_$v.so timeout 300 python tools/profile_sweep.py --cfg 5 --quiet > gpurun_out/ab_$v.log 2>&1; echo $v $(tail -1 gpurun_out/ab_$v.log | cut -c1-60)
done
for v in profA profH; do DD_PROF_LIB=paper_2001_10986_b200/libdd_gpu_$v.so timeout 300 python tools/phase_profile.py --cfg 5 --min-side 2048 > gpurun_out/phase_$v.log 2>&1; echo $v; cat gpurun_out/phase_$v.log | grep "kappa 0.5"; done
