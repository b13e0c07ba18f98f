# Experiment: tier 2 as 384 threads x 2 CTAs/SM (T2H) vs 768 x 1 (Q), boxes > 250 to tier G in both (same cells per tier);
# serialised tiers, ncu launch durations of the last cfg-5 sweep
mkdir -p gpurun_out
for v in Q T2H Q T2H; do
DD_LIB=paper_2001_10986_b200/libdd_gpu_$v.so DD_SERIAL_TIERS=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off -k regex:k1_cell --csv --log-file gpurun_out/t2h_$v.csv python tools/profile_sweep.py --cfg 5 --profile-last --onchip 250 --quiet > gpurun_out/t2h_$v.log 2>&1; echo $v rc=$?
grep -h "k1_cell" gpurun_out/t2h_$v.csv | awk -F'","' '{print $5, $(NF)}' | cut -c1-120
done
for v in Q T2H; do
DD_LIB=paper_2001_10986_b200/libdd_gpu_$v.so timeout 300 python tools/profile_sweep.py --cfg 5 --onchip 250 --quiet > gpurun_out/t2hw_$v.log 2>&1; echo $v wall $(tail -1 gpurun_out/t2hw_$v.log | cut -c1-40)
done
