mkdir -p gpurun_out
timeout 300 python tools/profile_sweep.py --cfg 4 --profile-last --quiet > gpurun_out/plain16.log 2>&1 && \
timeout 1500 ncu --section SpeedOfLight --section ComputeWorkloadAnalysis --section WarpStateStats --section InstructionStats --section SourceCounters --section Occupancy --section SchedulerStats --section LaunchStats --clock-control none --import-source on --profile-from-start off -k regex:k1_cell -o gpurun_out/k1_cfg4_v7 -f python tools/profile_sweep.py --cfg 4 --profile-last --quiet > gpurun_out/ncu_cfg4_v7.log 2>&1; echo ncu rc=$?
tail -2 gpurun_out/ncu_cfg4_v7.log
