for bb in 80 96 120 80 96 120; do
timeout 300 python tools/profile_sweep.py --cfg 5 --quiet --bcap-big $bb > gpurun_out/bb_$bb.log 2>&1; echo bb=$bb $(tail -1 gpurun_out/bb_$bb.log | cut -c1-40)
done
