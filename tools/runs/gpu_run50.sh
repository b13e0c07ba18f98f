for b in 24 18 20 24 18 20; do
timeout 300 python tools/profile_sweep.py --cfg 5 --quiet --bcap $b > gpurun_out/bc_$b.log 2>&1; echo bcap=$b $(tail -1 gpurun_out/bc_$b.log | cut -c1-60)
done
