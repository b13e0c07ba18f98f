mkdir -p gpurun_out
timeout 300 python tools/sanitize_small.py > gpurun_out/plain28.log 2>&1 && \
timeout 1500 compute-sanitizer --tool memcheck --print-limit 20 python tools/sanitize_small.py > gpurun_out/memcheck.log 2>&1; echo memcheck rc=$?
tail -8 gpurun_out/memcheck.log
