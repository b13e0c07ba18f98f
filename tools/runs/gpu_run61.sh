python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke61.log 2>&1; echo smoke rc=$?
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
