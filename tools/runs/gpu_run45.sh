timeout 900 python -m pytest "tests/test_gpu_parity.py::test_edge_geometries" -m gpu -q 2>&1 | grep -E "RuntimeError|passed|failed" | head -8
