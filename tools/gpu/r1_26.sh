set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sparse.py -x -q 2>&1 | tail -3
