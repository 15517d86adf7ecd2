set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "multiply_matches_oracle and (352 or 88-88 or 128-192 or 2816)" 2>&1 | tail -2
timeout 1800 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sparse.py -x -q -k "multiply_matches_oracle or sparse_multiply_matches or integer" 2>&1 | tail -15
