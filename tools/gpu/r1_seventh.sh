set -x
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -3
timeout 300 python tools/profile_multiply.py --M 8192 --N 8192 --K 8192 --bs 64 --path blocked --reps 3
timeout 300 python tools/profile_multiply.py --M 1408 --N 1408 --K 1982464 --bs 64 --path blocked --reps 2
