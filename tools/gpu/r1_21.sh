set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "multiply" 2>&1 | tail -2
timeout 600 python tools/profile_multiply.py --M 1408 --N 1408 --K 1982464 --bs 22 --path blocked --reps 2 2>&1 | tail -1
timeout 600 python tools/profile_multiply.py --M 5632 --N 5632 --K 5632 --bs 22 --path blocked --reps 3 2>&1 | tail -1
timeout 600 python tools/profile_multiply.py --M 11264 --N 11264 --K 11264 --bs 22 --path blocked --reps 2 2>&1 | tail -1
