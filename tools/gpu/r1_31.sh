set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "multiply_matches_oracle" 2>&1 | tail -2
timeout 600 python tools/profile_multiply.py --M 4096 --N 4096 --K 4096 --bs 4 --path blocked --reps 2 2>&1 | tail -1
timeout 600 python tools/profile_multiply.py --M 4096 --N 4096 --K 4096 --bs 8 --path blocked --reps 2 2>&1 | tail -1
timeout 600 python tools/profile_multiply.py --M 4095 --N 4095 --K 4095 --bs 5 --path blocked --reps 2 2>&1 | tail -1
