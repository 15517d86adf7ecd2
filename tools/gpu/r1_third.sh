set -x
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
timeout 300 python tools/profile_dgemm.py --reps 3
timeout 300 python tools/profile_dgemm.py --M 1408 --N 1408 --K 1982464 --reps 3
timeout 900 python bench.py --config sq64 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline
timeout 900 python bench.py --config sq22 --path blocked --steps 1 --warmup 1 --no-e2e --no-cpu-baseline
timeout 900 python bench.py --config sq22 --path densified --steps 1 --warmup 3 --no-e2e --no-cpu-baseline
timeout 600 python bench.py --config r22 --path blocked --steps 2 --warmup 3 --no-e2e --no-cpu-baseline
timeout 600 python bench.py --config r64 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline
