set -x
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -6
timeout 900 python -m pytest tests/test_gpu_fullsize.py -x -q 2>&1 | tail -6
timeout 900 python bench.py --config sq22 --path blocked --steps 1 --warmup 1 --no-e2e --no-cpu-baseline
timeout 600 python bench.py --config r22 --path blocked --steps 2 --warmup 3 --no-e2e --no-cpu-baseline
timeout 600 python bench.py --config r22 --path densified --steps 2 --warmup 3 --no-e2e --no-cpu-baseline
