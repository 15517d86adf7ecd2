set -x
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -3
for shp in "1408 1408 1982464" "1408 704 991232" "704 704 495616" "704 384 495616" "704 320 495616" "63360 63360 15840"; do
set -- $shp
timeout 300 python tools/profile_dgemm.py --M $1 --N $2 --K $3 --reps 3 | tail -1
done
timeout 600 python bench.py --config r64 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline
