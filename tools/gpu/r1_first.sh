set -x
nvidia-smi --query-gpu=name,clocks.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -30 > gpurun_out/r1_pytest_gpu.txt; cat gpurun_out/r1_pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r1_smoke.txt 2>&1; cat gpurun_out/r1_smoke.txt
timeout 600 python bench.py --config r64 --steps 3 --warmup 3 --no-e2e --cpu-rows 2 > gpurun_out/r1_bench_r64.json 2> gpurun_out/r1_bench_r64.err; tail -3 gpurun_out/r1_bench_r64.err; cat gpurun_out/r1_bench_r64.json
timeout 900 python bench.py --config sq64 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/r1_bench_sq64.json 2> gpurun_out/r1_bench_sq64.err; tail -3 gpurun_out/r1_bench_sq64.err; cat gpurun_out/r1_bench_sq64.json
