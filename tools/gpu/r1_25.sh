set -x
timeout 900 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r1_b25.json 2>&1 && \
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r1_launches_sq64.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r1_ncu25a.log 2>&1
tail -1 gpurun_out/r1_ncu25a.log
timeout 900 python bench.py --config sq22 --path blocked --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r1_b25b.json 2>&1 && \
timeout 2400 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/r1_launches_sq22_blocked.csv python bench.py --config sq22 --path blocked --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r1_ncu25b.log 2>&1
tail -1 gpurun_out/r1_ncu25b.log
