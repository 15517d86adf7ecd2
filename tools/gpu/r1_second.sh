set -x
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 500 > gpurun_out/r1_bench_clocks.csv &
CP=$!
timeout 1200 python bench.py > gpurun_out/r1_bench_default.json 2> gpurun_out/r1_bench_default.err
kill $CP
tail -3 gpurun_out/r1_bench_default.err; cat gpurun_out/r1_bench_default.json
timeout 600 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r1_plain.json 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r1_launches.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r1_ncu_list.log 2>&1
tail -2 gpurun_out/r1_ncu_list.log
timeout 300 python tools/profile_dgemm.py --reps 2 > gpurun_out/r1_profile_dgemm_plain.txt 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:dgemm -s 1 -c 1 -o gpurun_out/r1_dgemm_full python tools/profile_dgemm.py --reps 2 > gpurun_out/r1_ncu_full.log 2>&1
tail -3 gpurun_out/r1_ncu_full.log; cat gpurun_out/r1_profile_dgemm_plain.txt
