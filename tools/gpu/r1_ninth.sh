set -x
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -3
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 500 > gpurun_out/r1_bench9_clocks.csv &
CP=$!
timeout 1500 python bench.py > gpurun_out/r1_bench9_default.json 2> gpurun_out/r1_bench9_default.err
kill $CP
tail -2 gpurun_out/r1_bench9_default.err; cat gpurun_out/r1_bench9_default.json
timeout 300 python tools/profile_dgemm.py --M 63360 --N 63360 --K 16896 --reps 2 > gpurun_out/r1_pd9.txt 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:dgemm -s 1 -c 1 -o gpurun_out/r1_dgemm_persist python tools/profile_dgemm.py --M 63360 --N 63360 --K 16896 --reps 2 > gpurun_out/r1_ncu9.log 2>&1
tail -2 gpurun_out/r1_ncu9.log; cat gpurun_out/r1_pd9.txt
