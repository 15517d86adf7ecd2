set -x
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -8
timeout 300 python tools/profile_multiply.py --M 11264 --N 11264 --K 11264 --bs 22 --path blocked --reps 3
timeout 900 python bench.py --config sq22 --path blocked --steps 1 --warmup 1 --no-e2e --no-cpu-baseline
timeout 600 python bench.py --config r22 --path blocked --steps 2 --warmup 3 --no-e2e --no-cpu-baseline
timeout 300 python tools/profile_multiply.py --M 5632 --N 5632 --K 5632 --bs 22 --path blocked --reps 2 > gpurun_out/r1_pm_plain.txt 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:smm22 -s 1 -c 1 -o gpurun_out/r1_smm22b_full python tools/profile_multiply.py --M 5632 --N 5632 --K 5632 --bs 22 --path blocked --reps 2 > gpurun_out/r1_ncu_smm.log 2>&1
tail -3 gpurun_out/r1_ncu_smm.log
