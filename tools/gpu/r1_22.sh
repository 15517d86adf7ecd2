set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2
timeout 600 python tools/profile_multiply.py --M 1408 --N 1408 --K 1982464 --bs 22 --path blocked --reps 2 2>&1 | tail -1
timeout 600 python tools/profile_multiply.py --M 5632 --N 5632 --K 5632 --bs 22 --path blocked --reps 3 2>&1 | tail -1
timeout 600 python tools/profile_multiply.py --M 11264 --N 11264 --K 11264 --bs 22 --path blocked --reps 2 2>&1 | tail -1
timeout 600 python tools/profile_multiply.py --M 5632 --N 5632 --K 5632 --bs 22 --path blocked --reps 2 > gpurun_out/r1_pm22.txt 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:smm22q -s 1 -c 1 -o gpurun_out/r1_smm22q_b python tools/profile_multiply.py --M 5632 --N 5632 --K 5632 --bs 22 --path blocked --reps 2 > gpurun_out/r1_ncu22.log 2>&1
tail -1 gpurun_out/r1_ncu22.log
