set -x
timeout 600 python tools/profile_multiply.py --M 15840 --N 15840 --K 15840 --bs 22 --path blocked --reps 2 > /dev/null 2>&1 && \
timeout 1200 ncu --set full --clock-control none -k regex:"stackgen_kernel|undensify" -s 0 -c 1 -o gpurun_out/r1_stackgen python tools/profile_multiply.py --M 15840 --N 15840 --K 15840 --bs 22 --path blocked --reps 1 > gpurun_out/r1_ncu33.log 2>&1
tail -1 gpurun_out/r1_ncu33.log
