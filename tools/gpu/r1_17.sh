set -x
timeout 600 python tools/profile_multiply.py --M 1408 --N 1408 --K 1982464 --bs 64 --path densified --reps 2 > gpurun_out/r1_pm17.txt 2>&1 && \
timeout 1200 ncu --set full --clock-control none -k regex:densify -s 0 -c 2 -o gpurun_out/r1_densify_r64 python tools/profile_multiply.py --M 1408 --N 1408 --K 1982464 --bs 64 --path densified --reps 1 > gpurun_out/r1_ncu17.log 2>&1
tail -2 gpurun_out/r1_ncu17.log; cat gpurun_out/r1_pm17.txt
