set -x
for o in q lj; do
  DBM_DENSIFY_B_ORDER=$o timeout 600 python tools/profile_multiply.py --M 1408 --N 1408 --K 1982464 --bs 64 --path densified --reps 3 2>&1 | tail -1
  DBM_DENSIFY_B_ORDER=$o timeout 600 python tools/profile_multiply.py --M 1408 --N 1408 --K 1982464 --bs 22 --path densified --reps 3 2>&1 | tail -1
done
timeout 600 python tools/profile_multiply.py --M 31680 --N 31680 --K 31680 --bs 64 --path densified --reps 2 2>&1 | tail -1
timeout 600 python tools/profile_multiply.py --M 1408 --N 1408 --K 1982464 --bs 64 --path densified --reps 2 > gpurun_out/r1_pm17.txt 2>&1 && \
timeout 1200 ncu --set full --clock-control none -k regex:densify -s 0 -c 2 -o gpurun_out/r1_densify_r64 python tools/profile_multiply.py --M 1408 --N 1408 --K 1982464 --bs 64 --path densified --reps 1 > gpurun_out/r1_ncu17.log 2>&1
tail -2 gpurun_out/r1_ncu17.log
